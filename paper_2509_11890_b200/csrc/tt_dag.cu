// tt_dag.cu — host side of the persistent DAG executor (tt_dag.cuh): recording of stage GEMMs
// into tasks, the unit-size policy, topological queue order and the single launch.
//
// A sweep that runs on the DAG executor is written exactly like its stream version: the stage
// planners (enqueue_left / enqueue_right_mirror / enqueue_matvec_last, tt_core.cu) call
// launch_gemm, which appends a task to the active DagBuilder instead of launching.  Each task
// depends on the previous task of its lane (the stream it would have run on) plus the explicit
// dependencies the caller adds (the events it would have waited on).
#include "tt_internal.cuh"
#include "tt_dag.cuh"

namespace ttint {

thread_local DagBuilder* g_dag = nullptr;
thread_local int g_dag_mode = 0;
thread_local unsigned long long* g_dag_trace = nullptr;   // tt_debug_dag_trace
thread_local long long g_dag_trace_cap = 0;
thread_local int g_dag_last_units = 0, g_dag_last_tasks = 0;
thread_local std::vector<int> g_dag_last_unit0;   // first unit of each queued task (trace decoding)

namespace {
constexpr int kDagBM = 64, kDagBN = 64;

struct DagKernelInfo {
  int dev = -1;
  int per_sm[4] = {0, 0, 0, 0};
  cudaError_t err = cudaSuccess;
};
thread_local DagKernelInfo g_dag_info;

template <int BM, int BN, int WM, int WN, int ST, int MINB>
cudaError_t dag_launch_cfg(const tt::DagParams& prm, int slot, cudaStream_t s, int* grid_out) {
  using Cfg = tt::DagCfg<BM, BN, WM, WN, ST>;
  auto kern = tt::dag_gemm_kernel<BM, BN, WM, WN, ST, MINB>;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (g_dag_info.dev != dev) {
    g_dag_info = DagKernelInfo{};
    g_dag_info.dev = dev;
  }
  if (g_dag_info.per_sm[slot] == 0) {
    // per device: the attribute and the occupancy are queried on the current device
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Cfg::kSmemBytes)) != cudaSuccess)
      return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::kThreads,
                                                           Cfg::kSmemBytes)) != cudaSuccess)
      return e;
    g_dag_info.per_sm[slot] = std::max(per_sm, 1);
  }
  const long long slots = (long long)num_sms() * g_dag_info.per_sm[slot];
  const int grid = (int)std::max<long long>(1, std::min<long long>(prm.total_units, slots));
  *grid_out = grid;
  return launch_pdl(true, kern, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmemBytes, s, prm);
}
}  // namespace

size_t dag_scratch_bytes(long long partial_elems) {
  return align_up(sizeof(int) * (size_t)kDagCounterInts, 256) +
         align_up((size_t)partial_elems * sizeof(double), 256) + 256;
}

DagBuilder::DagBuilder(void* scratch, size_t bytes) {
  if (!scratch) {   // dry run: sizes the split-K partials, never launched
    dry = true;
    part_cap = 1LL << 60;
    return;
  }
  char* b = static_cast<char*>(scratch);
  char* c = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(b) + 255) & ~uintptr_t(255));
  const size_t cbytes = align_up(sizeof(int) * (size_t)kDagCounterInts, 256);
  if (bytes < (size_t)(c - b) + cbytes) {
    ok = false;
    return;
  }
  ctr = reinterpret_cast<int*>(c);
  part = reinterpret_cast<double*>(c + cbytes);
  part_cap = (long long)((bytes - (size_t)(c - b) - cbytes) / sizeof(double));
}

void DagBuilder::set_lane(int l) {
  if (l >= (int)lane_last.size()) lane_last.resize(size_t(l) + 1, -1);
  lane = l;
}

int DagBuilder::last_of(int l) const {
  return l < (int)lane_last.size() ? lane_last[size_t(l)] : -1;
}

// launch_gemm's recording path: one task per stage GEMM, with its unit-size policy
cudaError_t DagBuilder::add(bool a_kc, bool b_kc, const GemmParams& p) {
  if (!ok) return cudaErrorInvalidValue;
  const long long lim = (1LL << 31) - 1024;
  if (p.M >= lim || p.N >= lim || p.K >= lim || p.lda >= lim || p.ldb >= lim ||
      (int)tasks.size() >= tt::kDagMaxTasks) {
    ok = false;
    return cudaErrorInvalidValue;
  }
  tt::DagTask t{};
  t.A = p.A;
  t.B = p.B;
  t.C = p.C;
  t.P = nullptr;
  t.M = (int)p.M;
  t.N = (int)p.N;
  t.K = (int)p.K;
  t.lda = (int)p.lda;
  t.ldb = (int)p.ldb;
  t.rowmap = tt::to_map32(p.rowmap);
  t.colmap = tt::to_map32(p.colmap);
  const bool av = aligned16(p.A) && !(p.lda & 1) && !((a_kc ? p.K : p.M) & 1);
  const bool bv = aligned16(p.B) && !(p.ldb & 1) && !((b_kc ? p.K : p.N) & 1);
  t.flags = (a_kc ? 1 : 0) | (b_kc ? 2 : 0) | (av ? 4 : 0) | (bv ? 8 : 0);
  const long long tm = (p.M + kDagBM - 1) / kDagBM, tn = (p.N + kDagBN - 1) / kDagBN;
  t.tiles_n = (int)tn;
  t.KT = (int)((p.K + 15) / 16);
  // split-K: enough units to spread a small stage over the GPU, each unit >= 4 k-tiles
  long long ks = 1;
  const long long tiles = tm * tn;
  if (tiles < target_units) {
    ks = std::min<long long>((target_units + tiles - 1) / tiles, std::max(1, t.KT / 4));
    ks = std::min<long long>(ks, tt::kDagMaxSplit);
  }
  long long kper = (t.KT + ks - 1) / ks;
  ks = (t.KT + kper - 1) / kper;   // no empty split
  if (ks > 1) {
    const long long need = ks * p.M * p.N;
    if (part_used + need > part_cap || ticks + tiles > kDagCounterInts - 1 - tt::kDagMaxTasks) {
      ks = 1;
      kper = t.KT;
    } else {
      t.P = part + part_used;
      part_used += (need + 31) & ~31LL;
      t.tick0 = (int)ticks;
      ticks += tiles;
    }
  }
  t.ksplit = (int)ks;
  t.kt_per_split = (int)kper;
  Node nd;
  nd.t = t;
  nd.tiles = (int)tiles;
  nd.units = (int)(tiles * ks);
  const int prev = last_of(lane);
  if (prev >= 0) nd.deps.push_back(prev);
  for (int d0 : pending) nd.deps.push_back(d0);
  pending.clear();
  std::sort(nd.deps.begin(), nd.deps.end());
  nd.deps.erase(std::unique(nd.deps.begin(), nd.deps.end()), nd.deps.end());
  if ((int)nd.deps.size() > tt::kDagMaxDeps) {
    ok = false;
    return cudaErrorInvalidValue;
  }
  tasks.push_back(nd);
  lane_last[size_t(lane)] = (int)tasks.size() - 1;
  return cudaSuccess;
}

cudaError_t DagBuilder::launch(cudaStream_t s) {
  if (!ok || dry) return cudaErrorInvalidValue;
  if (tasks.empty()) return cudaSuccess;
  const int nt = (int)tasks.size();
  // queue order: by DAG level (longest dependency chain above the task), then recording order
  std::vector<int> level(nt, 0), order(nt, 0);
  for (int i = 0; i < nt; ++i) {
    for (int d0 : tasks[size_t(i)].deps) level[size_t(i)] = std::max(level[size_t(i)], level[size_t(d0)] + 1);
    order[size_t(i)] = i;
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return level[size_t(a)] < level[size_t(b)]; });
  std::vector<int> pos(nt, 0);
  for (int i = 0; i < nt; ++i) pos[size_t(order[size_t(i)])] = i;
  static_assert(sizeof(tt::DagParams) <= 32000, "kernel parameter block");
  std::unique_ptr<tt::DagParams> prm(new tt::DagParams{});
  prm->ntasks = nt;
  prm->ctr = ctr;
  long long units = 0;
  for (int i = 0; i < nt; ++i) {
    const Node& nd = tasks[size_t(order[size_t(i)])];
    tt::DagTask t = nd.t;
    t.unit0 = (int)units;
    units += nd.units;
    t.ndeps = (int)nd.deps.size();
    for (int q = 0; q < t.ndeps; ++q) {
      t.dep[q] = pos[size_t(nd.deps[size_t(q)])];
      t.need[q] = tasks[size_t(nd.deps[size_t(q)])].tiles;
    }
    prm->t[i] = t;
  }
  if (units >= (1LL << 31) - 1) return cudaErrorInvalidValue;
  prm->total_units = (int)units;
  prm->trace = (g_dag_trace && units <= g_dag_trace_cap) ? g_dag_trace : nullptr;
  g_dag_last_units = (int)units;
  g_dag_last_tasks = nt;
  g_dag_last_unit0.assign(size_t(nt) + 1, (int)units);
  for (int i = 0; i < nt; ++i) g_dag_last_unit0[size_t(i)] = prm->t[i].unit0;
  cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(int) * (size_t)(1 + nt + ticks), s);
  if (e != cudaSuccess) return e;
  ++g_launches;
  g_stage = TT_ST_DAG;
  int grid = 0;
  const long long tr = trace_begin(nt, units, 0, 0, s);
  if (g_dag_mode == 2)
    e = dag_launch_cfg<64, 64, 2, 4, 4, 2>(*prm, 1, s, &grid);
  else
    e = dag_launch_cfg<64, 64, 2, 2, 4, 2>(*prm, 0, s, &grid);
  trace_end(tr, s);
  ++g_launches;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace ttint
