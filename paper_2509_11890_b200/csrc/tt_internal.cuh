// tt_internal.cuh — declarations shared by the translation units of libtt_hotpath.so
// (tt_core.cu, tt_launch.cu, tt_api.cu, tt_solvers.cu, tt_dag.cu).  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <functional>
#include <initializer_list>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/tt_hotpath.h"
#include "tt_gemm.cuh"
#include "tt_gemm_v2.cuh"
#include "tt_dag.cuh"

using tt::GemmParams;
using tt::IndexMap;

namespace ttint {

// ---- per-thread state (definitions in tt_core.cu / tt_launch.cu) ----------------------------
extern thread_local std::string g_msg;
extern thread_local int64_t g_launches;
extern thread_local int64_t g_launches_last;
extern thread_local bool g_trace_on;
extern thread_local int g_stage;              // stage tag of the next launch (tracer)
extern thread_local int g_side_lowprio;
extern thread_local int g_dbg_flags;          // tt_debug_set_flags (bits in tt_hotpath_debug.h)
extern thread_local bool g_no_pdl;
extern thread_local int g_variant;
extern thread_local int g_force_ks;
extern thread_local const int* g_gate;        // device flag gating the solvers' GEMMs
extern thread_local double* g_pscratch;       // split-K scratch of the current stage
extern thread_local long long g_pscratch_elems;
extern thread_local int g_force_v1;
extern thread_local int g_eigen_elementwise;
extern thread_local int g_dag_mode;

struct TraceRec {
  int stage, tile;
  long long M, N, K;
  cudaEvent_t e0, e1;
};

struct SideStream {
  int dev = -1;
  cudaStream_t s = nullptr;
  cudaStream_t s_lo = nullptr;   // same, lowest priority (A/B hook: debug flag 2048)
  cudaEvent_t ev[64] = {};
  unsigned next = 0;
  void release();
};

constexpr int kPoolStreams = 4;
struct StreamPool {
  int dev = -1;
  cudaStream_t s[kPoolStreams] = {};
  cudaStream_t chain = nullptr;     // high priority (the W34 left chain)
  cudaStream_t capture = nullptr;   // graph-cache capture stream
  std::vector<cudaEvent_t> ev;
  void release();
};

struct GraphKey {
  std::vector<uint64_t> w;
  GraphKey& add(uint64_t v) { w.push_back(v); return *this; }
  GraphKey& add(const void* p) { w.push_back((uint64_t)(uintptr_t)p); return *this; }
  template <typename T>
  GraphKey& arr(const T* a, int64_t n) {   // host array contents (extents or pointers)
    w.push_back((uint64_t)(a != nullptr));
    if (a)
      for (int64_t i = 0; i < n; ++i) w.push_back((uint64_t)(uintptr_t)a[i]);
    return *this;
  }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
  uint64_t last = 0;
};

struct ThreadRes {   // tt_core.cu: everything a thread's calls created, destroyed at thread exit
  SideStream side;
  StreamPool pool;
  std::vector<SideStream> side_parked;
  std::vector<StreamPool> pool_parked;
  std::vector<GraphEntry> graphs;
  std::vector<GraphKey> seen;
  uint64_t clock = 0;
  ~ThreadRes();
};

struct Carver {
  char* base;
  size_t cap, off = 0;
  bool ok = true;
  double* take(long long elems) {
    uintptr_t p = reinterpret_cast<uintptr_t>(base) + off;
    uintptr_t q = (p + 255) & ~uintptr_t(255);
    size_t need = (q - reinterpret_cast<uintptr_t>(base)) + size_t(elems) * sizeof(double);
    if (need > cap) {
      ok = false;
      return nullptr;
    }
    off = need;
    return reinterpret_cast<double*>(q);
  }
};

constexpr int kPrepMax = 40;
struct PrepTable {
  const double* A[kPrepMax];
  const double* x[kPrepMax];
  double* Ahl[kPrepMax];
  double* Ahr[kPrepMax];
  double* xt[kPrepMax];
  int al[kPrepMax], n[kPrepMax], be[kPrepMax], a[kPrepMax], b[kPrepMax];
  int start[kPrepMax + 1];
  int cores;
  double* one0;
  double* one1;
};

struct Dims {
  long long a, n, b, al, be;
};

constexpr int kSmallChainMax = 8;
struct SmallChain {   // a run of consecutive small left updates in one CTA (tt_core.cu)
  int cores;
  int pmax;                             // doubles reserved for the running input interface
  int a[kSmallChainMax], b[kSmallChainMax], al[kSmallChainMax], be[kSmallChainMax],
      n[kSmallChainMax];
  const double* phi_in;                 // interface into the first core
  const double* x[kSmallChainMax];      // vector core (a, n, b) (or the transposed core)
  const double* Ah[kSmallChainMax];     // operator core in the prepared layout (al, j, i, be)
  double* phi_out[kSmallChainMax];      // output interfaces (b, be, b)
  double* T2keep[kSmallChainMax];       // optional stage-2 intermediates (a, n, be, b)
};

struct SplitScratch {   // scopes the split-K scratch to one stage launch
  SplitScratch(double* p, long long n) {
    g_pscratch = p;
    g_pscratch_elems = n;
  }
  ~SplitScratch() {
    g_pscratch = nullptr;
    g_pscratch_elems = 0;
  }
};

struct DimsPG {
  long long ap, a, n, bp, b, al, be;
};

struct CallScope {
  CallScope() {
    g_msg.clear();
    g_launches = 0;
  }
  ~CallScope() { g_launches_last = g_launches; }
};

extern thread_local std::vector<TraceRec> g_trace;
extern thread_local std::vector<cudaEvent_t> g_trace_pool;
extern thread_local ThreadRes g_res;
extern thread_local int g_graph_cache_on;

// ---- helpers (tt_core.cu) ---------------------------------------------------------------------
cudaError_t side_stream(cudaStream_t* out);
cudaError_t stream_dep(cudaStream_t from, cudaStream_t to);
cudaError_t pool_init(size_t nevents);
cudaError_t smem_attr(const void* kern, int bytes);   // per device opt-in shared memory
// eager multi-launch calls: replayed from a per-thread CUDA graph cache from the second call on
tt_status graph_cached(GraphKey& key, cudaStream_t s,
                       const std::function<tt_status(cudaStream_t)>& enqueue, const char* where);
void graph_cache_clear();
long long trace_begin(int tile, long long M, long long N, long long K, cudaStream_t s);
void trace_end(long long idx, cudaStream_t s);
tt_status fail(tt_status s, const std::string& m);
tt_status cuda_fail(cudaError_t e, const char* where);
bool mulc(long long& acc, long long v);
long long prod(std::initializer_list<long long> xs, bool& ok);
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
size_t ws_bytes(std::initializer_list<long long> elems);
double pdl_flops();
bool dims_valid(const Dims& d);
bool dims_pg_valid(const DimsPG& d);
tt_status check_dims(const Dims& d);
bool same(const void* p, const void* q);

// Launch with programmatic stream serialisation (PDL, tt_gemm.cuh pdl_wait/pdl_trigger) when
// `pdl`: the kernel may be scheduled while its stream predecessor drains and waits for it on
// the device.  Only kernels that call pdl_wait() before touching global memory are launched
// this way, and only latency-bound ones (small GEMMs, their split-K reduction, the sweep
// preparation): for the large matvec GEMMs of W5 the early-resident dependents hold SMs the
// concurrent interface chain could use (measured +1.1 % on the W5 sweep with PDL everywhere).
// Debug flag 4096 disables PDL (A/B).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && !g_no_pdl && !(g_dbg_flags & 4096)) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


// ---- GEMM launch policy (tt_launch.cu) ----------------------------------------------------------
int num_sms();
bool aligned16(const void* q);
bool v2_eligible(bool a_kc, bool b_kc, const GemmParams& p);
cudaError_t launch_gemm(bool a_kc, bool b_kc, const GemmParams& p, cudaStream_t s);
GemmParams gp(const double* A, long long lda, const double* B, long long ldb, double* C,
              long long M, long long N, long long K, IndexMap rm, IndexMap cm);

// ---- small kernels and stage plans (tt_core.cu) -------------------------------------------------
__global__ void __launch_bounds__(256) prep_all_kernel(const __grid_constant__ PrepTable t);
size_t small_chain_smem(const Dims& d);
size_t small_chain_work(const Dims& d);
bool small_update(const Dims& d);
cudaError_t launch_small_chain(const SmallChain& c, size_t smem, cudaStream_t s);
cudaError_t launch_perm(bool left, const double* A, double* out, long long al, long long n,
                        long long be, cudaStream_t s);
bool matvec_ws_elems(const Dims& d, long long K, long long& t1, long long& t2, long long& ah,
                     long long& pe);
bool iface_ws_elems(const Dims& d, long long& t1, long long& t2, long long& ah, long long& pe);
bool pg_ws_elems(const DimsPG& d, long long K, long long& t1, long long& t2, long long& ah,
                 long long& pe);
cudaError_t enqueue_matvec_last(const Dims& d, long long K, const double* T2, const double* phiR,
                                double* Y, double* P, long long pe, cudaStream_t s);
cudaError_t enqueue_matvec(const Dims& d, long long K, const double* phiL, const double* A,
                           const double* phiR, const double* X, double* Y, double* T1,
                           double* T2, double* Ah, double* P, long long pe, cudaStream_t s,
                           const double* Ah_pre = nullptr);
cudaError_t enqueue_left(const Dims& d, const double* phiL, const double* A, const double* x,
                         double* out, double* T1, double* T2, double* Ah, double* P,
                         long long pe, cudaStream_t s, int tag_s1 = TT_ST_IL_S1,
                         const double* Ah_pre = nullptr, cudaEvent_t ev_t2 = nullptr);
cudaError_t enqueue_right_mirror(const Dims& d, const double* phiR, const double* A,
                                 const double* x, double* out, double* T1, double* T2,
                                 double* Ah, double* P, long long pe, cudaStream_t s,
                                 const double* Ahr_pre = nullptr, const double* xt_pre = nullptr);
cudaError_t enqueue_right(const Dims& d, const double* phiR, const double* A, const double* x,
                          double* out, double* T1, double* T2, double* At, double* P,
                          long long pe, cudaStream_t s);
cudaError_t enqueue_matvec_pg(const DimsPG& d, long long K, const double* phiL, const double* A,
                              const double* phiR, const double* X, double* Y, double* T1,
                              double* T2, double* Ah, double* P, long long pe, cudaStream_t s);
cudaError_t enqueue_left_pg(const DimsPG& d, const double* phiL, const double* A,
                            const double* xb, const double* xk, double* out, double* T1,
                            double* T2, double* Ah, double* P, long long pe, cudaStream_t s);
cudaError_t enqueue_right_pg(const DimsPG& d, const double* phiR, const double* A,
                             const double* xb, const double* xk, double* out, double* T1,
                             double* T2, double* At, double* P, long long pe, cudaStream_t s);

// ---- fused S1 -> S2 matvec kernel (tt_fused.cu / tt_fused12.cuh) ---------------------------------
extern thread_local int g_fused_mode;
extern thread_local bool g_fused_misaligned;
bool fused12_shape_ok(const Dims& d, long long K);
bool fused12_wanted(const Dims& d, long long K);   // explicit fused mode: no T1 in the workspace
bool fused12_auto(const Dims& d, long long K);     // AUTO policy (T1 kept as the fallback)
bool fused12_iface_wanted(const Dims& d);   // interface updates keep their T1 workspace
cudaError_t launch_fused12(const Dims& d, long long K, const double* phiL, const double* Ah,
                           const double* X, double* T2, cudaStream_t s, bool& ok,
                           int stage_tag = TT_ST_MV_S1);

// ---- symmetric eigensolver (tt_solvers.cu) ------------------------------------------------------
extern thread_local int g_eigen_elementwise;
long long sym_eigen_scratch(long long n);
cudaError_t launch_sym_eigen(const double* G, double* V, double* lam, int n, double* scratch,
                             cudaStream_t s);

// ---- persistent DAG executor (tt_dag.cu / tt_dag.cuh) -------------------------------------------
// While a DagBuilder is active on the thread (g_dag), launch_gemm records a task instead of
// launching; each task depends on the previous task of the current lane and on add_dep()s.
constexpr int kDagCounterInts = 1 << 16;   // queue head + per-task tile counters + tickets
class DagBuilder {
 public:
  DagBuilder(void* scratch, size_t bytes);   // counters + split-K partials (dag_scratch_bytes)
  void set_lane(int lane);
  int last_of(int lane) const;               // last task recorded on a lane (-1: none)
  int count() const { return (int)tasks.size(); }
  void add_dep(int task) { if (task >= 0) pending.push_back(task); }
  cudaError_t add(bool a_kc, bool b_kc, const GemmParams& p);
  cudaError_t launch(cudaStream_t s);        // one memset of the counters + one kernel
  long long partials_needed() const { return part_used; }
  bool ok = true;
  long long target_units = 128;              // split-K aims for this many units per task

 private:
  struct Node {
    tt::DagTask t;
    int tiles = 0, units = 0;
    std::vector<int> deps;
  };
  std::vector<Node> tasks;
  std::vector<int> lane_last, pending;
  int lane = 0;
  bool dry = false;
  int* ctr = nullptr;
  double* part = nullptr;
  long long part_cap = 0, part_used = 0, ticks = 0;
};
extern thread_local DagBuilder* g_dag;
extern thread_local int g_dag_mode;
extern thread_local unsigned long long* g_dag_trace;
extern thread_local long long g_dag_trace_cap;
extern thread_local int g_dag_last_units, g_dag_last_tasks;
extern thread_local std::vector<int> g_dag_last_unit0;   // tt_debug_set_dag: 0 policy, -1 off, 1 force, 2 8-warp tiles
size_t dag_scratch_bytes(long long partial_elems);
struct DagScope {   // records launch_gemm calls into b for the scope's lifetime
  explicit DagScope(DagBuilder* b) : saved(g_dag) { g_dag = b; }
  ~DagScope() { g_dag = saved; }
  DagBuilder* saved;
};

}  // namespace ttint
