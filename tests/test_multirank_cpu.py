"""N>1 host logic of bench.py on CPU with the gloo backend (world_size 2): replicas only, the
only collective is the max-over-ranks timing reduction; the reference arm runs on rank 0."""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms = 10.0 + 5.0 * rank                      # per-rank device time
        mx = bench.max_over_ranks(ms, torch.device("cpu"))
        rate = bench.whole_job_rate(1e9, world, 4, mx)
        out[rank] = (mx, rate)
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][0] == out[1][0] == 15.0
    # whole-job rate: 2 ranks x 4 steps x 1 GFLOP in the slowest rank's 15 ms
    assert abs(out[0][1] - 2 * 4 * 1e9 / 15e-3 / 1e9) < 1e-9


def test_max_over_ranks_single_process_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(12.5, torch.device("cpu")) == 12.5


def test_reference_arm_other_ranks_exit_without_work():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_work_model_matches_survey():
    """Algorithmic FLOPs of the W5 workload (matvecs 3458.6, interfaces
    162.1 GFLOP) and the apply bytes (12.33 GB)."""
    sys.path.insert(0, ROOT)
    import bench
    import ttgen
    w = bench.w5_work(ttgen.CONFIGS[5])
    assert abs(w["matvec_flops"] / 1e9 - 3458.6) < 0.1
    assert abs(w["interface_flops"] / 1e9 - 162.1) < 0.1
    assert abs(w["apply_bytes"] / 1e9 - 12.33) < 0.01
