"""Full config-5 parity certificate ("the full oracle parity on config 5 is
run once as a recorded certificate").

GPU: the bench's launch configuration -- tt_sweep_als (W5, K = 32, both directions) and the
full unrounded tt_operator_apply.  Oracle: tt_oracle_sweep_interfaces for every interface,
tt_oracle_local_matvec_batched for every core and every Krylov column, tt_oracle_apply_core
for every core.  Cores are fixed in W5, so the forward and backward sweep's matvecs both
equal the oracle's matvec with the converged interfaces.  The oracle runs as it stands; the
(core, column) tasks are spread over a process pool to finish in minutes.

Writes profiles/<name>.json: max relative Frobenius error per output family and per array.
usage: python tools/config5_certificate.py [out.json]
"""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import ttgen  # noqa: E402

INP = None
PL = PR = None


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def task(args):
    k, c0, c1 = args
    X = np.ascontiguousarray(INP.X[k][:, :, c0:c1, :])
    return k, c0, c1, oracle.local_matvec_batched(PL[k], INP.A[k], PR[k + 1], X)


def main():
    global INP, PL, PR
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_config5_certificate.json"
    import torch
    import paper_2509_11890_b200 as tt
    INP = ttgen.make_inputs(5)
    d = len(INP.x)
    dev = torch.device("cuda")
    xs = [torch.from_numpy(c).to(dev) for c in INP.x]
    As = [torch.from_numpy(c).to(dev) for c in INP.A]
    Xs = [torch.from_numpy(c).to(dev) for c in INP.X]
    Yb = [torch.empty_like(X) for X in Xs]
    t0 = time.time()
    Yf, Yb, pl, pr = tt.tt_sweep_als(xs, As, Xs, None, Yb)
    torch.cuda.synchronize()
    gpu = {"Yf": [y.cpu().numpy() for y in Yf], "Yb": [y.cpu().numpy() for y in Yb],
           "phiL": [p.cpu().numpy() for p in pl], "phiR": [p.cpu().numpy() for p in pr]}
    t1 = time.time()
    PL, PR = oracle.sweep_interfaces(INP.x, INP.A, 3)
    t2 = time.time()
    K = INP.X[0].shape[2]
    chunk = 4
    tasks = [(k, c, min(K, c + chunk)) for k in range(d) for c in range(0, K, chunk)]
    Yo = [np.empty_like(X) for X in INP.X]
    nproc = min(len(os.sched_getaffinity(0)), 16)
    with mp.get_context("fork").Pool(nproc) as pool:
        for k, c0, c1, Y in pool.imap_unordered(task, tasks):
            Yo[k][:, :, c0:c1, :] = Y
    t3 = time.time()
    res = {"phiL": [], "phiR": [], "Yf": [], "Yb": [], "Yf_col_max": [], "apply": []}
    # W5 computes phiL[1..d-1] and phiR[1..d-1] (phiL[0] = phiR[d] = 1 set by the call)
    for k in range(d):
        res["phiL"].append(rel(gpu["phiL"][k], PL[k]))
        res["phiR"].append(rel(gpu["phiR"][k + 1], PR[k + 1]))
        res["Yf"].append(rel(gpu["Yf"][k], Yo[k]))
        res["Yb"].append(rel(gpu["Yb"][k], Yo[k]))
        res["Yf_col_max"].append(max(rel(gpu["Yf"][k][:, :, j, :], Yo[k][:, :, j, :])
                                     for j in range(K)))
    del gpu, Yo
    # full unrounded apply, one core at a time (12.3 GB in total)
    zs = [torch.empty((c.shape[0] * A.shape[0], A.shape[1], c.shape[2] * A.shape[3]),
                      dtype=torch.float64, device=dev) for c, A in zip(xs, As)]
    tt.tt_operator_apply(xs, As, zs)
    torch.cuda.synchronize()
    for k in range(d):
        zk = zs[k].cpu().numpy()
        res["apply"].append(rel(zk, oracle.apply_core(INP.x[k], INP.A[k])))
        zs[k] = None
    t4 = time.time()
    worst = {key: max(v) for key, v in res.items()}
    cert = {"config": 5, "workload": "W5 tt_sweep_als (K = 32, both directions) + tt_operator_apply",
            "metric": "relative Frobenius error per output array (DESIGN.md A8), bar 1e-11",
            "worst": worst, "pass": all(v <= 1e-11 for v in worst.values()),
            "per_array": res, "oracle_processes": nproc,
            "seconds": {"gpu": t1 - t0, "oracle_interfaces": t2 - t1,
                        "oracle_matvecs": t3 - t2, "apply_check": t4 - t3}}
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump(cert, f, indent=1)
    print(json.dumps({"worst": worst, "pass": cert["pass"], "seconds": cert["seconds"]}))


if __name__ == "__main__":
    main()
