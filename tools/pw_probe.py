"""Producer placement A/B at the config-5 interior matvec (K = 32): the stage GEMMs with thread 0
(debug bit 30) or the round-robin producer (default); the fused kernel with the round-robin
producer (mode 2), a 13th producer warp (194) or thread 0 (98)."""
import sys, os, torch
sys.path.insert(0, "/root/repo")
import paper_2509_11890_b200 as tt
a=b=256; al=be=36; K=32; n=4
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)
phiL, A, phiR, X = r(a, al, a), r(al, n, n, be), r(b, be, b), r(a, n, K, b)
tt.tt_set_graph_cache(False)
ref=None
for fused, flags in [(-1,1<<30),(-1,0),(2,0),(194,0),(98,0)]:   # fused: round-robin (2), producer warp (194), thread 0 (98)
    tt.tt_debug_set_fused(fused); tt.tt_debug_set_flags(flags)
    Y = torch.empty_like(X)
    for _ in range(2): tt.tt_local_matvec_batched(phiL, A, phiR, X, Y)
    torch.cuda.synchronize()
    tt.tt_trace_enable(64)
    tt.tt_local_matvec_batched(phiL, A, phiR, X, Y)
    torch.cuda.synchronize()
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()
    if ref is None: ref = Y.clone()
    st = " ".join(f"{q['stage']}[{q['tile']}]={q['ms']:.3f}ms/{2.0*q['M']*q['N']*q['K']/q['ms']/1e9:.2f}TF" for q in recs if q["stage"].startswith("mv_"))
    print(fused, hex(flags), st, "diff", float((Y-ref).norm()/ref.norm()), flush=True)
