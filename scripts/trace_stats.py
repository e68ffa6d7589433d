"""Per-phase cycle statistics of CTA 0 of the fwd/bwd kernel from a trace build
(UB_LIB=paper_2208_08124_b200/libub_trace.so python scripts/trace_stats.py [fwd|bwd] [dist]).
For every warp: mean/total cycles between consecutive events, keyed by (event -> next)."""
import ctypes as C, collections, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import _lib
import synth
from gpu_util import make_batch
which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
dist = sys.argv[2] if len(sys.argv) > 2 else "mlperf_like_v0"
pd = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0     # dropout p (with the materialised mask)
L = synth.gen_lengths(dist, 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
from paper_2208_08124_b200 import api as _api
mk = _api.dropout_mask(cu, int(off[-1]), 16, 512, pd) if pd > 0 else None
o, lse = ub.varlen_fmha_fwd(qd, cu, 512, p_dropout=pd, dropout_mask=mk)
for _ in range(3):
    if which == "fwd":
        o, lse = ub.varlen_fmha_fwd(qd, cu, 512, p_dropout=pd, dropout_mask=mk)
    else:
        ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512, p_dropout=pd, dropout_mask=mk)
torch.cuda.synchronize()
nw = 10 if which == "fwd" else 16
buf = np.zeros(nw * 1024, dtype=np.uint64)
f = getattr(_lib.lib(), f"ub_debug_{which}_trace"); f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t]
assert f(buf.ctypes.data_as(C.c_void_p), buf.nbytes) == 0
ev = (buf >> np.uint64(48)).astype(np.int64); ck = (buf & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
t0 = ck[ck > 0].min()
print(f"{which} {dist}: CTA0 span {ck.max() - t0} cycles")
for w in range(nw):
    row = [(int(ev[w * 1024 + i]), int(ck[w * 1024 + i] - t0)) for i in range(1024) if buf[w * 1024 + i]]
    if not row:
        continue
    st = collections.defaultdict(list)
    for (e0, c0), (e1, c1) in zip(row, row[1:]):
        st[(e0, e1)].append(c1 - c0)
    span = row[-1][1] - row[0][1]
    parts = sorted(st.items(), key=lambda kv: -sum(kv[1]))[:8]
    print(f"warp {w:2d} n={len(row)} first={row[0][1]} last={row[-1][1]} span={span}")
    for (a, b), v in parts:
        print(f"    {a:2d}->{b:2d} n={len(v):4d} mean={np.mean(v):8.0f} total={sum(v):8d} ({100*sum(v)/max(span,1):4.1f}%)")
