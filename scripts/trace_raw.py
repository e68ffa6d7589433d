"""Raw per-warp event timeline of CTA 0 from a trace build (dev tool):
UB_LIB=paper_2208_08124_b200/libub_trace.so python scripts/trace_raw.py fwd WARPS N"""
import ctypes as C, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import _lib
import synth
from gpu_util import make_batch
which = sys.argv[1]
warps = [int(w) for w in sys.argv[2].split(",")]
n = int(sys.argv[3])
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
for _ in range(3):
    if which == "fwd":
        o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
    else:
        ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512)
torch.cuda.synchronize()
nw = 10 if which == "fwd" else 16
buf = np.zeros(nw * 1024, dtype=np.uint64)
f = getattr(_lib.lib(), f"ub_debug_{which}_trace"); f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t]
assert f(buf.ctypes.data_as(C.c_void_p), buf.nbytes) == 0
ev = (buf >> np.uint64(48)).astype(np.int64); ck = (buf & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
t0 = ck[ck > 0].min()
for w in warps:
    row = [(int(ev[w * 1024 + i]), int(ck[w * 1024 + i] - t0)) for i in range(1024) if buf[w * 1024 + i]]
    print(f"--- warp {w}")
    print(" ".join(f"{e}@{c}" for e, c in row[:n]))
