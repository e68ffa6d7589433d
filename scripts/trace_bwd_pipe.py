"""Correlate the bwd Q/dO producer with the MMA issuer in a trace build (CTA 0):
per pair p, when the producer passed the stage-empty wait (23) and arrived (24), and when
the MMA saw qdo_full (18), issued S (10/11) and finished issuing grads (19)."""
import ctypes as C, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import _lib
import synth
from gpu_util import make_batch
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
for _ in range(3): ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512)
torch.cuda.synchronize()
buf = np.zeros(16 * 1024, dtype=np.uint64)
f = _lib.lib().ub_debug_bwd_trace; f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t]
assert f(buf.ctypes.data_as(C.c_void_p), buf.nbytes) == 0
ev = (buf >> np.uint64(48)).astype(np.int64); ck = (buf & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
t0 = ck[ck > 0].min()
def series(w, e):
    return [int(ck[w * 1024 + i] - t0) for i in range(1024) if buf[w * 1024 + i] and ev[w * 1024 + i] == e]
p23, p24, m18, m10, m11, m19 = series(12, 23), series(12, 24), series(13, 18), series(13, 10), series(13, 11), series(13, 19)
c2, c3, c4, c5, c7 = series(0, 2), series(0, 3), series(0, 4), series(0, 5), series(0, 7)
print("pair  prodStage prodArrive  mmaQ  mmaSiss mmaSdone  cmpSgot cmpLd cmpMath cmpGradOk cmpStored  mmaGradsIssued(p-1)")
for p in range(min(30, len(m18))):
    g = lambda a: a[p] if p < len(a) else -1
    print(f"{p:4d} {g(p23):9d} {g(p24):9d} {g(m18):7d} {g(m10):7d} {g(m11):8d} {g(c2):8d} {g(c3):6d} {g(c4):7d} {g(c5):8d} {g(c7):8d} {g(m19):8d}")
