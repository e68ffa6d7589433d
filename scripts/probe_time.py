"""Dev probe: rough fwd/bwd timing at BERT-large config 2 (not a bench number)."""
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
import synth
from gpu_util import make_batch
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
T = int(off[-1]); s2 = float((L.astype(np.int64)**2).sum())
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
tf = t(lambda: ub.varlen_fmha_fwd(qd, cu, 512, out=o, lse=lse))
tb = t(lambda: ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512))
print(f"T={T} fwd {tf:.1f} us ({4*16*64*s2/tf/1e6:.0f} TFLOP/s)  bwd {tb:.1f} us ({8*16*64*s2/tb/1e6:.0f} TFLOP/s strict)  total {T/(tf+tb):.1f} Mtok/s")
