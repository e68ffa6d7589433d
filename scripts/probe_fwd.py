"""Dev probe: forward parity on a few shapes + rough timing (not a bench number)."""
import math, sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
import synth
from gpu_util import make_batch, errors, oracle_seq_slice
from oracle import attention as oatt

def case(lengths, H, p=0.0, ms=512):
    lengths, off, qkv, dout = make_batch(lengths, H, 64)
    cu = torch.tensor(off.astype(np.int32)).cuda()
    o, lse = ub.varlen_fmha_fwd(qkv.cuda(), cu, ms, None, p, 7, 0)
    torch.cuda.synchronize()
    O, LSE = oatt.varlen_fwd(qkv.double().numpy(), off, int(max(lengths)), 1/8, p, 7, 0)
    print("lengths", list(lengths)[:16], "H", H, "p", p, "O err", errors(o.cpu().float().numpy(), O), "LSE err", errors(lse.cpu().numpy(), LSE), flush=True)

case([128], 1)
case([5], 1)
case([300], 1)
case([1, 127, 128, 129, 255, 256, 300, 512, 64, 2], 2)
case([1, 127, 128, 129, 255, 256, 300, 512, 64, 2], 2, p=0.1)
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda()
for _ in range(3): ub.varlen_fmha_fwd(qd, cu, 512)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20): ub.varlen_fmha_fwd(qd, cu, 512)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
T = int(off[-1]); fl = 4 * 16 * 64 * float((L.astype(np.int64)**2).sum())
print(f"fwd T={T} {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s  {T/ms/1e3:.1f} Mtok/s", flush=True)
o, lse = ub.varlen_fmha_fwd(qd, cu, 512); torch.cuda.synchronize()
ref = oracle_seq_slice(qkv, None, off, [int(np.argmax(L)), int(np.argmin(L))], 1/8, bwd=False)
for b,(O,LSE,_) in ref.items():
    s,e = off[b], off[b+1]
    print("seq", b, L[b], errors(o[s:e].cpu().float().numpy(), O), errors(lse[:, s:e].cpu().numpy(), LSE))
