"""Dev probe: ub_dropout_mask on the config-2 batch (time per call, CUDA events)."""
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
import synth
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
off = np.concatenate([[0], np.cumsum(L)]).astype(np.int32)
T = int(off[-1]); cu = torch.tensor(off).cuda()
m = ub.api.dropout_mask(cu, T, 16, 512, 0.1, 7, 0)
for _ in range(3): ub.api.dropout_mask(cu, T, 16, 512, 0.1, 7, 0, out=m)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20): ub.api.dropout_mask(cu, T, 16, 512, 0.1, 7, 0, out=m)
e1.record(); torch.cuda.synchronize()
print(f"dropout_mask: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call (T={T}, {m.numel() / 1e6:.1f} MB)")
