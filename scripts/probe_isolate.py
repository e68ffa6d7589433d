import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from gpu_util import make_batch
lengths, off, qkv, dout = make_batch([1, 127, 128, 129, 255, 256, 300, 512, 64, 2, 383, 384, 385], 2, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
torch.cuda.synchronize(); print("fwd ok", flush=True)
d = ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512)
torch.cuda.synchronize(); print("bwd ok", flush=True)
