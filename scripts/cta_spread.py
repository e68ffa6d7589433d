"""Per-CTA start / end times (globaltimer) of the fwd and bwd main kernels in a trace build
(UB_LIB=.../libub_trace.so python scripts/cta_spread.py [p]): the tail the persistent
schedule leaves (last CTA end - median CTA end)."""
import ctypes as C, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import _lib, api
import synth
from gpu_util import make_batch
pd = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
for seed in (0, 1, 2):
    L = synth.gen_lengths("mlperf_like_v0", 56, seed)
    lengths, off, qkv, dout = make_batch(L, 16, 64)
    cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
    T = int(off[-1])
    mk = api.dropout_mask(cu, T, 16, 512, pd) if pd > 0 else None
    for which in ("fwd", "bwd"):
        for _ in range(3):
            o, lse = ub.varlen_fmha_fwd(qd, cu, 512, p_dropout=pd, dropout_mask=mk, num_ctas=144)
            if which == "bwd":
                ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512, p_dropout=pd, dropout_mask=mk, num_ctas=144)
        torch.cuda.synchronize()
        buf = np.zeros(2 * 1024, dtype=np.uint64)
        f = getattr(_lib.lib(), f"ub_debug_{which}_cta_times"); f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t]
        assert f(buf.ctypes.data_as(C.c_void_p), buf.nbytes) == 0
        st, en = buf[0:288:2].astype(np.int64), buf[1:288:2].astype(np.int64)
        t0 = st.min()
        st, en = (st - t0) / 1e3, (en - t0) / 1e3
        print(f"seed {seed} {which}: span {en.max():.1f} us, CTA end min/median/max {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}, "
              f"start max {st.max():.1f}, tail (max - median) {en.max() - np.median(en):.1f} us, mean busy {np.mean(en - st):.1f}")
