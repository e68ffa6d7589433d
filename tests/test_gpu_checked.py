"""Checked mode (SURVEY §8(b) "Errors"): the device-side validation of cu_seqlens and the
entry points' behaviour with it on (they fail instead of launching on bad offsets) and off
(no validation, no sync)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ub():
    import paper_2208_08124_b200 as ub
    yield ub
    ub.set_checked(False)


def _cu(xs):
    return torch.tensor(xs, dtype=torch.int32, device="cuda")


def test_validate_codes(ub):
    assert ub.validate_cu_seqlens(_cu([0, 3, 10, 10]), 3, 8, 10) == 0
    assert ub.validate_cu_seqlens(_cu([1, 3, 10]), 2, 8, 10) == 1
    assert ub.validate_cu_seqlens(_cu([0, 5, 4]), 2, 8, 10) == 2
    assert ub.validate_cu_seqlens(_cu([0, 3, 13]), 2, 8, 20) == 3
    assert ub.validate_cu_seqlens(_cu([0, 3, 10]), 2, 8, 9) == 4
    # many sequences: the violation is found whichever thread owns it
    cu = np.arange(0, 4 * 700 + 1, 4, dtype=np.int32)
    assert ub.validate_cu_seqlens(_cu(cu.tolist()), 700, 4, int(cu[-1])) == 0
    cu[500] += 9
    assert ub.validate_cu_seqlens(_cu(cu.tolist()), 700, 4, int(cu[-1])) in (2, 3)


def test_checked_entry_points(ub):
    from paper_2208_08124_b200 import UbError
    H, D = 2, 64
    good = _cu([0, 5, 12])
    bad_len = _cu([0, 5, 140])                       # second sequence longer than max_seqlen 128
    qkv = torch.randn((140, 3, H, D), device="cuda").to(torch.bfloat16)
    ub.set_checked(True)
    o, lse = ub.varlen_fmha_fwd(qkv[:12], good, 128)
    with pytest.raises(UbError):
        ub.varlen_fmha_fwd(qkv, bad_len, 128)
    with pytest.raises(UbError):
        ub.unpad(torch.zeros((2, 128, 16), dtype=torch.uint8, device="cuda"), bad_len, 140)
    ub.set_checked(False)
    torch.cuda.synchronize()
