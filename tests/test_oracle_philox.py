"""Pins for oracle.philox (reading R5) -- CPU only."""
import numpy as np

from oracle import philox


def test_known_answer_vectors(golden):
    kat = golden["philox4x32_10_kat"]
    for v in kat["vectors"]:
        c = [np.uint64(int(x, 16)) for x in v["ctr"]]
        k = [np.uint64(int(x, 16)) for x in v["key"]]
        out = philox.philox4x32_10(*c, *k)
        assert ["%08x" % int(x) for x in out] == v["out"], kat["citation"]


def test_threshold():
    assert philox.dropout_threshold(0.0) == 0
    assert philox.dropout_threshold(0.5) == 32768
    assert philox.dropout_threshold(np.float32(0.1)) == 6553


def test_keep_fraction_binomial():
    p = 0.1
    m = philox.keep_mask_block(seed=0x2208, offset=0, t0=17, L=512, h=3, p=p)
    n = m.size
    keep_p = 1.0 - philox.dropout_threshold(p) / 65536.0
    sd = np.sqrt(n * keep_p * (1 - keep_p))
    assert abs(m.sum() - n * keep_p) < 5 * sd


def test_p0_keeps_everything_and_coordinates_matter():
    assert philox.keep_mask_block(1, 0, 0, 64, 0, 0.0).all()
    a = philox.keep_mask_block(1, 0, 0, 64, 0, 0.5)
    b = philox.keep_mask_block(1, 0, 0, 64, 1, 0.5)      # other head
    c = philox.keep_mask_block(2, 0, 0, 64, 0, 0.5)      # other seed
    d = philox.keep_mask_block(1, 1, 0, 64, 0, 0.5)      # other offset
    assert (a != b).any() and (a != c).any() and (a != d).any()
    # coordinate purity: rows of a longer block starting at the same t0 agree
    e = philox.keep_mask_block(1, 0, 0, 80, 0, 0.5)
    assert np.array_equal(e[:64, :64], a)
