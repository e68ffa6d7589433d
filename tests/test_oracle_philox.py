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


def test_threshold_and_scale():
    assert philox.dropout_threshold(0.0) == 0
    assert philox.dropout_threshold(0.5) == 128
    assert philox.dropout_threshold(np.float32(0.1)) == 25          # floor(25.6)
    assert philox.dropout_scale(0.5) == 2.0
    assert abs(philox.dropout_scale(0.1) - 256.0 / 231.0) < 1e-15  # 1 / (1 - 25/256)


def test_mask_layout_by_hand():
    """R5 written out for one row: key j reads byte (j & 3) of word ((j & 15) >> 2) of the
    Philox call with counter (j >> 4, t, h, offset)."""
    seed, off, t, h, p = 0x1234_5678_9ABC, 3, 9, 2, 0.4
    m = philox.keep_mask_block(seed, off, t, 40, h, p)
    thr = philox.dropout_threshold(p)
    for j in (0, 5, 15, 16, 33):
        w = philox.philox4x32_10(np.uint64(j // 16), np.uint64(t), np.uint64(h), np.uint64(off),
                                 np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32))
        byte = (int(w[(j % 16) // 4]) >> (8 * (j % 4))) & 0xFF
        assert m[0, j] == (byte >= thr)


def test_keep_fraction_binomial():
    p = 0.1
    m = philox.keep_mask_block(seed=0x2208, offset=0, t0=17, L=512, h=3, p=p)
    n = m.size
    keep_p = 1.0 - philox.dropout_threshold(p) / 256.0
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
