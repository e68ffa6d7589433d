"""Pins for oracle.varlen -- CPU only."""
import numpy as np
import pytest

from oracle import varlen
import synth


def test_batch_offset_worked_examples(golden):
    for ex in golden["spec_worked_examples"]["batch_offset"]:
        assert varlen.batch_offset(ex["lengths"]).tolist() == ex["offsets"], ex["cite"]


def test_batch_offset_differencing_and_errors():
    L = synth.gen_lengths("uniform", 1000, seed=3)
    off = varlen.batch_offset(L)
    assert off[0] == 0 and off[-1] == int(np.sum(L, dtype=np.int64))
    assert np.array_equal(np.diff(off), L)            # differencing reproduces the lengths
    with pytest.raises(ValueError):
        varlen.batch_offset([])
    with pytest.raises(ValueError):
        varlen.batch_offset([3, 0, 2])


def test_unpad_pad_worked_examples(golden):
    ex = golden["spec_worked_examples"]["unpad"][0]
    vals = np.asarray(ex["values"])
    lens = varlen.lengths_from_mask(np.asarray(ex["mask"]))
    assert varlen.unpad(vals, lens).tolist() == ex["packed"]
    assert varlen.batch_offset(lens).tolist() == ex["offsets"]
    ex = golden["spec_worked_examples"]["pad"][0]
    out = varlen.pad(np.asarray(ex["packed"]), ex["offsets"], ex["max_seq_len"], ex["pad_value"])
    assert out.tolist() == ex["padded"]


def test_nonzero_indices_worked_example_and_crosscheck(golden):
    ex = golden["spec_worked_examples"]["nonzero_indices"][0]
    assert varlen.nonzero_indices(np.asarray(ex["mask"])).tolist() == ex["indices"]
    lens = synth.gen_lengths("uniform", 7, seed=1, max_seqlen=512)
    mask = synth.gen_padded_mask(lens, 512)
    vals = np.random.default_rng(0).integers(0, 30000, size=(7, 512))
    idx = varlen.nonzero_indices(mask)
    assert np.array_equal(vals.reshape(-1)[idx], varlen.unpad(vals, lens))


def test_round_trips_bit_exact():
    rng = np.random.default_rng(5)
    lens = [3, 1, 8, 8, 5]
    S = 8
    padded = rng.standard_normal((5, S, 4)).astype(np.float32)
    for b, L in enumerate(lens):
        padded[b, L:] = 0
    off = varlen.batch_offset(lens)
    packed = varlen.unpad(padded, lens)
    assert packed.shape == (sum(lens), 4)
    assert np.array_equal(varlen.pad(packed, off, S, 0), padded)           # pad(unpad(p)) == p
    assert np.array_equal(varlen.unpad(varlen.pad(packed, off, S, 0), lens), packed)
    # fully valid batch: identity row-major copy
    full = rng.standard_normal((3, 4, 2))
    assert np.array_equal(varlen.unpad(full, [4, 4, 4]), full.reshape(12, 2))


def test_pad_capacity_and_pad_row():
    with pytest.raises(ValueError):
        varlen.pad(np.arange(5), [0, 5], 4)
    out = varlen.pad(np.ones((2, 3)), [0, 2], 3, pad_value=np.array([7, 8, 9]))
    assert out[0, 2].tolist() == [7, 8, 9] and out[0, 0].tolist() == [1, 1, 1]


def test_non_prefix_mask_rejected():
    with pytest.raises(ValueError):
        varlen.lengths_from_mask(np.array([[1, 0, 1]]))


def test_redundancy_of_length_fixture():
    """only 23.2% of samples are at max length and unpadding can give "more
    than 2x": the mlperf_like_v0 fixture must reproduce both statements."""
    L = synth.gen_lengths("mlperf_like_v0", 200000, seed=0)
    assert abs(np.mean(L == 512) - 0.232) < 0.005
    assert 512.0 / np.mean(L) > 2.0
    pmf = synth.length_pmf("mlperf_like_v0")
    assert abs(pmf.sum() - 1.0) < 1e-12
