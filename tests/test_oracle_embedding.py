"""Pins for oracle.embedding (reading R23) -- CPU only."""
import numpy as np

from oracle import embedding as oemb


def test_hand_worked():
    w_word = np.array([[1.0, 2.0], [10.0, 20.0], [100.0, 200.0]])
    w_pos = np.array([[0.5, 0.5], [0.25, 0.25]])
    w_type = np.array([[0.0, 0.0], [-1.0, -1.0]])
    out = oemb.embedding_fwd([2, 0, 2], [0, 1, 0], [0, 0, 1], w_word, w_pos, w_type)
    assert np.array_equal(out, [[100.5, 200.5], [1.25, 2.25], [99.5, 199.5]])
    dout = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    dw, dp, dt = oemb.embedding_bwd(dout, [2, 0, 2], [0, 1, 0], [0, 0, 1], 3, 2, 2)
    assert np.array_equal(dw, [[3.0, 4.0], [0.0, 0.0], [6.0, 8.0]])      # word 2 gets rows 0 and 2
    assert np.array_equal(dp, [[6.0, 8.0], [3.0, 4.0]])
    assert np.array_equal(dt, [[4.0, 6.0], [5.0, 6.0]])


def test_onehot_form_and_conservation():
    rng = np.random.default_rng(0)
    T, E, V = 300, 16, 50
    ids = rng.integers(0, V, T)
    pos = rng.integers(0, 8, T)
    seg = rng.integers(0, 2, T)
    dout = rng.standard_normal((T, E))
    dw, dp, dt = oemb.embedding_bwd(dout, ids, pos, seg, V, 8, 2)
    onehot = np.zeros((T, V)); onehot[np.arange(T), ids] = 1.0
    assert np.allclose(dw, onehot.T @ dout)
    for d in (dw, dp, dt):
        assert np.allclose(d.sum(axis=0), dout.sum(axis=0))
    unused = np.setdiff1d(np.arange(V), ids)
    assert np.all(dw[unused] == 0.0)


def test_packed_positions():
    assert list(oemb.packed_positions([0, 3, 4, 6])) == [0, 1, 2, 0, 0, 1]
