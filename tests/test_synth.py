"""The seeded generators: fingerprints, host/device twins, exactness in bf16 — no GPU."""
import numpy as np
import pytest
import torch

import synth
from synth import workloads as wl


def test_routing_fingerprints_seed0():
    """SURVEY §8(d) seed-0 fingerprints of the exact routing recipe."""
    ids = synth.route(synth.CONFIGS["mix"], 0)
    assert ids[0].tolist() == [7, 4]
    assert np.bincount(ids.ravel(), minlength=8).tolist() == [1029, 1009, 1020, 1047, 1026, 1000, 1032, 1029]
    ids = synth.route(synth.CONFIGS["ds"], 0)
    assert ids[0].tolist() == [36, 16, 61, 44, 40, 10]
    c = np.bincount(ids.ravel(), minlength=64)
    assert (c == 0).sum() == 16
    assert sorted(c)[::-1][:8] == [7552, 5780, 4247, 3332, 2714, 2211, 1909, 1634]
    assert c[c > 0].min() == 183
    assert np.bincount(synth.route(synth.CONFIGS["ep"], 0).ravel()).tolist() == \
        [8086, 8250, 8119, 8150, 8279, 8188, 8197, 8267]
    assert np.bincount(synth.route(synth.CONFIGS["dec1"], 0).ravel(), minlength=8).tolist() == [0, 0, 0, 0, 1, 0, 0, 1]
    assert np.bincount(synth.route(synth.CONFIGS["dec16"], 0).ravel(), minlength=8).tolist() == [4, 7, 2, 5, 7, 3, 0, 4]


def test_paper_scenarios():
    c = np.bincount(synth.route(synth.CONFIGS["paper_balanced"]).ravel(), minlength=64)
    assert (c == 512).all()
    c = np.bincount(synth.route(synth.CONFIGS["mix_balanced"]).ravel(), minlength=8)
    assert (c == 1024).all()
    c = np.bincount(synth.route(synth.CONFIGS["paper_best"]).ravel(), minlength=64)
    assert (c[:8] == 4096).all() and (c[8:] == 0).all()
    ids = synth.route(synth.CONFIGS["paper_worst"])
    c = np.bincount(ids.ravel(), minlength=64)
    assert (c[8:] == 1).all() and (c[:7] == 4096).all() and c[7] == 4096 - 56
    for t in range(ids.shape[0]):
        assert len(set(ids[t].tolist())) == 8


@pytest.mark.parametrize("mode", ["normal", "int"])
def test_numpy_torch_twins_identical(mode):
    x = synth.make_x(7, 33, 64, mode)
    xt = synth.make_x_torch(7, 33, 64, mode)
    assert xt.dtype == torch.bfloat16
    assert np.array_equal(x, xt.double().numpy())
    w = synth.make_w(7, 3, 64, 40, mode)
    wt = synth.make_w_torch(7, 3, 64, 40, mode, chunk=1000)
    assert np.array_equal(w, wt.double().numpy())
    assert np.array_equal(synth.make_w_torch(7, 3, 64, 40, mode, experts=range(1, 3)).double().numpy(), w[1:3])
    # column/row fetchers agree with the full arrays
    assert np.array_equal(wl.w_columns(7, 3, 64, 40, 2, np.array([0, 39]), mode), w[2][:, [0, 39]])
    assert np.array_equal(wl.x_rows(7, 33, 64, [5, 32], mode), x[[5, 32]])


def test_values_exact_in_bf16():
    x = synth.make_x(1, 64, 128)
    c = x * 2.0 ** 6
    assert np.array_equal(c, np.round(c)) and np.abs(c).max() <= 254
    # a float64 -> bf16 -> float64 round trip is the identity
    assert np.array_equal(torch.from_numpy(x).to(torch.bfloat16).double().numpy(), x)
    xi = synth.make_x(1, 64, 128, "int")
    assert set(np.unique(xi).tolist()) <= set(range(-4, 5))


def test_gumbel_top_k_properties():
    ids = synth.route_gumbel(11, 500, 10, 3, s=1.0, n_empty=4)
    assert ids.dtype == np.int32
    c = np.bincount(ids.ravel(), minlength=10)
    assert (c == 0).sum() >= 4
    for t in range(500):
        assert len(set(ids[t].tolist())) == 3
