"""CPU checks of the "gated" parity regime (A38) that the bf16 GPU parity tests rely on.

tests/helpers.gated_theta builds theta0 so that every hidden pre-activation satisfies |z| >= bias - margin
= 0.06 for ANY u8 input: half of the ReLU units are always off, the other half always on, and no rounding
(fp64, fp32 or bf16 operands) can flip a branch. These checks pin that claim with the oracle on extreme and
random inputs, and check that the regime does exercise the masks (off units get exactly zero gradient rows)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import gated_theta

MNIH = O.Net()
SCALED = O.NATURE_SCALED


@pytest.mark.parametrize("net", [MNIH, SCALED], ids=["mnih", "scaled"])
def test_every_hidden_preactivation_is_bounded_away_from_the_kink(net):
    th = gated_theta(net, 11).astype(np.float64)
    rng = np.random.default_rng(0)
    states = np.concatenate([
        np.zeros((1, 4, 84, 84), np.uint8), np.full((1, 4, 84, 84), 255, np.uint8),
        rng.integers(0, 256, (3, 4, 84, 84), dtype=np.uint8),
        (rng.random((2, 4, 84, 84)) < 0.5).astype(np.uint8) * 255])
    assert O.min_abs_preact(net, th, states) >= 0.0599


def test_off_units_have_zero_gradient_rows_and_on_units_do_not():
    """the masks matter: a random half of every hidden layer's units is always off and gets exactly zero
    gradient rows, the other half never does"""
    net = MNIH
    th = gated_theta(net, 12).astype(np.float64)
    rng = np.random.default_rng(1)
    s = rng.integers(0, 256, (4, 4, 84, 84), dtype=np.uint8)
    a = rng.integers(0, 6, 4).astype(np.int32)
    y = rng.normal(0, 1, 4)
    _, g = O.loss_grad(net, th, s, a, y)
    tt = O.tensor_table(net)
    (fo, fc), (bo, bc) = tt[4], tt[5]  # hidden FC layer: W [256][2592], b [256]
    on = th[bo:bo + bc] > 0
    assert on.sum() == 128 and not np.array_equal(on, np.arange(256) % 2 == 0)  # a random half, not by parity
    gw = g[fo:fo + fc].reshape(256, 2592)
    gb = g[bo:bo + bc]
    assert np.all(gw[~on] == 0.0) and np.all(gb[~on] == 0.0)   # units with bias -0.1: always off
    assert np.all(np.abs(gb[on]) > 0.0)                         # units with bias +0.1: always on
    (co, cc), (cbo, cbc) = tt[0], tt[1]  # conv1: W [16][4][8][8], b [16]
    on1 = th[cbo:cbo + cbc] > 0
    assert np.all(g[co:co + cc].reshape(16, -1)[~on1] == 0.0) and np.all(g[cbo:cbo + cbc][~on1] == 0.0)
    assert np.all(np.abs(g[cbo:cbo + cbc][on1]) > 0.0)
