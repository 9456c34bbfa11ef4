"""Oracle pins read from the cited text fixtures under tests/golden/ (DESIGN.md §4).

Each fixture names the passage its values come from: published known-answer vectors for the sampler's
generator, SPEC.md's hand-evaluated examples of Alg. 1's target and Alg. 2's update, and the paper's network
shapes with their exact parameter counts.
"""
import pathlib

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = pathlib.Path(__file__).parent / "golden"


def rows(name):
    out = []
    for line in (GOLDEN / name).read_text().splitlines():
        line = line.strip()
        if line and not line.startswith("#"):
            out.append(line.split())
    assert out, name
    return out


@pytest.mark.parametrize("row", rows("philox4x32_10_kat.txt"), ids=lambda r: r[0] + r[4])
def test_philox_kat_fixture(row):
    v = [int(x, 16) for x in row]
    assert O.philox4x32_10(v[0:4], v[4:6]) == v[6:10]


@pytest.mark.parametrize("row", rows("td_targets_spec.txt"))
def test_td_target_fixture(row):
    r, term, gamma, qmax, y = float(row[0]), int(row[1]), float(row[2]), float(row[3]), float(row[4])
    # a bias-only network: Q^(s', .) = its output biases whatever s' is, with max qmax at action 1
    net = O.Net(frames=1, height=2, width=2, convs=(), fcs=(), n_actions=3)
    th = np.zeros(O.param_count(net))
    th[-3:] = [qmax - 1.0, qmax, qmax - 2.0]
    got, am = O.targets(net, th, np.zeros((1, 1, 2, 2), np.uint8), [r], [term], gamma)
    assert got[0] == y
    if not term:
        assert am[0] == 1


@pytest.mark.parametrize("row", rows("rmsprop_spec.txt"))
def test_rmsprop_fixture(row):
    th0, r0, g, alpha, eps, th1, r1 = (float(x) for x in row)
    th, r = O.rmsprop(np.array([th0]), np.array([r0]), np.array([g]), alpha, 0.9, eps)
    assert abs(r[0] - r1) < 1e-15
    assert abs(th[0] - th1) < 1e-9


def parse_net(row):
    convs = tuple(tuple(int(x) for x in c.split(":")) for c in row[4].split(","))
    fcs = tuple(int(x) for x in row[5].split(","))
    return O.Net(frames=int(row[1]), height=int(row[2]), width=int(row[3]), convs=convs, fcs=fcs,
                 n_actions=int(row[6]))


@pytest.mark.parametrize("row", rows("network_shapes.txt"), ids=lambda r: r[0])
def test_network_shape_fixture(row):
    net = parse_net(row)
    c, h, w = (int(x) for x in row[7].split(":"))
    # valid convolutions: out = (in - k) / s + 1 per layer
    hh, ww = net.height, net.width
    for _, k, s in net.convs:
        hh, ww = (hh - k) // s + 1, (ww - k) // s + 1
    assert (net.convs[-1][0], hh, ww) == (c, h, w)
    tt = O.tensor_table(net)
    assert tt[2 * len(net.convs)][1] == net.fcs[0] * c * h * w       # first FC layer reads the flattened map
    assert O.param_count(net) == int(row[8])
    assert sum(n for _, n in tt) == int(row[8])
    # the per-layer (fan_in + 1) * units sum, written out
    total, cin = 0, net.frames
    for n, k, _ in net.convs:
        total += (cin * k * k + 1) * n
        cin = n
    d = c * h * w
    for u in net.fcs + (net.n_actions,):
        total += (d + 1) * u
        d = u
    assert total == int(row[8])
