"""The FC weight-gradient tiles of the Mnih bf16 path can write G through bulk shared -> global transfers (a plain
copy at n_push = 1, an fp32 reduce-add at L2 otherwise; the default uses them at n_push > 1; DQN_BULK_ACCUM=0: the
register read-modify-write everywhere, =1: bulk everywhere). Both add the same two fp32 operands with
round-to-nearest, so parameters, gradients and losses are bit-identical."""
import os

import numpy as np
import pytest

import paper_1508_04186_b200 as D
from tests.helpers import gated_theta, nets, replay

pytestmark = pytest.mark.gpu


def run(bulk, b, n_push):
    old = os.environ.get("DQN_BULK_ACCUM")
    os.environ["DQN_BULK_ACCUM"] = str(bulk)
    try:
        dc, on, _ = nets(minibatch=b, replay_capacity=600, precision=D.BF16, target_sync=2, lr=1e-5, rms_eps=1e-2,
                         n_push=n_push, convs=((16, 8, 4), (32, 4, 2)), fcs=(256,), n_actions=18)
        g = D.DQN(dc, init_params=gated_theta(on, 3))
        _, raw = replay(on, 600, 5)
        g.push(*raw)
        out = g.train(6, want_idx=True, want_loss=True)
        th, gr = g.params(D.PARAMS_SERVER), g.params(D.PARAMS_GRAD)
        g.close()
        return out["idx"], out["loss"], th, gr
    finally:
        if old is None:
            os.environ.pop("DQN_BULK_ACCUM", None)
        else:
            os.environ["DQN_BULK_ACCUM"] = old


@pytest.mark.parametrize("b,n_push", [(32, 1), (32, 3), (256, 1), (256, 3)])
def test_bulk_accum_is_bit_identical(b, n_push):
    ref = run(0, b, n_push)
    got = run(1, b, n_push)
    for x, y in zip(got, ref):
        assert np.array_equal(x, y), f"b={b} n_push={n_push}"
