"""bench.py's roofline accounting (CPU): the per-step algorithmic FLOPs of the regions add up to the
per-replica-step totals SURVEY.md §8(a) derives from the layer shapes (0.655 / 5.24 / 35.0 GFLOP), the
parameter counts match the oracle's, and the fused server round's byte count follows its formula."""
import bench
from oracle import oracle as O

REGIONS = ("conv_fwd", "fc1_fwd", "head_sample", "fc1_bwd", "conv_bwd")


def step_flops(net, b):
    return sum(bench.region_work(k, b, net)[0] for k in REGIONS)


def test_step_flops_match_the_survey_totals():
    for net, b, gflop in ((bench.MNIH, 32, 0.655), (bench.MNIH, 256, 5.24), (bench.SCALED, 512, 35.0)):
        assert abs(step_flops(net, b) / 1e9 - gflop) <= 0.002 * gflop


def test_flops_scale_linearly_in_b_and_conv1_dominates_the_mnih_forward():
    assert step_flops(bench.MNIH, 256) == 8 * step_flops(bench.MNIH, 32)
    c1 = bench.region_work("conv1_fwd", 32)[0]
    assert 0.5 < c1 / bench.region_work("conv_fwd", 32)[0] < 0.8  # conv1 is 55 % of forward MACs


def test_parameter_counts_agree_with_the_oracle():
    for net in (bench.MNIH, bench.SCALED):
        on = O.Net(**net)
        assert bench.region_work("rmsprop_update", 32, net)[1] == 24 * O.param_count(on)
        conv = sum(cnt for i, (off, cnt) in enumerate(O.tensor_table(on)) if i < 2 * len(net["convs"]))
        assert bench.conv_param_count(net) == conv


def test_server_round_bytes():
    P = O.param_count(O.Net(**bench.MNIH))
    for world in (2, 4, 8):
        shard = -(-P // (64 * world)) * 64
        assert bench.region_work("server_round_fused", 32, bench.MNIH, world)[1] == shard * (6 * world + 16)
