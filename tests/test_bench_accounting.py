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
        assert bench.region_work("rmsprop_update", 32, net)[1] == 22 * O.param_count(on)  # 22 B/param
        assert bench.region_work("rmsprop_update", 32, net, dtype="f32")[1] == 20 * O.param_count(on)
        assert bench.param_count_of(net) == O.param_count(on)
        conv = sum(cnt for i, (off, cnt) in enumerate(O.tensor_table(on)) if i < 2 * len(net["convs"]))
        assert bench.conv_param_count(net) == conv


def test_server_round_bytes():
    P = O.param_count(O.Net(**bench.MNIH))
    for world in (2, 4, 8):
        shard = -(-P // (64 * world)) * 64
        assert bench.region_work("server_round_fused", 32, bench.MNIH, world)[1] == shard * (6 * world + 16)


def test_gather_bytes_are_the_compulsory_u8_slots_and_activations_follow_the_dtype():
    """a2: conv1's forward reads the s and s' u8 slots, 56,448 B per transition; its
    output (and every later activation) is 2 B per element on the bf16 path, 4 B on the fp32 path."""
    b = 32
    f16, by16 = bench.region_work("conv1_fwd", b)
    _, by32 = bench.region_work("conv1_fwd", b, dtype="f32")
    out = 16 * 20 * 20
    assert by16 == b * 56448 + 2 * b * out * 2 and by32 == b * 56448 + 2 * b * out * 4


def test_roofline_reports_both_fractions_and_the_binding_one():
    regions = [dict(name=n, avg_us=us, steps=100, kernels=1) for n, us in
               (("conv_fwd", 14.0), ("fc1_fwd", 11.8), ("head_sample", 9.7), ("fc1_bwd_head_finish", 14.2),
                ("conv_bwd", 19.8), ("reduce_update", 7.6))]
    r = bench.roofline(regions, 32, bench.MNIH, 1, "bf16", 100)
    assert r["kernel"] == "conv_bwd" and r["bound"] in ("hbm", "tensor")
    assert abs(r["frac"] - r[r["bound"] if r["bound"] == "hbm" else "tensor"]["frac"]) < 1e-12
    assert abs(r["step"]["us"] - 77.1) < 1e-9
    assert 0 < r["step"]["tensor_frac"] < 0.02 and 0 < r["step"]["hbm_frac"] < 0.2
