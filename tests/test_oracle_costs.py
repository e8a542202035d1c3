"""Pins of the oracle's cost arithmetic (oracle/ir.py op_cost, stage_weights, sm_partition with
the a3 tile cap) against values fixed outside this repository:

* torchvision's published per-model cost and size (``Weights.meta["_ops"]``, GMACs at the
  weights' crop size, 3 decimals; ``meta["num_params"]``) -- library metadata, not computed here;
* SURVEY §8(a) a3's worked example (c2 all-concurrent -> R18/MBv2 = 76/72 SMs) and Appendix A's
  per-model B_op (materialised bytes at bf16, MB);
* hand-worked cap redistribution cases.

A dropped /groups (depthwise MACs), a residual counted twice, or a transposed F/B in the
stage weight each fails one of these.
"""
import functools

import pytest

from oracle import ir
from workloads import configs, zoo

tvm = pytest.importorskip("torchvision.models")

# zoo model -> (torchvision weights enum name, input size of its published cost)
PUBLISHED = {
    "resnet18": ("ResNet18_Weights", 224),
    "resnet34": ("ResNet34_Weights", 224),
    "resnet50": ("ResNet50_Weights", 224),
    "resnet101": ("ResNet101_Weights", 224),
    "mobilenet_v2": ("MobileNet_V2_Weights", 224),
    "vgg16": ("VGG16_Weights", 224),
    "squeezenet1_0": ("SqueezeNet1_0_Weights", 224),
    "alexnet": ("AlexNet_Weights", 224),
    "inception_v3": ("Inception_V3_Weights", 299),
}

# torchvision Inception-v3's num_params includes the auxiliary head (AuxLogits: conv0 1x1
# 768->128 + BN, conv1 5x5 128->768 + BN, fc 768->1000 + bias); the zoo graph has no aux head
# (transform_input off, aux_logits=False, R15)
INC3_AUX_PARAMS = (768 * 128 + 2 * 128) + (128 * 768 * 25 + 2 * 768) + (768 * 1000 + 1000)


@functools.lru_cache(maxsize=None)
def _graph(name, size=224):
    if name == "inception_v3":
        return zoo.inception_v3(size=size)
    return zoo.MODELS[name]()


def _total_cost(g, eb=2):
    F = B = 0
    for j in range(g.n_ops):
        f, b = ir.op_cost(g.nodes, j, g.batch, (g.in_c, g.in_h, g.in_w), eb)
        F += f
        B += b
    return F, B


@pytest.mark.parametrize("name", list(PUBLISHED))
def test_op_cost_flops_match_torchvision_published_gmacs(name):
    wname, size = PUBLISHED[name]
    meta = getattr(tvm, wname).IMAGENET1K_V1.meta
    F, _ = _total_cost(_graph(name, size))
    # F = 2 * MACs of every conv / FC; torchvision quotes GMACs rounded to 3 decimals
    assert abs(F / 2e9 - meta["_ops"]) <= 0.0006, (name, F / 2e9, meta["_ops"])


@pytest.mark.parametrize("name", list(PUBLISHED))
def test_zoo_parameter_counts_match_torchvision(name):
    """The weights op_cost counts (conv/FC weight tensors) plus the folded BN affine pairs and
    biases equal torchvision's parameter count, so the zoo graphs carry exactly torchvision's
    layers (the F pin above then pins op_cost's MAC arithmetic on the right layers)."""
    wname, size = PUBLISHED[name]
    meta = getattr(tvm, wname).IMAGENET1K_V1.meta
    g = _graph(name, size)
    n = 0
    for nd, p in zip(g.nodes, g.params):
        if nd["kind"] in (zoo.CONV, zoo.FC):
            n += p["weight"].size
            bn_folded = not ((p["scale"] == 1).all())      # identity scale: bias only (or none)
            if bn_folded:
                n += 2 * nd["out_c"]                       # BN gamma, beta
            elif nd["kind"] == zoo.FC or (p["shift"] != 0).any():
                n += nd["out_c"]                           # bias
    exp = meta["num_params"] - (INC3_AUX_PARAMS if name == "inception_v3" else 0)
    assert n == exp, (name, n, exp)


# SURVEY Appendix A, B_op MB at b=1 (bf16): every op's inputs + weights + residual + output
APPENDIX_A_BOP_MB = {"resnet18": 36.3, "mobilenet_v2": 34.4, "resnet50": 107.8, "vgg16": 337.3,
                     "inception_v3": 79.1, "squeezenet1_0": 23.1, "alexnet": 124.8,
                     "resnet34": 62.7, "resnet101": 173.0}


@pytest.mark.parametrize("name", list(APPENDIX_A_BOP_MB))
def test_op_cost_bytes_match_survey_appendix_a(name):
    _, B = _total_cost(_graph(name))
    # VGG-16: Appendix A lists 337.4 with the identity adaptive avg-pool (22 ops); the zoo
    # elides it (R6: 21 ops), which removes 2 x 25088 x 2 B = 0.1 MB
    assert abs(B / 1e6 - APPENDIX_A_BOP_MB[name]) <= 0.051, (name, B / 1e6)


def _eb(g):
    return 2 if g.precision == zoo.PREC_BF16 else 4


def test_stage_weights_and_partition_survey_worked_example_c2():
    """SURVEY §8(a) a3 worked example: c2 all-concurrent, BW = 8000, TC = 2 250 000, per-op
    materialised bytes -> R18 / MBv2 = 76 / 72 SMs (MBv2's bytes match R18's)."""
    gs = configs.tenants("c2")
    L = [g.n_ops for g in gs]
    st, ranges = ir.T(L, configs.all_concurrent_pointers(L))
    assert st[0] == ir.E_OK and len(ranges) == 1
    w = ir.stage_weights(gs, ranges, _eb)[0]
    assert ir.sm_partition(w, 148) == [76, 72]


def test_partition_c3_reading():
    """SURVEY's c3 figure is 30/108/10; the oracle gives 31/107/10 (R16: SURVEY's
    derivation, not the paper, and the one-SM shift is within its rounding of per-op bytes).
    Pinned here so a change of the arithmetic cannot pass silently."""
    gs = configs.tenants("c3")
    L = [g.n_ops for g in gs]
    _, ranges = ir.T(L, configs.all_concurrent_pointers(L))
    assert ir.sm_partition(ir.stage_weights(gs, ranges, _eb)[0], 148) == [31, 107, 10]


def test_stage_weight_is_roofline_time_max_not_sum():
    """One compute-bound op (F*BW > B*TC) weighs F*BW: its B*TC must not be added."""
    g = zoo.vgg16()
    j = 1      # conv3x3 64->64 @224: 3.7 GFLOP, 12.9 MB -> compute-bound at spec peaks
    F, B = ir.op_cost(g.nodes, j, 1, (3, 224, 224), 2)
    assert F * ir.BW_GBS > B * ir.TC_GFLOPS
    w = ir.stage_weights([g], [[(j, j + 1)]], _eb)
    assert w == [[F * ir.BW_GBS]]


def test_sm_partition_tile_cap_hand_examples():
    # uncapped 111 / 37 (see test_oracle_ir); tenant 0 capped at 20 -> the excess goes to 1
    assert ir.sm_partition([3, 1], 148, caps=[20, 1000]) == [20, 128]
    # caps that do not bind leave the proportional split unchanged
    assert ir.sm_partition([3, 1], 148, caps=[111, 37]) == [111, 37]
    # cascade: 0 over its cap first; after redistribution 1 goes over its cap too
    #   round 1 over {0,1,2}: R = 145 -> 1 + [72.5, 48.3, 24.2] -> [74, 49, 25]; 0 > 10
    #   round 2 over {1,2}, 138 SMs: R = 136 -> 1 + [90.7, 45.3] -> [92, 46]; 1 > 50
    #   round 3 over {2}, 88 SMs -> 88
    assert ir.sm_partition([6, 4, 2], 148, caps=[10, 50, 1000]) == [10, 50, 88]
    # every tenant capped: the proportional split stands (caps cannot absorb 148 SMs)
    assert ir.sm_partition([1, 1], 148, caps=[4, 4]) == [74, 74]
    # inactive tenants stay at 0, caps of 1 (single-tile ops)
    assert ir.sm_partition([None, 5, 5], 148, caps=[0, 1, 1000]) == [0, 1, 147]


def test_sm_partition_tile_cap_invariants():
    import random
    rnd = random.Random(5)
    for _ in range(400):
        n = rnd.randint(1, 6)
        w = [None if rnd.random() < 0.2 else rnd.randint(0, 10**12) for _ in range(n)]
        caps = [rnd.randint(1, 120) for _ in range(n)]
        out = ir.sm_partition(w, 148, caps)
        act = [t for t in range(n) if w[t] is not None]
        if not act:
            assert out == [0] * n
            continue
        assert sum(out) == 148
        assert all((out[t] >= 1) == (w[t] is not None) for t in range(n))
        if sum(caps[t] for t in act) >= 148:
            # a full GPU fits within the caps: no tenant exceeds its cap, none capped tenant
            # below its cap gets less than its share would be without the capped ones
            assert all(out[t] <= caps[t] for t in act) or all(out[t] > caps[t] for t in act)
