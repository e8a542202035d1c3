"""Pins of the forward oracle (oracle/forward.py, oracle/schedule.py) against independent library
routines (torch CPU fp64 functional ops, torchvision model definitions) and invariants."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import forward as fw
from oracle import ir
from oracle.schedule import run_schedule
from workloads import configs, zoo

RNG = np.random.default_rng(0)


def test_bf16_round_matches_torch_fp32_to_bf16():
    x = RNG.standard_normal(200000).astype(np.float32) * np.float32(3.0)
    # add exact ties: bf16 value + half a bf16 ulp, both parities
    base = torch.tensor(x[:1000]).to(torch.bfloat16).float().numpy()
    ulp = np.abs(base) * 2.0 ** -7
    ties = (base + ulp / 2).astype(np.float32)
    tiny = (RNG.standard_normal(1000) * 1e-39).astype(np.float32)    # fp32/bf16 subnormals
    big = np.array([3.3895e38, -3.3895e38, 1e38, 65504.0], np.float32)
    allx = np.concatenate([x, ties, tiny, big])
    ref = torch.tensor(allx).to(torch.bfloat16).double().numpy()
    got = fw.bf16_round(allx.astype(np.float64))
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("cin,cout,k,s,p,g,hw", [
    (3, 16, (3, 3), (1, 1), (1, 1), 1, (17, 19)),
    (8, 24, (5, 5), (2, 2), (2, 2), 1, (15, 16)),
    (16, 8, (1, 7), (1, 1), (0, 3), 1, (12, 12)),
    (16, 8, (7, 1), (1, 1), (3, 0), 1, (12, 12)),
    (32, 32, (3, 3), (2, 2), (1, 1), 32, (14, 13)),     # depthwise
    (8, 12, (3, 3), (1, 2), (1, 0), 2, (9, 11)),         # grouped, asymmetric stride/pad
    (3, 64, (7, 7), (2, 2), (3, 3), 1, (32, 32)),
    (3, 64, (11, 11), (4, 4), (2, 2), 1, (47, 47)),
])
def test_conv2d_vs_torch(cin, cout, k, s, p, g, hw):
    x = RNG.standard_normal((2, cin, *hw))
    w = RNG.standard_normal((cout, cin // g, *k))
    ref = F.conv2d(torch.tensor(x), torch.tensor(w), stride=s, padding=p, groups=g).numpy()
    got = fw.conv2d(x, w, s, p, g)
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("k,s,p,ceil,hw", [(3, 2, 1, False, (112, 112)), (2, 2, 0, False, (14, 14)),
                                           (3, 2, 0, True, (109, 109)), (3, 2, 0, True, (54, 54)),
                                           (3, 2, 0, True, (13, 13)), (3, 2, 0, False, (25, 25))])
def test_maxpool_vs_torch(k, s, p, ceil, hw):
    x = RNG.standard_normal((2, 5, *hw))
    ref = F.max_pool2d(torch.tensor(x), k, s, p, ceil_mode=ceil).numpy()
    np.testing.assert_array_equal(fw.maxpool2d(x, k, s, p, ceil), ref)


@pytest.mark.parametrize("k,s,p,ceil,cip,hw", [(3, 1, 1, False, True, (25, 25)),
                                               (3, 1, 1, False, False, (12, 12)),
                                               (3, 2, 1, True, True, (10, 10)),
                                               (3, 2, 1, True, False, (11, 11))])
def test_avgpool_vs_torch(k, s, p, ceil, cip, hw):
    x = RNG.standard_normal((2, 4, *hw))
    ref = F.avg_pool2d(torch.tensor(x), k, s, p, ceil_mode=ceil, count_include_pad=cip).numpy()
    np.testing.assert_allclose(fw.avgpool2d(x, k, s, p, ceil, cip), ref, rtol=1e-13, atol=1e-14)


def test_fc_and_gap_nodes_vs_torch():
    x = RNG.standard_normal((3, 16, 4, 4))
    w = RNG.standard_normal((10, 256)).astype(np.float32)
    b = RNG.standard_normal(10).astype(np.float32)
    node = dict(kind=fw.FC, act=1)
    y = fw.eval_node(node, dict(weight=w, scale=np.ones(10, np.float32), shift=b), [x], None)
    ref = F.relu(F.linear(torch.tensor(x).flatten(1), torch.tensor(w).double(), torch.tensor(b).double()))
    np.testing.assert_allclose(y.reshape(3, 10), ref.numpy(), rtol=1e-12, atol=1e-12)
    g = fw.eval_node(dict(kind=fw.GAP), {}, [x], None)
    np.testing.assert_allclose(g[:, :, 0, 0], F.adaptive_avg_pool2d(torch.tensor(x), 1).numpy()[:, :, 0, 0],
                               rtol=1e-13)


@pytest.mark.parametrize("act", [0, 1, 2])
def test_standalone_bn_relu_add_nodes_vs_torch(act):
    """The unfused BN / RELU / ADD operators (P:241 lists conv, bn, relu, pooling as the
    operator kinds; SURVEY a1 keeps standalone nodes schedulable) against torch's own BN
    (inference statistics), ReLU / ReLU6 and tensor sums."""
    C = 8
    x = RNG.standard_normal((2, C, 5, 6))
    acts = {0: lambda t: t, 1: F.relu, 2: F.relu6}
    # BN with running statistics, folded to (scale, shift) as the workload generator does
    mu, var = RNG.standard_normal(C), RNG.uniform(0.5, 2.0, C)
    gamma, beta, eps = RNG.uniform(0.5, 1.5, C), RNG.standard_normal(C), 1e-5
    scale = (gamma / np.sqrt(var + eps)).astype(np.float32)
    shift = (beta - mu * gamma / np.sqrt(var + eps)).astype(np.float32)
    ref = acts[act](F.batch_norm(torch.tensor(x), torch.tensor(mu), torch.tensor(var),
                                 torch.tensor(gamma), torch.tensor(beta), False, 0.0, eps)).numpy()
    y = fw.eval_node(dict(kind=fw.BN, act=act), dict(scale=scale, shift=shift), [x], None)
    np.testing.assert_allclose(y, ref, rtol=1e-6, atol=1e-6)   # fp32-rounded scale/shift
    # RELU node: its act field selects ReLU (1) or ReLU6 (2); 0 is the identity
    y = fw.eval_node(dict(kind=fw.RELU, act=act), {}, [x * 4], None)
    np.testing.assert_array_equal(y, acts[act](torch.tensor(x * 4)).numpy())
    # ADD of three inputs (+act): a sum, not a concat
    xs = [RNG.standard_normal((2, C, 5, 6)) for _ in range(3)]
    y = fw.eval_node(dict(kind=fw.ADD, act=act), {}, xs, None)
    ref = acts[act](torch.tensor(xs[0]) + torch.tensor(xs[1]) + torch.tensor(xs[2])).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-15, atol=1e-15)
    # storage rounding: bf16 mode rounds the op output like torch's fp32 -> bf16 cast
    yb = fw.eval_node(dict(kind=fw.ADD, act=act), {}, xs, None, mode="bf16")
    exp = torch.tensor(ref).float().bfloat16().double().numpy()
    np.testing.assert_array_equal(yb, exp)


# --- whole models vs torchvision (same weights, fp64) --------------------------------------

def _load_into_torchvision(graph, model):
    convs = [j for j, n in enumerate(graph.nodes) if n["kind"] == zoo.CONV]
    fcs = [j for j, n in enumerate(graph.nodes) if n["kind"] == zoo.FC]
    mods = list(model.modules())
    tconv = [m for m in mods if isinstance(m, torch.nn.Conv2d)]
    tfc = [m for m in mods if isinstance(m, torch.nn.Linear)]
    assert len(tconv) == len(convs) and len(tfc) == len(fcs)
    # the BN that follows each conv in registration order (if any)
    bn_after = {}
    last_conv = None
    for m in mods:
        if isinstance(m, torch.nn.Conv2d):
            last_conv = m
        elif isinstance(m, torch.nn.BatchNorm2d):
            bn_after[id(last_conv)] = m
    with torch.no_grad():
        for j, m in zip(convs, tconv):
            p = graph.params[j]
            assert tuple(m.weight.shape) == p["weight"].shape, (graph.name, j)
            m.weight.copy_(torch.tensor(p["weight"], dtype=torch.float64))
            bn = bn_after.get(id(m))
            if bn is not None:
                bn.running_mean.zero_()
                bn.running_var.fill_(1.0)
                bn.weight.copy_(torch.tensor(p["scale"], dtype=torch.float64) * np.sqrt(1.0 + bn.eps))
                bn.bias.copy_(torch.tensor(p["shift"], dtype=torch.float64))
            else:
                assert np.all(p["scale"] == 1)
                m.bias.copy_(torch.tensor(p["shift"], dtype=torch.float64))
        for j, m in zip(fcs, tfc):
            p = graph.params[j]
            m.weight.copy_(torch.tensor(p["weight"], dtype=torch.float64))
            m.bias.copy_(torch.tensor(p["shift"], dtype=torch.float64))


TV = {
    "resnet18": lambda tv: tv.resnet18(),
    "resnet50": lambda tv: tv.resnet50(),
    "mobilenet_v2": lambda tv: tv.mobilenet_v2(),
    "squeezenet1_0": lambda tv: tv.squeezenet1_0(),
    "inception_v3": lambda tv: tv.inception_v3(aux_logits=False, init_weights=False, transform_input=False),
    "vgg16": lambda tv: tv.vgg16(),
    "alexnet": lambda tv: tv.alexnet(),
    "resnet34": lambda tv: tv.resnet34(),
    "resnet101": lambda tv: tv.resnet101(),
}


@pytest.mark.parametrize("name", list(TV))
def test_model_zoo_and_oracle_vs_torchvision(name):
    """Pins both the zoo graph (structure, serialisation order, fusion) and the oracle forward
    pass against torchvision's own definitions, exact fp64 arithmetic (SURVEY c.4)."""
    tv = pytest.importorskip("torchvision.models")
    torch.manual_seed(0)
    g = zoo.MODELS[name]()
    model = TV[name](tv).double().eval()
    _load_into_torchvision(g, model)
    x = zoo.make_input(g)
    with torch.no_grad():
        ref = model(torch.tensor(x, dtype=torch.float64)).numpy()
    got = fw.forward(g, x, "exact")
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 1e-9 * scale


@pytest.mark.parametrize("name", ["tinyA", "tinyB"])
def test_tiny_models_vs_torch_functional(name):
    g = zoo.MODELS[name]()
    x = zoo.make_input(g)
    t = torch.tensor(x, dtype=torch.float64)
    acts = []
    for j, n in enumerate(g.nodes):
        p = g.params[j]
        src = t if n["inputs"] == [-1] else acts[n["inputs"][0]]
        if n["kind"] == zoo.CONV:
            y = F.conv2d(src, torch.tensor(p["weight"]).double(), stride=n["sh"], padding=n["ph"])
            y = y * torch.tensor(p["scale"]).double()[None, :, None, None] + \
                torch.tensor(p["shift"]).double()[None, :, None, None]
            y = F.relu(y)
        elif n["kind"] == zoo.GAP:
            y = F.adaptive_avg_pool2d(src, 1)
        elif n["kind"] == zoo.MAXPOOL:
            y = F.max_pool2d(src, n["kh"], n["sh"])
        elif n["kind"] == zoo.FC:
            y = F.linear(src.flatten(1), torch.tensor(p["weight"]).double(), torch.tensor(p["shift"]).double())
        acts.append(y)
    np.testing.assert_allclose(fw.forward(g, x, "exact"), acts[-1].numpy(), rtol=1e-10, atol=1e-12)


def test_storage_modes_bounded_drift():
    for name in ("tinyA", "tinyB"):
        g = zoo.MODELS[name]()
        x = zoo.make_input(g)
        ex = fw.forward(g, x, "exact")
        f32 = fw.forward(g, x, "fp32")
        b16 = fw.forward(g, x, "bf16")
        s = np.abs(ex).max()
        assert np.abs(f32 - ex).max() <= 1e-6 * s
        assert 0 < np.abs(b16 - ex).max() <= 1e-2 * s


def test_schedule_oracle_equals_sequential_forward():
    gs = configs.tenants("c1")
    L = [g.n_ops for g in gs]
    xs = [zoo.make_input(g) for g in gs]
    seq = [fw.forward(g, x, "fp32") for g, x in zip(gs, xs)]
    scheds = [configs.c1_schedule_pointers(), configs.all_concurrent_pointers(L),
              configs.sequential_pointers(L), configs.uniform_pointers(L)]
    for rho in scheds:
        st, ranges = ir.T(L, rho)
        assert st[0] == ir.E_OK
        outs = run_schedule(gs, ranges, xs, "fp32")
        for a, b in zip(outs, seq):
            np.testing.assert_array_equal(a, b)


def test_schedule_oracle_rejects_invalid():
    gs = configs.tenants("c1")
    xs = [zoo.make_input(g) for g in gs]
    with pytest.raises(ValueError):
        run_schedule(gs, [[(0, 3), (0, 6)]], xs)
