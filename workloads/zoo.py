"""Seeded synthetic workloads: tenant CNN graphs, weights, inputs.

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle.  It holds no arithmetic of the method (no convolution, pooling,
scheduling or stage logic): it only *describes* networks node by node and
draws seeded random numbers for their parameters and inputs.

Graph description = the paper's operator sequence (Eq.1):
each model is one list of operators in a topological order, multi-branch
models serialised (footnote P:268).  Operator granularity is the fused-kernel
granularity of DESIGN.md reading R6: a CONV node is conv -> per-channel affine
(folded BN or bias) -> (+ residual) -> activation.

Node fields mirror `mt_node` in include/mt.h:
  kind, inputs (ids < own id, -1 = graph input; several ids = channel concat for
  CONV/POOL/FC, elementwise sum for ADD), out_c/out_h/out_w, kh, kw, sh, sw, ph, pw,
  groups, ceil_mode, count_include_pad, act (0 none, 1 relu, 2 relu6), residual.
Parameter arrays (float32, PyTorch layouts):
  CONV weight [Cout][Cin/groups][kh][kw], FC weight [out][in] (in = NCHW flatten
  index of the, possibly concatenated, input), scale/shift [Cout].

Weight recipe: LeCun-normal N(0, 1/fan_in) weights,
biases U(+-1/sqrt(fan_in)), BN folded with identity running stats:
scale ~ U(0.9, 1.1), shift ~ U(-0.1, 0.1).  Weights and inputs are rounded to
bf16-representable float32 values (round-to-nearest-even on the float32 bit
pattern) so that bf16 storage on the GPU and fp64 arithmetic in the oracle see
exactly the same parameter values.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# op kinds (include/mt.h mt_op_kind)
CONV, BN, RELU, MAXPOOL, AVGPOOL, GAP, FC, ADD = 1, 2, 3, 4, 5, 6, 7, 8
KIND_NAMES = {CONV: "conv", BN: "bn", RELU: "relu", MAXPOOL: "maxpool", AVGPOOL: "avgpool",
              GAP: "gap", FC: "fc", ADD: "add"}
ACT_NONE, ACT_RELU, ACT_RELU6 = 0, 1, 2
PREC_BF16, PREC_FP32 = 0, 1

MODEL_IDS = {"tinyA": 0, "tinyB": 1, "resnet18": 2, "mobilenet_v2": 3, "resnet50": 4,
             "vgg16": 5, "inception_v3": 6, "squeezenet1_0": 7, "alexnet": 8,
             "resnet34": 9, "resnet101": 10}


def bf16_representable(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16-representable float32 (RNE on bits).

    Input generation only (makes the generated parameters exactly bf16); the
    oracle has its own independent rounding routine for activations.
    """
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


@dataclass
class Graph:
    name: str
    batch: int
    in_c: int
    in_h: int
    in_w: int
    precision: int
    nodes: list = field(default_factory=list)      # list of dicts (mt_node fields)
    params: list = field(default_factory=list)     # list of dicts {weight, scale, shift} or {}
    shapes: list = field(default_factory=list)     # (C, H, W) per node, from the builder

    @property
    def n_ops(self):
        return len(self.nodes)

    @property
    def out_classes(self):
        n = self.nodes[-1]
        return n["out_c"] * n["out_h"] * n["out_w"]


def _pool_out(size, k, s, p, ceil_mode):
    if ceil_mode:
        o = -(-(size + 2 * p - k) // s) + 1
        if (o - 1) * s >= size + p:
            o -= 1
        return o
    return (size + 2 * p - k) // s + 1


class GraphBuilder:
    """Builds one tenant graph node by node, drawing its parameters in node order."""

    def __init__(self, name, batch=1, in_c=3, in_h=224, in_w=224, precision=PREC_BF16, seed=None):
        self.g = Graph(name, batch, in_c, in_h, in_w, precision)
        if seed is None:
            seed = 1000 + MODEL_IDS[name]
        self.rng = np.random.default_rng(seed)

    # -- helpers ---------------------------------------------------------
    def _shape(self, x):
        if isinstance(x, (list, tuple)):
            shp = [self._shape(i) for i in x]
            assert all(s[1:] == shp[0][1:] for s in shp), "concat spatial mismatch"
            return (sum(s[0] for s in shp), shp[0][1], shp[0][2])
        if x == -1:
            return (self.g.in_c, self.g.in_h, self.g.in_w)
        return self.g.shapes[x]

    @staticmethod
    def _ids(x):
        return list(x) if isinstance(x, (list, tuple)) else [x]

    def _add(self, node, shape, params):
        base = dict(kind=0, inputs=[], out_c=0, out_h=0, out_w=0, kh=1, kw=1, sh=1, sw=1,
                    ph=0, pw=0, groups=1, ceil_mode=0, count_include_pad=0, act=ACT_NONE,
                    residual=-1)
        base.update(node)
        base["out_c"], base["out_h"], base["out_w"] = shape
        self.g.nodes.append(base)
        self.g.shapes.append(shape)
        self.g.params.append(params)
        return len(self.g.nodes) - 1

    def _w(self, shape, fan_in):
        w = self.rng.standard_normal(shape, dtype=np.float64) / math.sqrt(fan_in)
        return bf16_representable(w.astype(np.float32))

    # -- ops ---------------------------------------------------------------
    def conv(self, x, cout, k, s=1, p=0, groups=1, act=ACT_RELU, bn=True, bias=False,
             residual=None):
        cin, h, w = self._shape(x)
        kh, kw = (k, k) if isinstance(k, int) else k
        sh, sw = (s, s) if isinstance(s, int) else s
        ph, pw = (p, p) if isinstance(p, int) else p
        assert cin % groups == 0 and cout % groups == 0
        fan_in = (cin // groups) * kh * kw
        weight = self._w((cout, cin // groups, kh, kw), fan_in)
        if bn:
            scale = self.rng.uniform(0.9, 1.1, cout).astype(np.float32)
            shift = self.rng.uniform(-0.1, 0.1, cout).astype(np.float32)
        elif bias:
            bnd = 1.0 / math.sqrt(fan_in)
            scale = np.ones(cout, np.float32)
            shift = self.rng.uniform(-bnd, bnd, cout).astype(np.float32)
        else:
            scale = np.ones(cout, np.float32)
            shift = np.zeros(cout, np.float32)
        ho = (h + 2 * ph - kh) // sh + 1
        wo = (w + 2 * pw - kw) // sw + 1
        if residual is not None:
            assert self._shape(residual) == (cout, ho, wo)
        node = dict(kind=CONV, inputs=self._ids(x), kh=kh, kw=kw, sh=sh, sw=sw, ph=ph, pw=pw,
                    groups=groups, act=act, residual=-1 if residual is None else residual)
        return self._add(node, (cout, ho, wo), dict(weight=weight, scale=scale, shift=shift))

    def maxpool(self, x, k, s, p=0, ceil_mode=False):
        c, h, w = self._shape(x)
        ho, wo = _pool_out(h, k, s, p, ceil_mode), _pool_out(w, k, s, p, ceil_mode)
        node = dict(kind=MAXPOOL, inputs=self._ids(x), kh=k, kw=k, sh=s, sw=s, ph=p, pw=p,
                    ceil_mode=int(ceil_mode))
        return self._add(node, (c, ho, wo), {})

    def avgpool(self, x, k, s, p=0, count_include_pad=True, ceil_mode=False):
        c, h, w = self._shape(x)
        ho, wo = _pool_out(h, k, s, p, ceil_mode), _pool_out(w, k, s, p, ceil_mode)
        node = dict(kind=AVGPOOL, inputs=self._ids(x), kh=k, kw=k, sh=s, sw=s, ph=p, pw=p,
                    count_include_pad=int(count_include_pad), ceil_mode=int(ceil_mode))
        return self._add(node, (c, ho, wo), {})

    def gap(self, x):
        c, h, w = self._shape(x)
        node = dict(kind=GAP, inputs=self._ids(x), kh=h, kw=w)
        return self._add(node, (c, 1, 1), {})

    def fc(self, x, out, act=ACT_NONE, bias=True):
        c, h, w = self._shape(x)
        fan_in = c * h * w
        weight = self._w((out, fan_in), fan_in)
        bnd = 1.0 / math.sqrt(fan_in)
        shift = (self.rng.uniform(-bnd, bnd, out) if bias else np.zeros(out)).astype(np.float32)
        scale = np.ones(out, np.float32)
        node = dict(kind=FC, inputs=self._ids(x), act=act)
        return self._add(node, (out, 1, 1), dict(weight=weight, scale=scale, shift=shift))

    def add(self, xs, act=ACT_NONE):
        shp = [self._shape(i) for i in xs]
        assert all(s == shp[0] for s in shp)
        node = dict(kind=ADD, inputs=list(xs), act=act)
        return self._add(node, shp[0], {})

    def bn(self, x, act=ACT_NONE):
        c, h, w = self._shape(x)
        scale = self.rng.uniform(0.9, 1.1, c).astype(np.float32)
        shift = self.rng.uniform(-0.1, 0.1, c).astype(np.float32)
        node = dict(kind=BN, inputs=self._ids(x), act=act)
        return self._add(node, (c, h, w), dict(scale=scale, shift=shift))

    def relu(self, x, act=ACT_RELU):
        node = dict(kind=RELU, inputs=self._ids(x), act=act)
        return self._add(node, self._shape(x), {})

    def build(self):
        return self.g


# ----------------------------------------------------------------------------
# Model zoo (torchvision 0.26 architectures at fused granularity)
# ----------------------------------------------------------------------------

def tinyA(batch=1, precision=PREC_FP32):
    """Config 1 TinyA: 4 conv+BN+ReLU, GAP, FC 64->10; 32x32 input."""
    b = GraphBuilder("tinyA", batch, 3, 32, 32, precision)
    x = b.conv(-1, 16, 3, 1, 1)
    x = b.conv(x, 32, 3, 2, 1)
    x = b.conv(x, 32, 3, 1, 1)
    x = b.conv(x, 64, 3, 2, 1)
    x = b.gap(x)
    b.fc(x, 10)
    return b.build()


def tinyB(batch=1, precision=PREC_FP32):
    """Config 1 TinyB: conv5x5 3->8, conv3x3 8->16, conv3x3 16->16 s2, conv1x1 16->32,
    maxpool 2x2, FC 2048->10."""
    b = GraphBuilder("tinyB", batch, 3, 32, 32, precision)
    x = b.conv(-1, 8, 5, 1, 2)
    x = b.conv(x, 16, 3, 1, 1)
    x = b.conv(x, 16, 3, 2, 1)
    x = b.conv(x, 32, 1, 1, 0)
    x = b.maxpool(x, 2, 2)
    b.fc(x, 10)
    return b.build()


def _resnet(name, block, layers, batch, precision):
    b = GraphBuilder(name, batch, 3, 224, 224, precision)
    x = b.conv(-1, 64, 7, 2, 3)
    x = b.maxpool(x, 3, 2, 1)
    cin = 64
    for stage, (planes, n) in enumerate(zip((64, 128, 256, 512), layers)):
        for i in range(n):
            stride = 2 if (i == 0 and stage > 0) else 1
            if block == "basic":
                cout = planes
                need_ds = stride != 1 or cin != cout
                h = b.conv(x, planes, 3, stride, 1)
                if need_ds:
                    # torch.fx order: conv1, conv2/bn2, downsample, add, relu -> the
                    # downsample conv absorbs the residual add + ReLU (R5).
                    h = b.conv(h, planes, 3, 1, 1, act=ACT_NONE)
                    x = b.conv(x, cout, 1, stride, 0, act=ACT_RELU, residual=h)
                else:
                    x = b.conv(h, planes, 3, 1, 1, act=ACT_RELU, residual=x)
            else:
                cout = planes * 4
                need_ds = stride != 1 or cin != cout
                h = b.conv(x, planes, 1, 1, 0)
                h = b.conv(h, planes, 3, stride, 1)          # v1.5: stride on the 3x3
                if need_ds:
                    h = b.conv(h, cout, 1, 1, 0, act=ACT_NONE)
                    x = b.conv(x, cout, 1, stride, 0, act=ACT_RELU, residual=h)
                else:
                    x = b.conv(h, cout, 1, 1, 0, act=ACT_RELU, residual=x)
            cin = cout
    x = b.gap(x)
    b.fc(x, 1000)
    return b.build()


def resnet18(batch=1, precision=PREC_BF16):
    return _resnet("resnet18", "basic", (2, 2, 2, 2), batch, precision)


def resnet34(batch=1, precision=PREC_BF16):
    return _resnet("resnet34", "basic", (3, 4, 6, 3), batch, precision)


def resnet50(batch=1, precision=PREC_BF16):
    return _resnet("resnet50", "bottleneck", (3, 4, 6, 3), batch, precision)


def resnet101(batch=1, precision=PREC_BF16):
    return _resnet("resnet101", "bottleneck", (3, 4, 23, 3), batch, precision)


def mobilenet_v2(batch=1, precision=PREC_BF16):
    b = GraphBuilder("mobilenet_v2", batch, 3, 224, 224, precision)
    x = b.conv(-1, 32, 3, 2, 1, act=ACT_RELU6)
    cin = 32
    setting = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
               (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]
    for t, c, n, s in setting:
        for i in range(n):
            stride = s if i == 0 else 1
            hidden = cin * t
            use_res = stride == 1 and cin == c
            h = x
            if t != 1:
                h = b.conv(h, hidden, 1, 1, 0, act=ACT_RELU6)
            h = b.conv(h, hidden, 3, stride, 1, groups=hidden, act=ACT_RELU6)
            x = b.conv(h, c, 1, 1, 0, act=ACT_NONE, residual=x if use_res else None)
            cin = c
    x = b.conv(x, 1280, 1, 1, 0, act=ACT_RELU6)
    x = b.gap(x)
    b.fc(x, 1000)
    return b.build()


def vgg16(batch=1, precision=PREC_BF16):
    """VGG-16 without BN; the adaptive avg-pool is the identity at 224 and is elided."""
    b = GraphBuilder("vgg16", batch, 3, 224, 224, precision)
    x = -1
    for v in (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
              512, 512, 512, "M"):
        if v == "M":
            x = b.maxpool(x, 2, 2)
        else:
            x = b.conv(x, v, 3, 1, 1, bn=False, bias=True)
    x = b.fc(x, 4096, act=ACT_RELU)
    x = b.fc(x, 4096, act=ACT_RELU)
    b.fc(x, 1000)
    return b.build()


def alexnet(batch=1, precision=PREC_BF16):
    b = GraphBuilder("alexnet", batch, 3, 224, 224, precision)
    x = b.conv(-1, 64, 11, 4, 2, bn=False, bias=True)
    x = b.maxpool(x, 3, 2)
    x = b.conv(x, 192, 5, 1, 2, bn=False, bias=True)
    x = b.maxpool(x, 3, 2)
    x = b.conv(x, 384, 3, 1, 1, bn=False, bias=True)
    x = b.conv(x, 256, 3, 1, 1, bn=False, bias=True)
    x = b.conv(x, 256, 3, 1, 1, bn=False, bias=True)
    x = b.maxpool(x, 3, 2)
    x = b.fc(x, 4096, act=ACT_RELU)
    x = b.fc(x, 4096, act=ACT_RELU)
    b.fc(x, 1000)
    return b.build()


def squeezenet1_0(batch=1, precision=PREC_BF16):
    b = GraphBuilder("squeezenet1_0", batch, 3, 224, 224, precision)
    x = b.conv(-1, 96, 7, 2, 0, bn=False, bias=True)
    x = b.maxpool(x, 3, 2, 0, ceil_mode=True)

    def fire(x, sq, e1, e3):
        s = b.conv(x, sq, 1, 1, 0, bn=False, bias=True)
        a = b.conv(s, e1, 1, 1, 0, bn=False, bias=True)
        c = b.conv(s, e3, 3, 1, 1, bn=False, bias=True)
        return [a, c]

    x = fire(x, 16, 64, 64)
    x = fire(x, 16, 64, 64)
    x = fire(x, 32, 128, 128)
    x = b.maxpool(x, 3, 2, 0, ceil_mode=True)
    x = fire(x, 32, 128, 128)
    x = fire(x, 48, 192, 192)
    x = fire(x, 48, 192, 192)
    x = fire(x, 64, 256, 256)
    x = b.maxpool(x, 3, 2, 0, ceil_mode=True)
    x = fire(x, 64, 256, 256)
    x = b.conv(x, 1000, 1, 1, 0, bn=False, bias=True)
    b.gap(x)
    return b.build()


def inception_v3(batch=1, precision=PREC_BF16, size=224):
    """Inception-v3 at 224x224 (R15), no aux head, transform_input off.  `size` only
    serves the oracle pin against torchvision's published cost at its native 299x299."""
    b = GraphBuilder("inception_v3", batch, 3, size, size, precision)
    C = b.conv
    x = C(-1, 32, 3, 2, 0)
    x = C(x, 32, 3, 1, 0)
    x = C(x, 64, 3, 1, 1)
    x = b.maxpool(x, 3, 2)
    x = C(x, 80, 1, 1, 0)
    x = C(x, 192, 3, 1, 0)
    x = b.maxpool(x, 3, 2)

    def block_a(x, pool_features):
        b1 = C(x, 64, 1)
        b5 = C(C(x, 48, 1), 64, 5, 1, 2)
        b3 = C(C(C(x, 64, 1), 96, 3, 1, 1), 96, 3, 1, 1)
        bp = C(b.avgpool(x, 3, 1, 1), pool_features, 1)
        return [b1, b5, b3, bp]

    def block_b(x):
        b3 = C(x, 384, 3, 2, 0)
        bd = C(C(C(x, 64, 1), 96, 3, 1, 1), 96, 3, 2, 0)
        bp = b.maxpool(x, 3, 2)
        return [b3, bd, bp]

    def block_c(x, c7):
        b1 = C(x, 192, 1)
        b7 = C(C(C(x, c7, 1), c7, (1, 7), 1, (0, 3)), 192, (7, 1), 1, (3, 0))
        bd = C(x, c7, 1)
        bd = C(bd, c7, (7, 1), 1, (3, 0))
        bd = C(bd, c7, (1, 7), 1, (0, 3))
        bd = C(bd, c7, (7, 1), 1, (3, 0))
        bd = C(bd, 192, (1, 7), 1, (0, 3))
        bp = C(b.avgpool(x, 3, 1, 1), 192, 1)
        return [b1, b7, bd, bp]

    def block_d(x):
        b3 = C(C(x, 192, 1), 320, 3, 2, 0)
        b7 = C(x, 192, 1)
        b7 = C(b7, 192, (1, 7), 1, (0, 3))
        b7 = C(b7, 192, (7, 1), 1, (3, 0))
        b7 = C(b7, 192, 3, 2, 0)
        bp = b.maxpool(x, 3, 2)
        return [b3, b7, bp]

    def block_e(x):
        b1 = C(x, 320, 1)
        b3 = C(x, 384, 1)
        b3a = C(b3, 384, (1, 3), 1, (0, 1))
        b3b = C(b3, 384, (3, 1), 1, (1, 0))
        bd = C(C(x, 448, 1), 384, 3, 1, 1)
        bda = C(bd, 384, (1, 3), 1, (0, 1))
        bdb = C(bd, 384, (3, 1), 1, (1, 0))
        bp = C(b.avgpool(x, 3, 1, 1), 192, 1)
        return [b1, b3a, b3b, bda, bdb, bp]

    x = block_a(x, 32)
    x = block_a(x, 64)
    x = block_a(x, 64)
    x = block_b(x)
    x = block_c(x, 128)
    x = block_c(x, 160)
    x = block_c(x, 160)
    x = block_c(x, 192)
    x = block_d(x)
    x = block_e(x)
    x = block_e(x)
    x = b.gap(x)
    b.fc(x, 1000)
    return b.build()


MODELS = {"tinyA": tinyA, "tinyB": tinyB, "resnet18": resnet18, "resnet34": resnet34,
          "resnet50": resnet50, "resnet101": resnet101, "mobilenet_v2": mobilenet_v2,
          "vgg16": vgg16, "alexnet": alexnet, "squeezenet1_0": squeezenet1_0,
          "inception_v3": inception_v3}


def make_input(graph: Graph, seed: int = 1) -> np.ndarray:
    """Shared synthetic input x ~ N(0,1), NCHW float32, bf16-representable (d.1, seed 1)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((graph.batch, graph.in_c, graph.in_h, graph.in_w), dtype=np.float64)
    return bf16_representable(x.astype(np.float32))
