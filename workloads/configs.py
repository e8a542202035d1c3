"""BASELINE.json configs as seeded synthetic workloads and the
seeded candidate-schedule generator of config 5 (reading R13).

Pure data: lists of tenant graphs and pointer matrices.  No schedule semantics
(validation, stage construction) lives here -- infeasible candidates are kept and
filtered by the library / oracle validation, as the paper filters them.
"""
from __future__ import annotations

import random

from . import zoo

CONFIGS = {
    # name: (tenant model names, batch, precision, description)
    "c1": (("tinyA", "tinyB"), 1, zoo.PREC_FP32,
           "2 tiny CNNs (4 conv+pool+FC, 32x32x3, batch 1), hand-written 3-stage schedule"),
    "c2": (("resnet18", "mobilenet_v2"), 1, zoo.PREC_BF16, "ResNet-18 + MobileNet-V2, 224x224 b1"),
    "c3": (("resnet50", "vgg16", "mobilenet_v2"), 1, zoo.PREC_BF16,
           "ResNet-50 + VGG-16 + MobileNet-V2, 224x224 b1"),
    "c4": (("resnet50", "inception_v3", "vgg16", "mobilenet_v2", "squeezenet1_0"), 1,
           zoo.PREC_BF16, "5-tenant mix b1"),
    "c4b8": (("resnet50", "inception_v3", "vgg16", "mobilenet_v2", "squeezenet1_0"), 8,
             zoo.PREC_BF16, "5-tenant mix b8"),
    # paper zoo mixes (Table I, Table II) -- SURVEY §8(f) f2
    "vgg_r18": (("vgg16", "resnet18"), 1, zoo.PREC_BF16, "Table I VGG+R18"),
    "r18_r34": (("resnet18", "resnet34"), 1, zoo.PREC_BF16, "Table I R18+R34"),
    "r34_r50": (("resnet34", "resnet50"), 1, zoo.PREC_BF16, "Table I R34+R50"),
    "r50_r101": (("resnet50", "resnet101"), 1, zoo.PREC_BF16, "Table I R50+R101"),
    "vgg_r18_r50": (("vgg16", "resnet18", "resnet50"), 1, zoo.PREC_BF16, "Table I/II VGG+R18+R50"),
    "r18_r34_r50": (("resnet18", "resnet34", "resnet50"), 1, zoo.PREC_BF16, "Table I/II R18+R34+R50"),
    "zoo5": (("vgg16", "resnet18", "resnet34", "resnet50", "resnet101"), 1, zoo.PREC_BF16,
             "Table I VGG+R18+R34+R50+R101"),
    "alex_vgg_r18": (("alexnet", "vgg16", "resnet18"), 1, zoo.PREC_BF16, "Table II Alex+VGG+R18"),
    "r18_r34_r101": (("resnet18", "resnet34", "resnet101"), 1, zoo.PREC_BF16, "Table II R18+R34+R101"),
    "r18_r50_r101": (("resnet18", "resnet50", "resnet101"), 1, zoo.PREC_BF16, "Table II R18+R50+R101"),
    # the f2 architectures not in configs 1-4, for per-op parity
    "f2_models": (("alexnet", "resnet34", "resnet101"), 1, zoo.PREC_BF16, "AlexNet+R34+R101 (parity)"),
    # single tenants (profiling the per-op dependency chain)
    "mbv2": (("mobilenet_v2",), 1, zoo.PREC_BF16, "MobileNet-V2 alone"),
    "r18": (("resnet18",), 1, zoo.PREC_BF16, "ResNet-18 alone"),
    "r50": (("resnet50",), 1, zoo.PREC_BF16, "ResNet-50 alone"),
    "vgg": (("vgg16",), 1, zoo.PREC_BF16, "VGG-16 alone"),
    "inc3": (("inception_v3",), 1, zoo.PREC_BF16, "Inception-v3 alone"),
    "sqz": (("squeezenet1_0",), 1, zoo.PREC_BF16, "SqueezeNet 1.0 alone"),
    "vgg_b8": (("vgg16",), 8, zoo.PREC_BF16, "VGG-16 alone, batch 8"),
}


def tenants(config: str, precision=None, batch=None):
    names, b, prec, _ = CONFIGS[config]
    prec = prec if precision is None else precision
    b = b if batch is None else batch
    return [zoo.MODELS[n](batch=b, precision=prec) for n in names]


def c1_schedule_pointers():
    """Config 1 hand-written 3-stage schedule (d.1): A rho=(2,4) -> [1,2],[3,4],[5,6];
    B rho=(1,4) -> [1],[2,3,4],[5,6]."""
    return [[2, 4], [1, 4]]


def all_concurrent_pointers(lengths):
    """P = 0: one stage holding every tenant's whole sequence."""
    return [[] for _ in lengths]


def sequential_pointers(lengths):
    """P = N-1; row i = (0,..,0, L_i,..,L_i) with the first L_i at position i (SURVEY c.4)."""
    n = len(lengths)
    return [[0] * i + [L] * (n - 1 - i) for i, L in enumerate(lengths)]


def uniform_pointers(lengths, stages=4):
    """rho_i[k] = floor(k*L_i/stages + 1/2), k = 1..stages-1 (d.1 'uniform 4-stage')."""
    return [[(2 * k * L + stages) // (2 * stages) for k in range(1, stages)] for L in lengths]


def sample_candidates(lengths, n, seed=14255, p_max=8):
    """Config-5 candidate generator (reading R13): candidates 0 and 1 are the two
    extremes; the rest draw P ~ U{1..p_max} and P i.i.d. U{0..L_i} per row, sorted
    (non-decreasing rows).  Exact duplicate matrices are re-drawn.  Infeasible
    matrices (an all-empty stage) are NOT removed here: validation filters them."""
    rng = random.Random(seed)
    out = [all_concurrent_pointers(lengths), sequential_pointers(lengths)]
    seen = {repr(out[0]), repr(out[1])}
    while len(out) < n:
        P = rng.randint(1, p_max)
        rho = [sorted(rng.randint(0, L) for _ in range(P)) for L in lengths]
        key = repr(rho)
        if key in seen:
            continue
        seen.add(key)
        out.append(rho)
    return out[:n]
