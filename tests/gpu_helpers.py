"""Shared helpers of the -m gpu parity tests (CUDA path vs the CPU oracle)."""
import numpy as np

from oracle import forward as fw
from workloads import zoo


def act_to_nchw(a, dtype_is_bf16):
    """GPU activation (NHWC, bf16 as uint16 or fp32) -> float64 NCHW"""
    if dtype_is_bf16:
        a = (a.astype(np.uint32) << 16).view(np.float32)
    return a.astype(np.float64).transpose(0, 3, 1, 2)


def gpu_activations(mix, t):
    """all op outputs of tenant t except the final op, as float64 NCHW"""
    g = mix.graphs[t]
    bf = g.precision == zoo.PREC_BF16
    acts = {}
    for j in range(g.n_ops - 1):
        c, h, w = g.shapes[j]
        raw = mix.ctx.get_activation(t, j, (g.batch, h, w, c), np.uint16 if bf else np.float32)
        acts[j] = act_to_nchw(raw, bf)
    return acts


def rel_err(got, ref):
    s = np.abs(ref).max()
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / (s if s > 0 else 1.0))


def teacher_forced_errors(mix, x, t):
    """per-op errors: the oracle recomputes op j from the GPU's own inputs (SURVEY c.5)"""
    g = mix.graphs[t]
    mode = "bf16" if g.precision == zoo.PREC_BF16 else "fp32"
    acts = gpu_activations(mix, t)
    out = mix.outputs[t].cpu().numpy().reshape(g.batch, -1)
    errs = []
    for j in range(g.n_ops):
        ref = fw.eval_op_teacher_forced(g, j, acts, x, mode)
        got = acts[j] if j < g.n_ops - 1 else None
        if got is None:
            errs.append(rel_err(out, ref.reshape(g.batch, -1)))
        else:
            errs.append(rel_err(got, ref))
    return errs
