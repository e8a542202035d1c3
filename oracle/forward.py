"""Forward oracle: the plain tenant-network forward pass (TEST INFRASTRUCTURE ONLY).

What a schedule computes: a schedule changes WHEN operators run, never
WHAT they compute -- within a model data-flow order is kept ("operators ... must be performed
in certain order according to the data flow dependency"), across models operators are
independent and barriers only delay.  So the result of any valid schedule is
y_i = M_i(x_i), the ordinary forward pass of every tenant network on the shared input.

This module writes that forward pass out in float64, NCHW (deliberately unlike the GPU's NHWC),
with plain definitions:
  conv  : y[n,o,p,q] = sum_{c,r,s} w[o,c,r,s] * xpad[n, c, p*sh + r, q*sw + s]   (per tap,
          numpy tensordot is the library matmul step); groups split channels;
  fused : y = act(scale[o] * conv + shift[o] + residual)       (conv -> folded BN/bias -> add -> act)
  pools : max / average over the PyTorch window definition (padding, ceil_mode,
          count_include_pad), global average = mean over H*W;
  fc    : y = W x + b over the NCHW flatten of the (concatenated) input;
  concat: several inputs of a CONV/POOL/FC are concatenated along channels, summed for ADD.

Storage emulation (mode):
  'exact' -- no rounding (fp64 throughout);
  'bf16'  -- inputs/parameters rounded to bf16 and every op output rounded to bf16 (RNE) before
             the next op; the graph's final op is rounded to fp32 (the GPU writes fp32 logits);
  'fp32'  -- every op output rounded to fp32.
"""
from __future__ import annotations

import numpy as np

CONV, BN, RELU, MAXPOOL, AVGPOOL, GAP, FC, ADD = 1, 2, 3, 4, 5, 6, 7, 8


def bf16_round(x):
    """Round float64 values to the nearest bfloat16 value, ties to even, directly from fp64.
    bf16 = 8 significant bits, exponent range of fp32 (min normal 2^-126, subnormal quantum
    2^-133, max (2 - 2^-7) * 2^127)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    nz = (x != 0) & np.isfinite(x)
    m, e = np.frexp(x[nz])                          # x = m * 2^e, 0.5 <= |m| < 1
    q_exp = np.maximum(e - 8, -133)                 # quantum exponent
    v = np.ldexp(np.rint(np.ldexp(x[nz], -q_exp)), q_exp)   # rint: half to even
    maxv = np.ldexp(2.0 - 2.0 ** -7, 127)
    v = np.where(np.abs(v) > maxv, np.copysign(np.inf, v), v)
    out[nz] = v
    out[~np.isfinite(x)] = x[~np.isfinite(x)]
    return out


def fp32_round(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def _round(x, mode):
    if mode == "bf16":
        return bf16_round(x)
    if mode == "fp32":
        return fp32_round(x)
    return np.asarray(x, dtype=np.float64)


def conv2d(x, w, stride=(1, 1), pad=(0, 0), groups=1):
    """Cross-correlation as in every DNN framework, summed tap by tap."""
    n, c, h, wd = x.shape
    o, cg, kh, kw = w.shape
    sh, sw = stride
    ph, pw = pad
    ho = (h + 2 * ph - kh) // sh + 1
    wo = (wd + 2 * pw - kw) // sw + 1
    xp = np.zeros((n, c, h + 2 * ph, wd + 2 * pw), dtype=np.float64)
    xp[:, :, ph:ph + h, pw:pw + wd] = x
    y = np.zeros((n, o, ho, wo), dtype=np.float64)
    og = o // groups
    for r in range(kh):
        for s in range(kw):
            patch = xp[:, :, r:r + sh * (ho - 1) + 1:sh, s:s + sw * (wo - 1) + 1:sw]
            if groups == 1:
                y += np.tensordot(w[:, :, r, s], patch, axes=([1], [1])).transpose(1, 0, 2, 3)
            elif groups == c and cg == 1 and og == 1:
                y += w[:, 0, r, s][None, :, None, None] * patch
            else:
                for g in range(groups):
                    wg = w[g * og:(g + 1) * og, :, r, s]
                    pg = patch[:, g * cg:(g + 1) * cg]
                    y[:, g * og:(g + 1) * og] += np.tensordot(wg, pg, axes=([1], [1])).transpose(1, 0, 2, 3)
    return y


def _pool_out(size, k, s, p, ceil_mode):
    if ceil_mode:
        o = -(-(size + 2 * p - k) // s) + 1
        if (o - 1) * s >= size + p:     # last window must start inside input or left padding
            o -= 1
        return o
    return (size + 2 * p - k) // s + 1


def maxpool2d(x, k, s, p, ceil_mode=False):
    n, c, h, w = x.shape
    ho, wo = _pool_out(h, k, s, p, ceil_mode), _pool_out(w, k, s, p, ceil_mode)
    y = np.full((n, c, ho, wo), -np.inf)
    for i in range(ho):
        h0, h1 = max(i * s - p, 0), min(i * s - p + k, h)
        for j in range(wo):
            w0, w1 = max(j * s - p, 0), min(j * s - p + k, w)
            y[:, :, i, j] = x[:, :, h0:h1, w0:w1].max(axis=(2, 3))
    return y


def avgpool2d(x, k, s, p, ceil_mode=False, count_include_pad=True):
    n, c, h, w = x.shape
    ho, wo = _pool_out(h, k, s, p, ceil_mode), _pool_out(w, k, s, p, ceil_mode)
    y = np.zeros((n, c, ho, wo))
    for i in range(ho):
        hs = i * s - p
        he = min(hs + k, h + p)
        for j in range(wo):
            ws = j * s - p
            we = min(ws + k, w + p)
            div = (he - hs) * (we - ws)
            h0, h1, w0, w1 = max(hs, 0), min(he, h), max(ws, 0), min(we, w)
            if not count_include_pad:
                div = (h1 - h0) * (w1 - w0)
            y[:, :, i, j] = x[:, :, h0:h1, w0:w1].sum(axis=(2, 3)) / div
    return y


def act_fn(y, act):
    if act == 1:
        return np.maximum(y, 0.0)
    if act == 2:
        return np.minimum(np.maximum(y, 0.0), 6.0)
    return y


def eval_node(node, params, ins, residual, mode="exact", is_last=False):
    """Evaluate one fused operator on float64 NCHW inputs (already in storage precision).
    ins: list of input tensors (concatenated along C for CONV/POOL/FC, summed for ADD)."""
    k = node["kind"]
    if k == ADD:
        y = ins[0].copy()
        for t in ins[1:]:
            y = y + t
        y = act_fn(y, node["act"])
    else:
        x = ins[0] if len(ins) == 1 else np.concatenate(ins, axis=1)
        if k == CONV:
            w = _round(params["weight"].astype(np.float64), mode)
            y = conv2d(x, w, (node["sh"], node["sw"]), (node["ph"], node["pw"]), node["groups"])
            y = y * params["scale"].astype(np.float64)[None, :, None, None] + \
                params["shift"].astype(np.float64)[None, :, None, None]
            if residual is not None:
                y = y + residual
            y = act_fn(y, node["act"])
        elif k == BN:
            y = x * params["scale"].astype(np.float64)[None, :, None, None] + \
                params["shift"].astype(np.float64)[None, :, None, None]
            y = act_fn(y, node["act"])
        elif k == RELU:
            y = act_fn(x, node["act"])
        elif k == MAXPOOL:
            y = maxpool2d(x, node["kh"], node["sh"], node["ph"], bool(node["ceil_mode"]))
        elif k == AVGPOOL:
            y = avgpool2d(x, node["kh"], node["sh"], node["ph"], bool(node["ceil_mode"]),
                          bool(node["count_include_pad"]))
        elif k == GAP:
            y = x.mean(axis=(2, 3), keepdims=True)
        elif k == FC:
            w = _round(params["weight"].astype(np.float64), mode)
            flat = x.reshape(x.shape[0], -1)
            y = flat @ w.T * params["scale"].astype(np.float64)[None, :] + \
                params["shift"].astype(np.float64)[None, :]
            y = act_fn(y, node["act"]).reshape(x.shape[0], -1, 1, 1)
        else:
            raise ValueError(f"unknown op kind {k}")
    if is_last and mode == "bf16":
        return fp32_round(y)
    return _round(y, mode)


def forward(graph, x, mode="exact", return_all=False):
    """Whole-network forward pass of one tenant (op order = the node order, Eq.1)."""
    acts = []
    xin = _round(np.asarray(x, dtype=np.float64), mode)
    last = len(graph.nodes) - 1
    for j, nd in enumerate(graph.nodes):
        ins = [xin if i == -1 else acts[i] for i in nd["inputs"]]
        res = acts[nd["residual"]] if nd["residual"] >= 0 else None
        acts.append(eval_node(nd, graph.params[j], ins, res, mode, is_last=(j == last)))
    out = acts[-1].reshape(graph.batch, -1)
    return (out, acts) if return_all else out


def eval_op_teacher_forced(graph, j, acts_nchw, x, mode="bf16"):
    """Recompute op j from given input activations (e.g. the GPU's own, converted to NCHW
    float64) -- the per-op 'teacher-forced' check of SURVEY c.5."""
    nd = graph.nodes[j]
    xin = _round(np.asarray(x, dtype=np.float64), mode)
    ins = [xin if i == -1 else acts_nchw[i] for i in nd["inputs"]]
    res = acts_nchw[nd["residual"]] if nd["residual"] >= 0 else None
    return eval_node(nd, graph.params[j], ins, res, mode, is_last=(j == len(graph.nodes) - 1))
