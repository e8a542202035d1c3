"""Candidate-sharded schedule profiling across GPUs (Alg.1 L7-L9).

Every rank holds the same seeded candidate list, profiles candidates c = rank, rank+G, ... on its
own GPU through mt_profile_batch (no communication while timing), then one all_gather (NCCL over
NVLink on GPUs, gloo in the CPU tests) assembles the full latency/status vectors on every rank.
Host plumbing only: which candidate runs where and how results are reassembled.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist


def shard_indices(n: int, rank: int, world: int):
    """candidates owned by `rank`: c = rank, rank + world, ..."""
    return list(range(rank, n, world))


def gather_results(local_lat, local_st, n: int, rank: int, world: int, device=None, group=None):
    """All-gather per-rank results (padded to ceil(n/world)) and un-permute them into candidate
    order.  Returns (lat[n] float32, status[n] int32) identical on every rank."""
    n_loc = math.ceil(n / world) if n else 0
    dev = device if device is not None else torch.device("cpu")
    buf = torch.full((n_loc, 2), float("nan"), dtype=torch.float64, device=dev)
    k = len(local_lat)
    if k:
        buf[:k, 0] = torch.as_tensor(np.asarray(local_lat, np.float64), device=dev)
        buf[:k, 1] = torch.as_tensor(np.asarray(local_st, np.float64), device=dev)
    if world > 1:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
    else:
        parts = [buf]
    lat = np.full(n, np.nan, np.float32)
    st = np.full(n, -1, np.int32)
    for r, p in enumerate(parts):
        p = p.cpu().numpy()
        for j, c in enumerate(shard_indices(n, r, world)):
            lat[c] = p[j, 0]
            st[c] = int(p[j, 1])
    return lat, st


def rank_scales(ref_lat, ref_st, rank: int, world: int, device=None, group=None):
    """Per-GPU normalisation (SURVEY §7 hard part 5, §8(e)): every rank times the same reference
    schedules; rank r's scale = mean over the feasible references k of (mean over ranks of
    lat_k) / lat_k(r).  Multiplying a rank's latencies by its scale puts all ranks on the clock
    of the average GPU.  Returns (scales[world], refs[world][n_ref])."""
    n_ref = len(ref_lat)
    dev = device if device is not None else torch.device("cpu")
    buf = torch.tensor([[float(v) if int(s) == 0 else float("nan") for v, s in zip(ref_lat, ref_st)]],
                       dtype=torch.float64, device=dev).reshape(1, n_ref)
    if world > 1:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        refs = torch.cat(parts).cpu().numpy()
    else:
        refs = buf.cpu().numpy()
    ok = np.all(np.isfinite(refs), axis=0) & np.all(refs > 0, axis=0)
    if not ok.any():
        return np.ones(world), refs
    mean_k = refs[:, ok].mean(axis=0)
    scales = (mean_k[None, :] / refs[:, ok]).mean(axis=1)
    return scales, refs


def profile_distributed(profile_fn, cands, rank: int, world: int, device=None, group=None,
                        ref=None, info=None):
    """profile_fn(list of candidates) -> (lat, status) on this rank's GPU (e.g.
    Context.profile_batch_pointers); returns the gathered full vectors on every rank.
    ref: indices of reference candidates (e.g. (0, 1), the two extreme schedules) that every rank
    also profiles; each rank's latencies are then scaled to the average GPU (rank_scales) before
    the gather.  info (dict, optional) receives the scales and the per-rank reference latencies."""
    mine = [cands[i] for i in shard_indices(len(cands), rank, world)]
    extra = [cands[i] for i in ref] if ref else []
    todo = mine + extra
    lat_all, st_all = profile_fn(todo) if todo else (np.zeros(0, np.float32), np.zeros(0, np.int32))
    lat, st = np.asarray(lat_all[:len(mine)], np.float64), np.asarray(st_all[:len(mine)])
    if ref:
        scales, refs = rank_scales(lat_all[len(mine):], st_all[len(mine):], rank, world, device, group)
        lat = lat * scales[rank]
        if info is not None:
            info["scales"] = [float(v) for v in scales]
            info["ref_lat"] = refs.tolist()
    return gather_results(lat, st, len(cands), rank, world, device, group)
