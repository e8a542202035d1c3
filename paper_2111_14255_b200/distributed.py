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


def profile_distributed(profile_fn, cands, rank: int, world: int, device=None, group=None):
    """profile_fn(list of candidates) -> (lat, status) on this rank's GPU (e.g.
    Context.profile_batch_pointers); returns the gathered full vectors on every rank."""
    mine = [cands[i] for i in shard_indices(len(cands), rank, world)]
    lat, st = profile_fn(mine) if mine else (np.zeros(0, np.float32), np.zeros(0, np.int32))
    return gather_results(lat, st, len(cands), rank, world, device, group)
