"""Multi-GPU plumbing: streams are sharded across ranks (one process per GPU).

The temporal dependency of the path is intra-stream (pipeline.py:276-277), so
independent video streams partition with no per-frame exchange.  The only
collective is the end-of-run gather of per-stream, per-frame statistics
(SURVEY.md 8(e)): counts, coverage and device times, a few KB per stream,
gathered with one all_gather over NCCL (gloo on CPU tests).
"""

from __future__ import annotations

import numpy as np

STAT_FIELDS = ("frame", "n_detected", "n_propagated", "n_total", "n_dropped", "coverage", "ms")


def shard(n_streams: int, rank: int, world: int) -> list[int]:
    """Contiguous stream ranges: rank r gets [r*S/G, (r+1)*S/G)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = n_streams * rank // world
    hi = n_streams * (rank + 1) // world
    return list(range(lo, hi))


def pack_stats(stream_ids, reports, ms_per_frame=None) -> np.ndarray:
    """[n_local_streams, n_frames, 1 + len(STAT_FIELDS)] float64 (col 0 = stream id)."""
    n_f = max((len(r) for r in reports), default=0)
    out = np.zeros((len(stream_ids), n_f, 1 + len(STAT_FIELDS)), np.float64)
    for i, (sid, reps) in enumerate(zip(stream_ids, reports)):
        for n, r in enumerate(reps):
            ms = 0.0 if ms_per_frame is None else float(ms_per_frame[n])
            out[i, n] = (sid, r.frame, r.n_detected, r.n_propagated, r.n_total, r.n_dropped, r.coverage, ms)
    return out


def gather_stats(local: np.ndarray, n_streams_total: int, device=None) -> np.ndarray | None:
    """All-gather per-stream stats; returns [S_total, n_frames, F] ordered by stream id on every rank."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        full = local
    else:
        world = dist.get_world_size()
        # pad to the largest shard so all_gather sees equal shapes
        max_local = -(-n_streams_total // world)
        pad = np.zeros((max_local,) + local.shape[1:], np.float64)
        pad[:, :, 0] = -1.0
        pad[: local.shape[0]] = local
        t = torch.from_numpy(pad)
        if device is not None:
            t = t.to(device)
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        full = np.concatenate([o.cpu().numpy() for o in outs], 0)
        full = full[full[:, 0, 0] >= 0] if full.shape[1] else full
    order = np.argsort(full[:, 0, 0], kind="stable") if full.shape[1] else np.arange(full.shape[0])
    return full[order]


HIST_FIELDS = ("n_detected", "n_propagated", "n_total", "n_dropped", "coverage", "frame", "n_survivors",
               "n_candidates")


def gather_stream_history(hist, stream_ids, step_ms, n_streams_total: int):
    """End-of-run statistics gather on the device (the path's one collective).

    hist: this rank's [S_local, F, 8] float64 CUDA tensor filled by
    FeatureEngine.set_history; step_ms: [F] per-frame device step times of this
    rank.  Returns [n_streams_total, F, 10] (stream id, the 8 HIST_FIELDS, ms)
    ordered by stream id, on every rank.  One all_gather over the process
    group's backend (NCCL over NVLink on the GPU box, gloo in CPU tests)."""
    import torch
    import torch.distributed as dist

    S, F = hist.shape[0], hist.shape[1]
    ids = torch.as_tensor(list(stream_ids), dtype=torch.float64, device=hist.device)
    ms = torch.as_tensor(step_ms, dtype=torch.float64, device=hist.device).reshape(1, F, 1).expand(S, F, 1)
    local = torch.cat([ids.view(S, 1, 1).expand(S, F, 1), hist, ms], 2)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        full = local
        if dist.is_available() and dist.is_initialized():
            outs = [torch.empty_like(local)]
            dist.all_gather(outs, local)
            full = outs[0]
    else:
        world = dist.get_world_size()
        max_local = -(-n_streams_total // world)
        pad = torch.full((max_local, F, 10), -1.0, dtype=torch.float64, device=hist.device)
        pad[:S] = local
        outs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad)
        full = torch.cat(outs, 0)
        full = full[full[:, 0, 0] >= 0] if F else full
    order = torch.argsort(full[:, 0, 0], stable=True) if F else torch.arange(full.shape[0], device=full.device)
    return full[order]
