"""One-process-per-GPU plumbing for the pipeline (launched by torchrun, one rank = one stage).

The data path is the engine's own transport: CUDA-IPC peer-memory rings pushed by the copy
engine over NVLink (gp_link_ipc, the default) or NCCL send/recv (gp_link_nccl: one 2-rank
communicator per stage boundary). torch.distributed (gloo) is only the control plane:
blob / unique-id exchange, the epoch barrier and max-over-ranks timing.

`message_schedule` is the host-side statement of the transport order the engine follows in
gp_run_epoch (engines_impl.hpp:784-870): it is what guarantees that every ncclSend of
stage s meets the matching ncclRecv of stage s+1 in the same order (no deadlock), and it
yields the per-stage ledger (4 bytes per value, fabric.hpp:59).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple


def stage_ranges(num_layers: int, num_stages: int) -> List[Tuple[int, int]]:
    """make_stage_assignment (engines.cpp:8-21): first L mod S stages get one more layer."""
    if num_stages == 0 or num_stages > num_layers:
        raise ValueError("stage assignment needs 1 <= stages <= layers")
    q, r = divmod(num_layers, num_stages)
    out, at = [], 0
    for s in range(num_stages):
        take = q + (1 if s < r else 0)
        out.append((at, at + take))
        at += take
    return out


def message_schedule(order: Sequence[int], stage: int, num_stages: int, sync: bool = False):
    """Ordered transport operations of one stage for one epoch.

    Returns a list of (op, chunk) with op in {"recv_fwd", "send_fwd", "recv_bwd", "send_bwd"}.
    Stale mode interleaves per chunk (forward in `order`, backward in reverse order); sync
    mode receives all chunks, computes, then sends all (engines_impl.hpp:800-814, :850-870).
    """
    first, last = stage == 0, stage == num_stages - 1
    ops = []
    K = len(order)
    if not sync:
        for k in order:
            if not first:
                ops.append(("recv_fwd", k))
            if not last:
                ops.append(("send_fwd", k))
        for k in reversed(order):
            if not last:
                ops.append(("recv_bwd", k))
            if not first:
                ops.append(("send_bwd", k))
    else:
        if not first:
            ops += [("recv_fwd", k) for k in order]
        if not last:
            ops += [("send_fwd", k) for k in order]
        if not last:
            ops += [("recv_bwd", order[kk]) for kk in range(K - 1, -1, -1)]
        if not first:
            ops += [("send_bwd", order[kk]) for kk in range(K - 1, -1, -1)]
    return ops


def stage_ledger(order, stage, num_stages, chunk_rows, out_width, in_width, h0_width=0, sync=False):
    """Bytes this stage sends per MsgTag: (ForwardEmb, BackwardGrad), 4 B/value."""
    fwd = bwd = 0
    for op, k in message_schedule(order, stage, num_stages, sync):
        if op == "send_fwd":
            fwd += chunk_rows[k] * (out_width + h0_width) * 4
        elif op == "send_bwd":
            bwd += chunk_rows[k] * (in_width + h0_width) * 4
    return fwd, bwd


def exchange_unique_ids(dist, rank: int, world: int, make_id: Callable[[], bytes]) -> List[bytes]:
    """Rank 0 creates one NCCL unique id per stage boundary and broadcasts them."""
    ids = [make_id() for _ in range(world - 1)] if rank == 0 else [None] * (world - 1)
    if world > 1:
        dist.broadcast_object_list(ids, src=0)
    return ids


def boundary_ids(ids: Sequence[bytes], rank: int, world: int):
    """(up_id, down_id) of this stage: boundary b joins stage b (rank 0 of the comm) and b+1."""
    up = ids[rank - 1] if rank > 0 else None
    down = ids[rank] if rank < world - 1 else None
    return up, down


def exchange_ipc_blobs(dist, rank: int, world: int, mine) -> Tuple[Optional[bytes], Optional[bytes]]:
    """All-gather every stage's (up, down) IPC blobs (StageEngine.ipc_export) and
    return this stage's (up_peer, down_peer) for StageEngine.link_ipc: the `down`
    blob of stage s-1 and the `up` blob of stage s+1."""
    allb = [None] * world
    if world > 1:
        dist.all_gather_object(allb, tuple(mine))
    else:
        allb[0] = tuple(mine)
    up = allb[rank - 1][1] if rank > 0 else None
    down = allb[rank + 1][0] if rank < world - 1 else None
    return up, down


def exchange_group_blobs(dist, stage: int, grank: int, group_size: int, blob: bytes) -> List[Optional[bytes]]:
    """All-gather (stage, group rank, blob) and return the blobs of this stage's group
    in group-rank order (for StageEngine.link_group_ipc)."""
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    allb = [None] * world
    if world > 1:
        dist.all_gather_object(allb, (stage, grank, blob))
    else:
        allb[0] = (stage, grank, blob)
    out: List[Optional[bytes]] = [None] * group_size
    for st, r, b in allb:
        if st == stage:
            out[r] = b
    return out


def max_over_ranks(dist, x: float) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
