"""Multi-GPU sharding of one VeLoPIR query (R15).

Records split into contiguous power-of-two shards [r*M/G, (r+1)*M/G), one per rank (process per GPU).  Per
query: the query ciphertexts are broadcast from rank 0, every rank evaluates its shard down to the shard's
aggregation-tree root (l_S ciphertexts), the roots are gathered to rank 0 (a gather, not an all-gather: only rank 0 combines), and rank 0 runs the top log2 G tree levels
(vlp_program_create_combine).  Because the tree pairs (i, i+k) never cross a power-of-two shard boundary
for k < M/G, the result is byte-identical to the single-GPU evaluation.  torch.distributed is plumbing only
(NCCL on GPUs; gloo in the CPU tests); the evaluation callbacks are the library's kernels.
"""
from __future__ import annotations


def shard_range(M: int, world: int, rank: int):
    """(first, count) of rank's contiguous shard; M/world must be a power of two (R15)."""
    if world == 1:
        return 0, M  # a single shard needs no tree boundary alignment
    if world < 1 or M % world:
        raise ValueError("M must be divisible by the number of ranks")
    count = M // world
    if count & (count - 1):
        raise ValueError("shards must hold a power-of-two number of records")
    if world & (world - 1):
        raise ValueError("the number of ranks must be a power of two")
    return rank * count, count


def sharded_step(q, eval_shard, combine, world: int, rank: int, gathered=None):
    """One query: broadcast q (rank 0's), eval_shard(q) -> shard root tensor [l_S, 632], gather all roots to
    rank 0, which returns combine(roots [G*l_S, 632]); other ranks return None.  Single rank: eval_shard(q)."""
    if world == 1:
        return eval_shard(q)
    import torch
    import torch.distributed as dist
    staged = q.is_cuda and dist.get_backend() != "nccl"  # gloo: collectives on host copies of device tensors
    if staged:
        qh = q.cpu()
        dist.broadcast(qh, src=0)
        q.copy_(qh)
    else:
        dist.broadcast(q, src=0)
    part = eval_shard(q)
    if gathered is None:  # concatenated along dim 0: [G * l_S, 632] (rank order = shard order)
        gathered = torch.empty((world * part.shape[0],) + tuple(part.shape[1:]), dtype=part.dtype, device=part.device)
    send = part.contiguous().cpu() if staged else part.contiguous()
    if rank == 0:
        if staged:
            host = torch.empty(gathered.shape, dtype=gathered.dtype)
            dist.gather(send, gather_list=list(host.chunk(world, dim=0)), dst=0)
            gathered.copy_(host)
        else:
            dist.gather(send, gather_list=list(gathered.chunk(world, dim=0)), dst=0)
        return combine(gathered)
    dist.gather(send, dst=0)
    return None
