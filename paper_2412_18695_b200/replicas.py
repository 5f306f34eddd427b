"""Host-side orchestration of agent-partitioned replicas (one process per GPU).

BASELINE.json: "Agents are partitioned across the GPUs of one 8xB200 box as independent
replicas, with one NCCL allgather over NVLink per scheduling round so the global utility
ordering stays exact" (KV never leaves its GPU).  The engine
(rt_step) issues that allgather on EVERY call when world > 1, so every rank must call rt_step
the same number of times; these helpers keep the ranks in lockstep.  They need only a
torch.distributed process group (nccl on the GPU box, gloo in the CPU tests) and never touch
the device data path.
"""


def partition(n_agents, rank, world):
    """Agents of this replica: a -> rank a mod world."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(range(rank, n_agents, world))


def global_request_id(local_seq, rank, world):
    """The id rt_submit_request assigns (include/rt.h: local_seq * world + rank): unique
    across replicas, and the merge's final tie-break (AMB-10)."""
    return local_seq * world + rank


def owner_rank(request_id, world):
    return request_id % world


def bootstrap_nccl_id(dist, rank, make_id):
    """Rank 0 makes the 128-byte ncclUniqueId (rt.nccl_unique_id) and broadcasts it."""
    obj = [make_id() if rank == 0 else None]
    if dist is not None:
        dist.broadcast_object_list(obj, src=0)
    return obj[0]


def any_busy(dist, busy):
    """True while any rank still has work (one small all-reduce)."""
    if dist is None:
        return bool(busy)
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([1 if busy else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return bool(t.item())


def lockstep_until_idle(step, dist, max_rounds=100000):
    """Call step() (one rt_step; returns the round info dict) until NO rank is running or
    waiting anything.  Every rank makes the same number of calls, so the per-round
    allgathers pair up across ranks (a rank that drained early keeps stepping idle rounds).
    Returns the number of calls."""
    n = 0
    while n < max_rounds:
        info = step()
        n += 1
        if not any_busy(dist, info["n_running"] > 0 or info["n_waiting"] > 0):
            break
    return n


def reduce_throughput(dist, units, ms):
    """Whole-job throughput: units summed over ranks / the slowest rank's device time
    (max over ranks, never wall clock).  Returns (total units, max ms)."""
    if dist is None:
        return float(units), float(ms)
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    u = torch.tensor([float(units)], dtype=torch.float64, device=dev)
    dist.all_reduce(u)
    return float(u.item()), float(t.item())
