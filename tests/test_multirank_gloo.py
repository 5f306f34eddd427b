"""World-size-2 CPU (gloo) tests of the replica path's host-side logic.

test_two_replicas_gloo: the oracle's view — agent partition a -> rank a mod N, global request
ids local_seq * N + rank, one all-gather of per-rank top-K candidates per round whose merge
equals the top-K of the union (AMB-22 / pin P13), and max-over-ranks timing.

test_product_replica_orchestration_gloo: the product's host code bench.py --gpus N runs
(paper_2412_18695_b200/replicas.py): partition, id rule, the ncclUniqueId broadcast, the
lockstep drain that keeps every rank's rt_step count equal (each rt_step is a collective when
world > 1: here every step performs an all-gather, so a count mismatch would hang), and the
whole-job throughput reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.engine import OracleEngine
        from oracle.merge import merge_rank_topk, global_topk
        from synth import make_vocab, engine_params, compose_workload
        v = make_vocab(512)
        p = engine_params("paper-4090", max_batch=4, max_tasks=256, max_ctx=256, n_pages=128)
        e = OracleEngine(p, v.tok_skill, v.tok_exec_min_us, v.eos_id, v.vocab, rank=rank, world=world)
        reqs = compose_workload(16, 4.0, 8, range(1, 9), 4.0, 3, v, prompt_len_range=(10, 40))
        mine = [r for r in reqs if r.agent_id % world == rank]
        ids = [e.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, 0,
                        script=r.plan) for r in mine]
        assert all(i % world == rank for i in ids)
        all_ids = [None] * world
        dist.all_gather_object(all_ids, ids)
        flat = [i for lst in all_ids for i in lst]
        assert len(flat) == len(set(flat))            # global ids unique across replicas
        ok_rounds = 0
        for _ in range(40):
            e.step()
            waiting = [r for r in e.reqs.values() if r.state == 1]
            for r in waiting:
                e._key(r, e.t)
            cand = [(getattr(r, "pri", 0.0), r.arrival, r.id, rank) for r in waiting]
            local = global_topk(cand, 16)
            gathered = [None] * world
            dist.all_gather_object(gathered, (local, cand))
            merged = merge_rank_topk([g[0] for g in gathered], 16)
            union = [c for g in gathered for c in g[1]]
            assert merged == global_topk(union, 16)
            ok_rounds += 1
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == float(world)
        q.put((rank, ok_rounds))
    finally:
        dist.destroy_process_group()


def test_two_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, 40), (1, 40)]


def _worker_product(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_18695_b200 import replicas as R
        from oracle.engine import OracleEngine
        from synth import make_vocab, engine_params, compose_workload
        n_agents = 13
        mine = R.partition(n_agents, rank, world)
        every = [None] * world
        dist.all_gather_object(every, mine)
        assert sorted(a for lst in every for a in lst) == list(range(n_agents))   # each agent once
        assert all(a % world == rank for a in mine)
        uid = R.bootstrap_nccl_id(dist, rank, lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        # the engine's id rule vs the product helper (the oracle follows the same reading)
        v = make_vocab(512)
        p = engine_params("paper-4090", max_batch=4, max_tasks=256, max_ctx=256, n_pages=128)
        e = OracleEngine(p, v.tok_skill, v.tok_exec_min_us, v.eos_id, v.vocab, rank=rank, world=world)
        # rank-dependent load: rank 1 gets 3x the requests, so it drains much later
        reqs = compose_workload(n_agents, 4.0, 8, range(1, 9), 2.0 + 4.0 * rank, 3 + rank, v,
                                prompt_len_range=(10, 40))
        reqs = [r for r in reqs if r.agent_id % world == rank]
        for i, r in enumerate(reqs):
            rid = e.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, 0,
                           script=r.plan)
            assert rid == R.global_request_id(i, rank, world) and R.owner_rank(rid, world) == rank
        idle_at = [None]

        def step():   # one round + the per-round collective (the engine's candidate allgather)
            info = e.step()
            g = [None] * world
            dist.all_gather_object(g, (rank, info["n_running"]))
            if idle_at[0] is None and info["n_running"] == 0 and info["n_waiting"] == 0:
                idle_at[0] = n_calls[0]
            n_calls[0] += 1
            return info

        n_calls = [0]
        n = R.lockstep_until_idle(step, dist)
        counts = [None] * world
        dist.all_gather_object(counts, (n, idle_at[0]))
        assert counts[0][0] == counts[1][0]                     # same number of rounds on every rank
        assert counts[0][1] is not None and counts[0][1] < counts[1][1]   # rank 0 idled first
        units, ms = R.reduce_throughput(dist, 100 * (rank + 1), 2.0 + rank)
        assert (units, ms) == (300.0, 3.0)
        q.put((rank, n))
    finally:
        dist.destroy_process_group()


def test_product_replica_orchestration_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_product, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res[0][1] == res[1][1] > 0
