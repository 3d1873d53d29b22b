"""N > 1 host logic on CPU with the gloo backend, world size 2 (-m "not gpu").

* the fixed row partition agrees across ranks and covers [0, n);
* the NCCL unique id moves from rank 0 to every rank over the process group;
* max/sum reductions used by bench.py's max-over-ranks timing;
* the decomposition the sharded solver implements — column partials of the g-pass per
  sub-split of each fixed row block, merged per block on the rank, the block partials gathered
  and merged in block order — reproduces the unsharded fp64 oracle, for one g-update and for a
  whole sharded Sinkhorn run (oracle arithmetic; the gloo all_gather stands in for
  ncclAllGather).
"""
import os
import socket

import numpy as np
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
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from oracle import oracle as O
        from paper_2206_07630_b200 import dist as skd
        from workloads import gen

        # 1. partition
        n = 70000
        plan = skd.shard_plan(n, world)
        mine = plan[rank]
        spans = [None] * world
        dist.all_gather_object(spans, mine)
        assert spans == plan
        assert plan[0][0] == 0 and plan[-1][0] + plan[-1][1] == n
        assert all(a[0] + a[1] == b[0] for a, b in zip(plan, plan[1:]))

        # 2. unique id broadcast (rank 0's bytes reach every rank)
        uid = bytes(np.random.default_rng(123).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None
        got = skd.exchange_unique_id(uid)
        assert got == bytes(np.random.default_rng(123).integers(0, 256, 128, dtype=np.uint8))

        # 3. reductions
        assert skd.max_over_ranks([float(rank + 1)])[0] == float(world)
        assert skd.sum_over_ranks([1.0, float(rank)]) == [float(world), float(sum(range(world)))]

        # 4. the sharded g-pass decomposition with a gathered exchange, fp64 oracle arithmetic
        p = gen.c4(n=2600, ns=16)
        x, y, eps = p.x, p.y, p.eps
        r0, nl = skd.shard_plan(len(x), world)[rank]
        rows = slice(r0, r0 + nl)

        # the solver's two-level merge tree: each fixed row block (SK_SHARD_BLOCKS of them) is cut
        # into sub-splits; a rank merges its blocks' sub-split partials per block (K6a), the block
        # partials are all-gathered (ncclAllGather in the library) and merged in block order
        B8 = 8
        bs = -(-len(x) // B8)
        bs = -(-bs // 256) * 256

        def lse_merge(parts):
            M = np.max([p_[0] for p_ in parts], axis=0)
            S = np.zeros_like(M)
            for Mp, Sp in parts:
                S = S + Sp * np.exp(Mp - M)
            return M, S

        def sharded_g(f, split_q=3):
            mine = []
            for b in range(B8):
                lo, hi = max(b * bs, r0), min((b + 1) * bs, r0 + nl)
                if lo >= hi:
                    continue
                cuts = [lo + (hi - lo) * u // split_q for u in range(split_q + 1)]
                subs = [O.column_partials(x[c0:c1], y, f[c0:c1], eps) for c0, c1 in zip(cuts, cuts[1:]) if c1 > c0]
                mine.append((b, lse_merge(subs)))
            gathered = [None] * world
            dist.all_gather_object(gathered, mine)
            blocks = sorted((b, ms) for part in gathered for b, ms in part)
            return O.merge_partials([ms for _, ms in blocks], np.full(len(y), 1 / len(y)), eps)

        f = np.random.default_rng(7).standard_normal(len(x)) * 0.01
        g_sh = sharded_g(f)
        g_ref = O.g_update(x, y, f, eps)
        assert np.abs(g_sh - g_ref).max() < 1e-12

        # whole sharded Sinkhorn (row pass local, column pass via partials) = unsharded oracle
        f = np.zeros(len(x))
        for _ in range(6):
            g = sharded_g(f)
            f_loc = O.f_update(x[rows], y, g, eps, a=np.full(nl, 1 / len(x)))
            parts = [None] * world
            dist.all_gather_object(parts, f_loc)
            f = np.concatenate(parts)
        ref = O.sinkhorn(x, y, eps, tol=0, max_iter=6)
        assert np.abs(f - ref.f).max() < 1e-10 and np.abs(g - ref.g).max() < 1e-10
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=280) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
