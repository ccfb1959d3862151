"""Multi-rank (world_size 2 and 3) CPU test of the row-partitioned apply protocol over gloo.

Each rank owns a contiguous row slab, builds its halo plan with the library's host-only
`bk_plan_halo` (the same planner bk_csr_create runs), exchanges the requested ghost ids with
its owners (all_to_all of counts + ids, as comm.cpp does with NCCL), sends the requested rows
and receives its ghost rows, then applies its renumbered slab with the CPU oracle.  The union
over ranks must equal the global apply BITWISE (integer-exact inputs), and the Gram allreduce
must give every rank identical bits.
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


def _worker(rank, world, port, cfg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2504_02117_b200 as bk
        import synth
        nx, ny, nz, k = cfg
        A = synth.richards3d(nx, ny, nz, integer=True)
        N = A.n_rows
        X = synth.multivector(N, k, 3, integer=True).numpy()
        plane = nx * ny
        rb = [(nz * r // world) * plane for r in range(world + 1)]     # z-slabs
        r0, r1 = rb[rank], rb[rank + 1]
        slab = A.rows(r0, r1)
        plan = bk.plan_halo(world, rank, rb, slab.row_ptr.numpy(), slab.col.numpy())
        gid, gown = plan["ghost_ids"], plan["ghost_owner"]
        # 1. request exchange: counts then ids (all_to_all via send/recv pairs)
        need = [gid[gown == q] for q in range(world)]
        cnt = torch.tensor([len(x) for x in need], dtype=torch.int64)
        allcnt = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allcnt, cnt)
        give_cnt = [int(allcnt[q][rank]) for q in range(world)]
        reqs, gives = [], {}
        for q in range(world):
            if q == rank:
                continue
            if len(need[q]):
                reqs.append(dist.isend(torch.from_numpy(need[q].astype(np.int64)), q))
            if give_cnt[q]:
                buf = torch.zeros(give_cnt[q], dtype=torch.int64)
                reqs.append(dist.irecv(buf, q))
                gives[q] = buf
        for r_ in reqs:
            r_.wait()
        # 2. ghost exchange: send requested rows of my slab, receive my ghosts (owner order)
        Xloc = X[r0:r1]
        reqs, recv = [], {}
        for q in range(world):
            if q == rank:
                continue
            if q in gives:
                rows = gives[q].numpy() - r0
                assert rows.min() >= 0 and rows.max() < r1 - r0
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(Xloc[rows])), q))
            if len(need[q]):
                buf = torch.zeros(len(need[q]), k, dtype=torch.float64)
                reqs.append(dist.irecv(buf, q))
                recv[q] = buf
        for r_ in reqs:
            r_.wait()
        ghosts = np.concatenate([recv[q].numpy() for q in range(world) if q in recv], axis=0) \
            if recv else np.zeros((0, k))
        assert np.array_equal(ghosts, X[gid])          # ghost buffer ordered like ghost_ids
        Xext = np.concatenate([Xloc, ghosts], axis=0)
        local = synth.Csr(slab.n_rows, Xext.shape[0], slab.row_ptr, torch.from_numpy(plan["col_local"]), slab.val)
        Yloc = oracle.spmm(local, Xext)
        ok_apply = bool(np.array_equal(Yloc, oracle.spmm(A, X)[r0:r1]))
        # 3. Gram allreduce: identical bits everywhere, equal to the global Gram (integers: exact)
        G = torch.from_numpy(oracle.gram(Yloc, Xloc))
        dist.all_reduce(G)
        Gall = [torch.zeros_like(G) for _ in range(world)]
        dist.all_gather(Gall, G)
        same = all(torch.equal(Gall[0], g) for g in Gall)
        exact = bool(np.array_equal(G.numpy(), oracle.gram(oracle.spmm(A, X), X)))
        out_q.put((rank, ok_apply, same, exact, len(gid), int(plan["is_boundary"].sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [(2, (6, 5, 8, 4)), (3, (5, 4, 9, 3))])
def test_row_partition_protocol_over_gloo(world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nx, ny, nz, k = cfg
    for rank, ok_apply, same, exact, n_ghost, n_bnd in sorted(res):
        assert ok_apply and same and exact
        nb = (rank > 0) + (rank < world - 1)
        assert n_ghost == nb * nx * ny and n_bnd == nb * nx * ny      # two ghost planes at most
