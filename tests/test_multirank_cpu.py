"""World-size-2 CPU (gloo) test of the multi-GPU host protocol:
every rank splits the Morton-ordered leaves with the library's host partition
(ddm_split_costs), owns the rows of its leaf range, exchanges them with a
padded all-gather (the layout ncclAllGather uses in allgather_sorted) and
all-reduces per-rank partial dot products (the GMRES CGS2 reduction).  The
reassembled vector and the dots must equal the single-rank values exactly."""
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
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1812_05087_b200 as D
        rng = np.random.default_rng(42)            # identical on every rank
        nleaves = 300
        counts = rng.integers(1, 65, nleaves)       # elements per leaf (Morton order)
        nsrc = rng.integers(30, 3000, nleaves)
        cost = counts * (nsrc + 20)
        pre = np.concatenate([[0], np.cumsum(cost)[:-1]]).astype(np.int64)
        split = D.split_costs(pre, int(cost.sum()), world)
        el_start = np.concatenate([[0], np.cumsum(counts)])
        n = int(el_start[-1])
        ncomp = 3
        full = rng.normal(size=(n, ncomp))           # the vector every rank needs
        lo, hi = el_start[split[rank]], el_start[split[rank + 1]]
        rows = [el_start[split[r + 1]] - el_start[split[r]] for r in range(world)]
        maxrows = max(rows)
        send = torch.zeros(maxrows * ncomp, dtype=torch.float64)
        send[:(hi - lo) * ncomp] = torch.from_numpy(full[lo:hi].reshape(-1))
        recv = [torch.zeros_like(send) for _ in range(world)]
        dist.all_gather(recv, send)
        out = np.zeros((n, ncomp))
        for r in range(world):
            a, b = el_start[split[r]], el_start[split[r + 1]]
            out[a:b] = recv[r].numpy()[:(b - a) * ncomp].reshape(-1, ncomp)
        # partial dots of k+1 basis vectors with w over the owned rows
        V = rng.normal(size=(5, n * ncomp))
        w = rng.normal(size=n * ncomp)
        part = torch.from_numpy(V[:, lo * ncomp:hi * ncomp] @ w[lo * ncomp:hi * ncomp])
        dist.all_reduce(part)
        q.put((rank, split.tolist(), bool(np.array_equal(out, full)),
               float(np.abs(part.numpy() - V @ w).max() / np.abs(V @ w).max())))
    finally:
        dist.destroy_process_group()


def test_two_rank_partition_allgather_allreduce():
    pytest.importorskip("paper_1812_05087_b200")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    splits = {tuple(r[1]) for r in res}
    assert len(splits) == 1                       # every rank computes the same split
    sp = list(splits)[0]
    assert sp[0] == 0 and sp[-1] == 300 and 0 < sp[1] < 300
    assert all(r[2] for r in res)                 # exact reassembly
    assert all(r[3] < 1e-14 for r in res)         # all-reduced dots = global dots


def _shard_worker(rank, world, port, q):
    """The sharded upward pass's communication pattern with an
    exactly combinable stand-in for the multipole (per-cell sums of a seeded
    per-element value, which M2M-like child -> parent sums reproduce exactly):
    rank r sums its complete cells (ddm_shard_owner) from its own elements,
    the ranks all-gather the packed values (padded, as allgather_mpole), and
    every rank completes the straddling cells from their children, deepest
    level first."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1812_05087_b200 as D
        from oracle import tree as OT
        from synth import make_config
        g = make_config(2)
        t = OT.build_tree(g.xc, g.yc, 32)
        nc = t.n_cells
        leaves = np.nonzero(t.is_leaf)[0]
        leaves = leaves[np.argsort(t.start[leaves], kind="stable")]   # Morton order
        cost = t.count[leaves].astype(np.int64) * 7 + 3
        pre = np.concatenate([[0], np.cumsum(cost)[:-1]]).astype(np.int64)
        split = D.split_costs(pre, int(cost.sum()), world)
        lo = np.array([t.start[leaves[s]] if s < leaves.size else g.n for s in split[:-1]] + [g.n],
                      dtype=np.int64)
        owner = D.shard_owner(t.start, t.count, lo)
        val = np.random.default_rng(7).normal(size=g.n)       # per sorted element
        cs = np.concatenate([[0.0], np.cumsum(val)])
        exact = cs[t.start + t.count] - cs[t.start]            # reference cell sums
        mine = np.nonzero(owner == rank)[0]
        # complete cells from own elements only (leaves directly, parents from children)
        m = np.full(nc, np.nan)
        for c in sorted(mine, key=lambda c: -t.level[c]):
            if t.is_leaf[c]:
                a, b = t.start[c], t.start[c] + t.count[c]
                assert lo[rank] <= a and b <= lo[rank + 1]
                m[c] = val[a:b].sum()
            else:
                kids = range(t.first_child[c], t.first_child[c] + t.n_child[c])
                m[c] = sum(m[k] for k in kids)
        counts = [int((owner == r).sum()) for r in range(world)]
        pad = max(counts)
        send = torch.zeros(pad, dtype=torch.float64)
        send[:len(mine)] = torch.from_numpy(m[mine])
        recv = [torch.zeros_like(send) for _ in range(world)]
        dist.all_gather(recv, send)
        for r in range(world):
            cells = np.nonzero(owner == r)[0]
            m[cells] = recv[r].numpy()[:cells.size]
        strad = np.nonzero(owner < 0)[0]
        for c in sorted(strad, key=lambda c: -t.level[c]):
            assert not t.is_leaf[c]                                # leaves never straddle
            kids = range(t.first_child[c], t.first_child[c] + t.n_child[c])
            m[c] = sum(m[k] for k in kids)
        crosses = np.array([any(t.start[c] < x < t.start[c] + t.count[c] for x in lo[1:-1])
                            for c in range(nc)])
        q.put((rank, bool(np.allclose(m, exact, rtol=1e-12, atol=1e-12)),
               bool(np.array_equal(owner < 0, crosses)), counts, int(strad.size)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_upward_pass_pattern(world):
    pytest.importorskip("paper_1812_05087_b200")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] for r in res)          # every cell's value right on every rank
    assert all(r[2] for r in res)          # straddling = ranges crossing a rank boundary
    assert len({tuple(r[3]) for r in res}) == 1
    assert all(0 < r[4] < 40 for r in res)   # a few straddling cells (ancestors of boundaries)
