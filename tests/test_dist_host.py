"""CPU: the distributed path's host logic -- partition,
ghost lists, local column renumbering, interior/boundary split, and the
send lists learned by the all-to-all -- in liblbk's C++ (no device needed),
checked bit-exact against the App. B restatement (oracle/port.cpp) and by
brute force; then the whole halo protocol is run across world_size-2 gloo
processes and the resulting distributed SpMV (numpy over the maps) is
compared with the global oracle SpMV."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2011_08879_b200 import dist as D


def _maps(O, A, P):
    out = []
    for rank in range(P):
        rp, cols, vals = D.local_rows(A.row_ptr, A.cols, A.vals, P, rank)
        out.append((D.DistMap(A.nrows, P, rank, rp, cols), rp, cols, vals))
    return out


@pytest.mark.parametrize("kind,m,P", [("7pt", 8, 1), ("7pt", 8, 2), ("7pt", 10, 3),
                                      ("27pt", 9, 4), ("5pt", 33, 5), ("7pt", 6, 8)])
def test_maps_bitexact_vs_restatement(O, kind, m, P):
    A = O.stencil(kind, m)
    for rank, (mp_, rp, cols, vals) in enumerate(_maps(O, A, P)):
        b, e = O.part_range(A.nrows, P, rank)
        assert (mp_.info.begin, mp_.info.end) == (b, e) == D.part_range(A.nrows, P, rank)
        g, off = mp_.ghosts()
        gref = O.part_ghosts(A, P, rank)
        assert np.array_equal(g, gref)
        assert np.array_equal(mp_.local_cols(), O.part_local_cols(A, P, rank, gref))
        for q in range(P):  # ghost runs by owner
            qb, qe = O.part_range(A.nrows, P, q)
            assert np.all((g[off[q]:off[q + 1]] >= qb) & (g[off[q]:off[q + 1]] < qe))
        inter, bnd = mp_.rows()
        has_ghost = np.array([np.any((cols[rp[r]:rp[r + 1]] < b) | (cols[rp[r]:rp[r + 1]] >= e))
                              for r in range(e - b)], bool)
        assert np.array_equal(bnd, np.nonzero(has_ghost)[0])
        assert np.array_equal(inter, np.nonzero(~has_ghost)[0])


def test_send_lists_and_halo_spmv_in_process(O):
    A = O.stencil("27pt", 10)
    P = 3
    maps = _maps(O, A, P)
    D.exchange_requests_local([m for m, *_ in maps])
    x = O.seeded_values(A.ncols, 11)
    yref = O.spmv_csr(A, x)
    for rank, (m, rp, cols, vals) in enumerate(maps):
        off, idx = m.sends()
        b, e = D.part_range(A.nrows, P, rank)
        for q in range(P):
            want = maps[q][0].requests()[rank]
            assert np.array_equal(idx[off[q]:off[q + 1]] + b, want)
        # halo: the values each peer sends, landing in ghost order
        g, goff = m.ghosts()
        xg = np.empty(len(g))
        for q in range(P):
            qoff, qidx = maps[q][0].sends()
            qb, _ = D.part_range(A.nrows, P, q)
            xg[goff[q]:goff[q + 1]] = x[qb + qidx[qoff[rank]:qoff[rank + 1]]]
        xe = np.concatenate([x[b:e], xg])
        lc = m.local_cols()
        yl = np.zeros(e - b)
        for r in range(e - b):
            s = 0.0
            for k in range(rp[r], rp[r + 1]):
                s += vals[k] * xe[lc[k]]
            yl[r] = s
        assert np.array_equal(yl, yref[b:e])  # same k order -> same bits


def test_bad_requests_rejected(O):
    A = O.stencil("7pt", 6)
    rp, cols, _ = D.local_rows(A.row_ptr, A.cols, A.vals, 2, 0)
    m = D.DistMap(A.nrows, 2, 0, rp, cols)
    from paper_2011_08879_b200 import larch as lk
    with pytest.raises(lk.FormatError):  # id owned by rank 1
        m.set_sends([np.zeros(0, np.int32), np.array([A.nrows - 1], np.int32)])
    with pytest.raises(lk.ShapeError):
        D.DistMap(A.nrows, 2, 0, rp[:-1], cols)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        A = O.stencil("7pt", 12, 0.5)
        rp, cols, vals = D.local_rows(A.row_ptr, A.cols, A.vals, world, rank)
        m = D.DistMap(A.nrows, world, rank, rp, cols)
        D.exchange_requests(m)  # all-to-all over gloo
        b, e = D.part_range(A.nrows, world, rank)
        x = O.seeded_values(A.ncols, 11)
        # halo over gloo: each rank publishes its packed send buffer
        off, idx = m.sends()
        packed = [x[b + idx[off[p]:off[p + 1]]].tolist() for p in range(world)]
        every = [None] * world
        dist.all_gather_object(every, packed)
        g, goff = m.ghosts()
        xg = np.empty(len(g))
        for p in range(world):
            xg[goff[p]:goff[p + 1]] = every[p][rank]
        xe = np.concatenate([x[b:e], xg])
        lc = m.local_cols()
        y = np.zeros(e - b)
        for r in range(e - b):
            s = 0.0
            for k in range(rp[r], rp[r + 1]):
                s += vals[k] * xe[lc[k]]
            y[r] = s
        yref = O.spmv_csr(A, x)[b:e]
        # dot over gloo: the scalar allreduce of the solver
        import torch
        t = torch.tensor([float(np.dot(y, y))], dtype=torch.float64)
        dist.all_reduce(t)
        # the peer communicator's slot size: max over ranks of the largest
        # per-peer halo (both directions); 7-pt 12^3 split in two: one plane
        cap = D.peer_halo_cap(m)
        q.put((rank, bool(np.array_equal(y, yref)), float(t.item()), float(np.dot(O.spmv_csr(A, x),
                                                                                  O.spmv_csr(A, x))),
               cap, m.halo_count()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, tot, ref, cap, mine in res:
        assert ok, rank
        assert abs(tot - ref) <= 1e-12 * ref
        assert cap == 12 * 12 and mine == 12 * 12  # one 12x12 plane each way
