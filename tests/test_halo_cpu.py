"""Multi-rank host logic on the CPU (no GPU): element partition, ghost columns and halo
lists of libsdrt, exchanged for real between gloo ranks (world_size 2 and 4) and checked
against the ORACLE's global face pairing.

Every rank fills its trace array T[row][v][col] with a code of (global element, row, v),
packs its send lists, exchanges per slab exactly as paper_2105_08632_b200.dist does
(tags 2d+side, recv into the opposite slab), unpacks into its ghost columns, and then
checks, for every local element and face point, that the column the kernels read for
the neighbour (sdrt_mesh_neighbor) holds the code of the neighbour element and point
that the oracle's brute-force coordinate matching assigns.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NV = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _code(g, row, v):
    return g * 10000.0 + row * 10.0 + v


def _worker(rank, ws, port, etype, p, N, pgrid, force, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        if ws > 1:
            dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
        from paper_2105_08632_b200 import sdrt
        from paper_2105_08632_b200.dist import global_ids
        from oracle.mesh import build_mesh
        D = len(N)
        lo, hi = [0.0] * D, [1.0 + 0.25 * d for d in range(D)]
        m = sdrt.mesh_create(etype, p, N, lo, hi, rank=rank, nranks=ws, pgrid=pgrid)
        sdrt.mesh_set_halo(m, force)
        info = sdrt.mesh_info(m)
        K, Kt, nx, nfp, nf = info["K"], info["K_trace"], info["next"], info["nfp"], info["nfaces"]
        gid = global_ids(info)
        T = np.full((nx, NV, Kt), np.nan)
        rows = np.arange(nx)[:, None, None]
        vs = np.arange(NV)[None, :, None]
        T[:, :, :K] = _code(gid[None, None, :], rows, vs)
        slabs = sdrt.mesh_halo_lists(m)
        index = {(d, s): i for i, (_, d, s, *_r) in enumerate(slabs)}
        recvd = {}
        if ws > 1:
            ops, bufs = [], []
            for i, (peer, d, side, sr, sc, rr, rc) in enumerate(slabs):
                j = index[(d, 1 - side)]
                send = torch.from_numpy(np.ascontiguousarray(T[sr, :, sc]).reshape(-1))
                recv = torch.empty(len(slabs[j][5]) * NV, dtype=torch.float64)
                ops.append(dist.P2POp(dist.isend, send, peer, tag=2 * d + side))
                ops.append(dist.P2POp(dist.irecv, recv, slabs[j][0], tag=2 * d + side))
                bufs.append((send, recv, j))
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            for send, recv, j in bufs:
                recvd[j] = recv.numpy().reshape(-1, NV)
        else:  # loopback: slab (d, s) receives what slab (d, 1-s) sent
            for i, (peer, d, side, sr, sc, rr, rc) in enumerate(slabs):
                j = index[(d, 1 - side)]
                recvd[j] = T[sr, :, sc].reshape(-1, NV)
        for j, vals in recvd.items():
            _, _, _, sr, sc, rr, rc = slabs[j]
            assert len(vals) == len(rr)
            T[rr, :, rc] = vals
        # oracle global pairing
        M = build_mesh(etype, p, tuple(N), lo, hi)
        nchecked = nghost = 0
        for e in range(K):
            g = gid[e]
            for f in range(nf):
                col, f2 = sdrt.mesh_neighbor(m, e, f)
                for qq in range(nfp):
                    rho = f * nfp + qq
                    gn, rn = M.nbr_elem[rho, g], M.nbr_pt[rho, g]
                    assert rn // nfp == f2
                    got = T[rn, :, col]
                    exp = _code(gn, rn, np.arange(NV))
                    assert np.array_equal(got, exp), (rank, e, f, qq, col, got, exp)
                    nchecked += 1
                    nghost += col >= info["K_pad"]
        q.put((rank, "ok", nchecked, nghost))
        if ws > 1:
            dist.destroy_process_group()
    except Exception as ex:  # report to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc(), 0))


def _run(etype, p, N, pgrid, ws, force=False):
    from paper_2105_08632_b200.build import build
    build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, etype, p, N, pgrid, force, q)) for r in range(ws)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(ws)]
    for pr in procs:
        pr.join(timeout=60)
    for r in res:
        assert r[1] == "ok", r[2]
    return res


@pytest.mark.parametrize("etype,p,N,pgrid", [
    ("quad", 2, [4, 3], [2, 1]),
    ("tri", 2, [4, 4], [1, 2]),
    ("hex", 1, [4, 3, 3], [2, 1, 1]),
    ("tet", 1, [3, 4, 3], [1, 2, 1]),
])
def test_halo_two_ranks_gloo(etype, p, N, pgrid):
    res = _run(etype, p, N, pgrid, 2)
    assert all(r[3] > 0 for r in res)  # ghost columns were exercised on every rank


def test_halo_four_ranks_gloo():
    res = _run("tri", 1, [4, 4], [2, 2], 4)
    assert all(r[3] > 0 for r in res)


@pytest.mark.parametrize("etype,p,N", [("quad", 2, [3, 4]), ("tet", 2, [3, 3, 3])])
def test_halo_loopback_single_rank(etype, p, N):
    res = _run(etype, p, N, None, 1, force=True)
    assert res[0][3] > 0
