"""GPU checks of the partitioned path.

* loopback: one rank, every periodic wrap routed through ghost columns + the device
  pack/unpack kernels (the library exchanges with itself) -> parity with the oracle;
* two ranks as two processes sharing cuda:0, pgrid splitting one axis, halo exchange
  through torch.distributed gloo with host staging (no kernel waits on another rank,
  B200_PROFILING.md) -> every rank's block equals the oracle's global run there.
"""
import os
import socket

import numpy as np
import pytest

from sdrt_inputs import CONFIGS, initial_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-11


def _rel(a, b):
    nv = a.shape[1]
    groups = [[0]] if nv == 1 else [[0], list(range(1, nv - 1)), [nv - 1]]
    return max(float(np.abs(a[:, g] - b[:, g]).max() / max(np.abs(b[:, g]).max(), 1e-300)) for g in groups)


def _oracle_run(cfg, N, steps):
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual, integrate
    m = build_mesh(cfg.etype, cfg.p, tuple(N), cfg.lo, cfg.hi)
    R = Residual(m, Physics(cfg.eq, cfg.nd, **cfg.physics_kwargs()))
    U0 = initial_state(cfg, m.sol_coords())
    return U0, R(U0), integrate(R, U0, cfg.dt, steps)


@pytest.mark.parametrize("name,N,steps", [("c1", [4, 5], 6), ("c2", [4, 4], 4), ("c3", [3, 3, 4], 3),
                                          ("c4", [3, 4, 3], 3), ("c5", [3, 3, 3], 2)])
def test_loopback_halo_parity(name, N, steps):
    from paper_2105_08632_b200.solver import Solver
    cfg = CONFIGS[name]
    U0, r_ref, u_ref = _oracle_run(cfg, N, steps)
    S = Solver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, force_self_halo=True, **cfg.physics_kwargs())
    assert S.info["K_trace"] > S.info["K_pad"]
    r = S.to_host(S.residual(S.to_device(U0)))
    assert _rel(r, r_ref) <= TOL
    U = S.to_device(U0)
    S.rk_step(U, cfg.dt, steps)
    assert _rel(S.to_host(U), u_ref) <= TOL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, name, N, pgrid, steps, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
        torch.cuda.set_device(0)
        from paper_2105_08632_b200.dist import DistSolver, global_ids
        cfg = CONFIGS[name]
        U0g, r_ref, u_ref = _oracle_run(cfg, N, steps)
        S = DistSolver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, device="cuda:0", pgrid=pgrid, staging=True,
                       **cfg.physics_kwargs())
        gid = global_ids(S.info)
        r = S.to_host(S.residual(S.to_device(U0g[:, :, gid])))
        e1 = _rel(r, r_ref[:, :, gid])
        U = S.to_device(U0g[:, :, gid])
        S.rk_step(U, cfg.dt, steps)
        e2 = _rel(S.to_host(U), u_ref[:, :, gid])
        q.put((rank, "ok", e1, e2, S.exchanges))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc(), 0, 0))


@pytest.mark.parametrize("name,N,pgrid,steps", [("c4", [4, 3, 3], [2, 1, 1], 2), ("c5", [3, 4, 3], [1, 2, 1], 1),
                                                ("c2", [4, 4], [2, 1], 3)])
def test_two_rank_gloo_on_one_gpu(name, N, pgrid, steps):
    import torch.multiprocessing as mp
    from paper_2105_08632_b200.build import build
    build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, name, N, pgrid, steps, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    for r in res:
        assert r[1] == "ok", r[2]
        assert r[2] <= TOL and r[3] <= TOL, r
        assert r[4] > 0


@pytest.mark.parametrize("name,N,steps", [("c4", [24, 4, 4], 2), ("c5", [6, 4, 4], 1), ("c2", [24, 4], 2)])
def test_overlapped_stage_parts_bitwise(name, N, steps):
    """The overlapped stage: interior tiles while the exchange is in
    flight, boundary tiles after the unpack (sdrt_stage_*_part, DistSolver.rk_step).
    Single-rank loopback halo on every axis; meshes long enough in x that interior tiles
    exist.  Must equal the unsplit library step bit for bit."""
    from paper_2105_08632_b200 import sdrt
    from paper_2105_08632_b200.dist import DistSolver
    from paper_2105_08632_b200.solver import Solver

    class Loopback(DistSolver):
        def start_exchange(self, which):
            st = self._stream()
            sdrt.halo_pack(self.ctx, which, self.send.data_ptr(), st)
            index = {(d, s): i for i, (d, s) in enumerate(zip(self.sd, self.sside))}
            for i in range(len(self.sd)):
                j = index[(self.sd[i], 1 - self.sside[i])]
                self.recv[self.off[i]:self.off[i + 1]].copy_(self.send[self.off[j]:self.off[j + 1]])
            return which

        def finish_exchange(self, which):
            if which is None:
                return
            sdrt.halo_unpack(self.ctx, which, self.recv.data_ptr(), self._stream())
            self.exchanges += 1

    cfg = CONFIGS[name]
    S1 = Loopback(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, device="cuda", force_self_halo=True,
                  transport="torch", **cfg.physics_kwargs())
    S0 = Solver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, device="cuda", force_self_halo=True,
                **cfg.physics_kwargs())
    U0 = initial_state(cfg, S0.sol_coords())
    U1, U2 = S1.to_device(U0), S0.to_device(U0)
    S1.rk_step(U1, cfg.dt, steps)
    S0.rk_step(U2, cfg.dt, steps)
    a, b = S1.to_host(U1), S0.to_host(U2)
    assert S1.exchanges > 0
    assert np.array_equal(a, b), float(np.abs(a - b).max())
    # the RK54 stages through the same overlapped sequence
    S1.rk54_step(U1, cfg.dt, 1)
    S0.rk54_step(U2, cfg.dt, 1)
    a, b = S1.to_host(U1), S0.to_host(U2)
    assert np.array_equal(a, b), float(np.abs(a - b).max())


@pytest.mark.parametrize("name,N,steps", [("c4", [24, 4, 4], 3), ("c5", [6, 4, 4], 2), ("c2", [24, 4], 3),
                                          ("c3", [6, 3, 3], 2)])
def test_library_nccl_exchange(name, N, steps):
    """NCCL inside libsdrt (sdrt_comm_unique_id / sdrt_ctx_attach_comm): a one-rank
    communicator whose periodic faces are all halo slabs, so every stage packs its face
    traces, exchanges them with grouped ncclSend/ncclRecv on the library's comm stream
    (here to itself), unpacks them into the ghost columns and overlaps the interior tiles
    -- the multi-rank code path end to end on one GPU.  Must equal the single-rank
    library step bit for bit and the oracle to 1e-11; RK54 and the all-reduced
    divergence check run through it too."""
    from paper_2105_08632_b200 import sdrt
    from paper_2105_08632_b200.dist import DistSolver
    from paper_2105_08632_b200.solver import Solver
    cfg = CONFIGS[name]
    S1 = DistSolver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, device="cuda", force_self_halo=True,
                    transport="library", **cfg.physics_kwargs())
    assert S1.transport == "library"
    S0 = Solver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    U0, r_ref, u_ref = _oracle_run(cfg, N, steps)
    r1 = S1.to_host(S1.residual(S1.to_device(U0)))
    assert _rel(r1, r_ref) <= TOL
    U1, U2 = S1.to_device(U0), S0.to_device(U0)
    S1.rk_step(U1, cfg.dt, steps, check_every=1)
    S0.rk_step(U2, cfg.dt, steps)
    a, b = S1.to_host(U1), S0.to_host(U2)
    assert np.array_equal(a, b), float(np.abs(a - b).max())
    assert _rel(a, u_ref) <= TOL
    S1.rk54_step(U1, cfg.dt, 1)
    S0.rk54_step(U2, cfg.dt, 1)
    assert np.array_equal(S1.to_host(U1), S0.to_host(U2))
    if cfg.nvars > 1:  # a bad state is reported through the all-reduced check
        Ub = S1.to_device(U0)
        Ub[:, 0, 3] = -1.0
        with pytest.raises(sdrt.SdrtError) as e:
            S1.rk_step(Ub, 0.0, 1, check_every=1)
        assert e.value.code == -7
