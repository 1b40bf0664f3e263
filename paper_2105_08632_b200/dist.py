"""Element-partitioned multi-rank SDRT: one rank per GPU, pattern-block
partition (pgrid), face-trace halo exchange through torch.distributed point-to-point
(NCCL over NVLink on GPUs; gloo with host staging for CPU-side / single-device tests).

Per RK stage (row A12 of SURVEY §8(a)): the U traces of the stage input and, for
viscous equations, the published viscous normal-flux traces are the only values that
cross a partition face; both are exactly the arrays the fused kernels exchange through
HBM on one GPU, so the partitioned result equals the single-rank one element by element.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import sdrt
from .solver import Solver


def default_pgrid(nranks, nd):
    """Pattern-block partition over the SLOW axes (3-D: z, y, z, ...; 2-D: y):
    3-D 1 -> 1x1x1, 2 -> 1x1x2, 4 -> 1x2x2, 8 -> 1x2x4.  The fused kernels' tiles are runs
    of consecutive elements along x, so a partition face normal to x would make the first
    and last tile of every x-row a boundary tile (SURVEY §8(e)'s 2x2x2 leaves 44 % of the
    c4 tiles interior); with x never cut, a tile is boundary only in the y/z pattern layers
    next to a partition face: 88 % of c4's tiles run while the halo exchange is in flight
    (the interior-first effect of §8(e) without reordering the ABI element order)."""
    g = [1, 1, 1]
    axes = [2, 1] if nd == 3 else [1]
    k, i = nranks, 0
    while k > 1:
        if k % 2:
            raise ValueError("nranks must be a power of two")
        g[axes[i % len(axes)]] *= 2
        k //= 2
        i += 1
    return g[:nd]


class DistSolver(Solver):
    """Solver over this rank's block.

    transport = "library" (default for CUDA devices without host staging): the halo
    exchange runs inside libsdrt over NCCL (sdrt_comm_unique_id on rank 0, broadcast with
    torch.distributed, sdrt_ctx_attach_comm on every rank); rk_step / residual are then the
    plain library calls.  transport = "torch": the staged API with the exchange through
    torch.distributed point-to-point (gloo with host staging: CPU-side and single-device
    multi-process tests)."""

    def __init__(self, etype, p, N, lo, hi, eq, device="cuda", group=None, pgrid=None, staging=False,
                 force_self_halo=False, transport=None, **phys):
        self.group = group
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        D = 2 if etype in ("quad", "tri") else 3
        pgrid = list(pgrid) if pgrid is not None else default_pgrid(nranks, D)
        self._force = force_self_halo
        super().__init__(etype, p, N, lo, hi, eq, device=device, rank=rank, nranks=nranks, pgrid=pgrid,
                         _pre_ctx=self._set_halo, **phys)
        self.rank = rank
        self.nranks = nranks
        self.staging = staging
        self.peers, self.sd, self.sside, self.off = sdrt.halo_info(self.ctx)
        n = self.off[-1] if self.off else 0
        self.send = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.recv = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.exchanges = 0
        if transport is None:
            transport = "library" if (self.device.type == "cuda" and not staging and len(self.peers) > 0) else "torch"
        self.transport = transport
        if transport == "library":
            uid = [sdrt.comm_unique_id() if rank == 0 else None]
            if nranks > 1:
                dist.broadcast_object_list(uid, src=0, group=group)
            sdrt.ctx_attach_comm(self.ctx, uid[0], rank, nranks)

    def _set_halo(self, mesh):
        sdrt.mesh_set_halo(mesh, self._force)

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def exchange(self, which):
        """Pack this rank's outgoing traces, P2P exchange per slab, unpack into ghosts."""
        self.finish_exchange(self.start_exchange(which))

    def start_exchange(self, which):
        """Pack on the compute stream and post the P2P sends/receives (NCCL runs them on
        its own stream, ordered after the pack); returns a handle for finish_exchange."""
        nslab = len(self.peers)
        if nslab == 0:
            return None
        st = self._stream()
        sdrt.halo_pack(self.ctx, which, self.send.data_ptr(), st)
        send, recv = self.send, self.recv
        if self.staging:
            send = self.send.cpu()
            recv = torch.empty_like(send)
        ops = []
        index = {(d, s): i for i, (d, s) in enumerate(zip(self.sd, self.sside))}
        for i in range(nslab):
            d, side = self.sd[i], self.sside[i]
            j = index[(d, 1 - side)]
            seg_s = send[self.off[i]:self.off[i + 1]]
            seg_r = recv[self.off[j]:self.off[j + 1]]
            # what I send from slab (d, side) lands in the peer's slab (d, 1-side); what I
            # receive in slab (d, 1-side) the peer there sent from its slab (d, side)
            ops.append(dist.P2POp(dist.isend, seg_s, self.peers[i], group=self.group, tag=2 * d + side))
            ops.append(dist.P2POp(dist.irecv, seg_r, self.peers[j], group=self.group, tag=2 * d + side))
        if self.staging:
            torch.cuda.synchronize(self.device)
        return which, dist.batch_isend_irecv(ops), recv

    def finish_exchange(self, h):
        """Wait for the posted transfers (a stream dependency for NCCL) and unpack."""
        if h is None:
            return
        which, works, recv = h
        for r in works:
            r.wait()
        if self.staging:
            self.recv.copy_(recv)
        sdrt.halo_unpack(self.ctx, which, self.recv.data_ptr(), self._stream())
        self.exchanges += 1

    def residual(self, U, out=None):
        if self.transport == "library":
            return Solver.residual(self, U, out)
        out = torch.empty_like(U) if out is None else out
        st = self._stream()
        sdrt.stage_traces(self.ctx, U.data_ptr(), st)
        self.exchange(0)
        if self.visc:
            sdrt.stage_grad(self.ctx, U.data_ptr(), -1, st)
            self.exchange(1)
        sdrt.stage_flux(self.ctx, U.data_ptr(), -1, 0.0, out.data_ptr(), st)
        return out

    def rk54_step(self, U, dt, nsteps=1, check_every=0):
        """RK54 over the same overlapped staged sequence (stage codes 10..14)."""
        if self.transport == "library":
            return Solver.rk54_step(self, U, dt, nsteps, check_every)
        return self._checked(U, dt, nsteps, check_every, [sdrt.RK54_STAGE0 + s for s in range(5)])

    def rk_step(self, U, dt, nsteps=1, check_every=0):
        if self.transport == "library":
            return Solver.rk_step(self, U, dt, nsteps, check_every)
        return self._checked(U, dt, nsteps, check_every, [0, 1, 2, 3])

    def _checked(self, U, dt, nsteps, check_every, stages):
        """torch transport: the steps in chunks of check_every with an all-reduced
        finite / positive-density / positive-energy check after each (the library does
        the same on its own transport, SDRT_E_DIVERGED on every rank together)."""
        done = 0
        while done < nsteps:
            n = min(check_every, nsteps - done) if check_every > 0 else nsteps - done
            self._steps(U, dt, n, stages)
            done += n
            if check_every > 0:
                u = U[:, :, :self.K]
                ok = bool(torch.isfinite(u).all())
                if ok and self.nv > 1:
                    ok = bool((u[:, 0] > 0).all()) and bool((u[:, -1] > 0).all())
                flag = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64,
                                    device=self.device if dist.is_initialized() and
                                    dist.get_backend(self.group) == "nccl" else "cpu")
                if dist.is_initialized():
                    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
                if flag.item() < 1.0:
                    raise sdrt.SdrtError(-7, f"diverged after step {done} (rank {self.rank}: "
                                             f"{'bad' if not ok else 'ok'} locally)")
        return U

    def _steps(self, U, dt, nsteps, stages):
        """Time steps with the halo exchange overlapped with interior work: each
        exchange is posted, the interior tiles (no ghost reads) run while it is in
        flight, then the boundary tiles after the unpack.  Same arithmetic per element
        as the unsplit stage, so the result is identical."""
        st = self._stream()
        U_ptr = U.data_ptr()
        sdrt.stage_traces(self.ctx, U_ptr, st)
        h0 = self.start_exchange(0)
        for _ in range(nsteps):
            for s in stages:
                if self.visc:
                    sdrt.stage_grad_part(self.ctx, U_ptr, s, 1, st)
                    self.finish_exchange(h0)
                    sdrt.stage_grad_part(self.ctx, U_ptr, s, 2, st)
                    h1 = self.start_exchange(1)
                    sdrt.stage_flux_part(self.ctx, U_ptr, s, dt, 0, 1, st)
                    self.finish_exchange(h1)
                else:
                    sdrt.stage_flux_part(self.ctx, U_ptr, s, dt, 0, 1, st)
                    self.finish_exchange(h0)
                sdrt.stage_flux_part(self.ctx, U_ptr, s, dt, 0, 2, st)
                h0 = self.start_exchange(0)
        self.finish_exchange(h0)
        return U


def global_ids(info):
    """Global element ids of this rank's local elements (pattern x fastest, then sub-cell)."""
    nd, nsub = info["nd"], info["nsub"]
    N, Ng, off = info["N"], info["Nglobal"], info["offset"]
    K = info["K"]
    e = np.arange(K)
    pat = e // nsub
    c = []
    for d in range(nd):
        c.append(pat % N[d] + off[d])
        pat = pat // N[d]
    g = np.zeros(K, dtype=np.int64)
    mul = 1
    for d in range(nd):
        g += mul * c[d]
        mul *= Ng[d]
    return g * nsub + e % nsub
