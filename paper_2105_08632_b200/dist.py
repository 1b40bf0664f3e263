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
    """1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2 (x first)."""
    g = [1, 1, 1]
    k, d = nranks, 0
    while k > 1:
        if k % 2:
            raise ValueError("nranks must be a power of two")
        g[d % nd] *= 2
        k //= 2
        d += 1
    return g[:nd]


class DistSolver(Solver):
    """Solver over this rank's block; rk_step / residual run the staged API with a halo
    exchange after every trace-producing kernel."""

    def __init__(self, etype, p, N, lo, hi, eq, device="cuda", group=None, pgrid=None, staging=False,
                 force_self_halo=False, **phys):
        self.group = group
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        D = 2 if etype in ("quad", "tri") else 3
        pgrid = list(pgrid) if pgrid is not None else default_pgrid(nranks, D)
        self._force = force_self_halo
        super().__init__(etype, p, N, lo, hi, eq, device=device, rank=rank, nranks=nranks, pgrid=pgrid,
                         _pre_ctx=self._set_halo, **phys)
        self.rank = rank
        self.staging = staging
        self.peers, self.sd, self.sside, self.off = sdrt.halo_info(self.ctx)
        n = self.off[-1] if self.off else 0
        self.send = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.recv = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.exchanges = 0

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
        return self._steps(U, dt, nsteps, [sdrt.RK54_STAGE0 + s for s in range(5)])

    def rk_step(self, U, dt, nsteps=1, check_every=0):
        return self._steps(U, dt, nsteps, [0, 1, 2, 3])

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
