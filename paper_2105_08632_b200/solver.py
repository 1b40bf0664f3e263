"""Solver: owns a mesh, operators and a device context over torch-allocated memory.

Plumbing only: torch provides the device workspace, state tensors and streams;
every step of the residual / RK4 path runs in libsdrt.so's kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import sdrt


class Solver:
    def __init__(self, etype, p, N, lo, hi, eq, device="cuda", rank=0, nranks=1, pgrid=None, _pre_ctx=None,
                 force_self_halo=False, scheme="sdrt", periodic=None, farfield=None, **phys):
        D = 2 if etype in ("quad", "tri") else 3
        Nl = list(N) if np.ndim(N) else [int(N)] * D
        self.mesh = sdrt.mesh_create(etype, p, Nl, lo, hi, rank=rank, nranks=nranks, pgrid=pgrid,
                                     periodic=periodic)
        if _pre_ctx is not None:
            _pre_ctx(self.mesh)
        elif force_self_halo:
            sdrt.mesh_set_halo(self.mesh, True)   # loopback halo: the library exchanges itself
        self.ops = sdrt.operators_build(etype, p, scheme)
        self.info = sdrt.mesh_info(self.mesh)
        self.phys = sdrt.physics(eq, **phys)
        self.nv = 1 if eq in ("linadv", "linadvdiff") else D + 2
        self.visc = eq in ("linadvdiff", "ns")
        self.device = torch.device(device)
        nbytes = sdrt.ctx_workspace_bytes(self.mesh, self.ops, self.phys)
        if nbytes == 0:
            raise RuntimeError("workspace query failed: " + sdrt.last_error())
        self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.ws.data_ptr()
        self._ws_ptr = (base + 255) // 256 * 256
        self._ws_bytes = nbytes
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.ctx = sdrt.ctx_create(self.mesh, self.ops, self.phys, self._ws_ptr, nbytes, stream)
        if farfield is not None:  # exterior state of the non-periodic axes
            sdrt.ctx_set_farfield(self.ctx, farfield, stream)

    @property
    def shape(self):
        return (self.info["nsol"], self.nv, self.info["K_pad"])

    @property
    def K(self):
        return self.info["K"]

    def sol_coords(self):
        return sdrt.mesh_sol_coords(self.mesh)

    def to_device(self, U_np):
        """(N_sol, N_V, K) numpy -> padded device tensor (N_sol, N_V, K_pad)."""
        U = torch.zeros(self.shape, dtype=torch.float64, device=self.device)
        U[:, :, : self.K] = torch.from_numpy(np.ascontiguousarray(U_np))
        return U

    def to_host(self, U):
        return U[:, :, : self.K].cpu().numpy()

    def residual(self, U, out=None):
        out = torch.empty_like(U) if out is None else out
        sdrt.residual(self.ctx, U.data_ptr(), out.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
        return out

    def face_flux(self, U):
        """(dU/dt, F): the residual and the common flux F each element applied at each of
        its external points, [N_ext][N_V][K_pad] (reading O28; sdrt_face_flux)."""
        out = torch.empty_like(U)
        F = torch.zeros((self.info["next"], self.nv, self.info["K_pad"]), dtype=torch.float64, device=self.device)
        sdrt.face_flux(self.ctx, U.data_ptr(), out.data_ptr(), F.data_ptr(),
                       torch.cuda.current_stream(self.device).cuda_stream)
        return out, F

    def rk_step(self, U, dt, nsteps=1, check_every=0):
        sdrt.rk_step(self.ctx, U.data_ptr(), dt, nsteps, check_every,
                     torch.cuda.current_stream(self.device).cuda_stream)
        return U

    def rk54_step(self, U, dt, nsteps=1, check_every=0):
        """RK54 (five stages, two registers)."""
        sdrt.rk54_step(self.ctx, U.data_ptr(), dt, nsteps, check_every,
                       torch.cuda.current_stream(self.device).cuda_stream)
        return U

    def host_steps(self, H, U, dt, nsteps, rk54=False, chunks=8):
        """Advance a HOST-resident state H (pinned, self.shape) by nsteps RK steps, each step a
        full round trip: H -> device (U, scratch), one sdrt_rk_step / sdrt_rk54_step, device
        -> H; step i+1 reads step i's result from H.  The copies go in `chunks` contiguous
        pieces on two copy streams ordered per piece by events: piece k of step i+1's upload
        waits only for piece k of step i's download, so the two PCIe directions run
        concurrently while keeping the dependency.  All asynchronous on the current stream
        (no host synchronisation)."""
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        if not hasattr(self, "_copy_streams"):
            self._copy_streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        sd, sh = self._copy_streams
        fh, fu = H.view(-1), U.view(-1)
        n = fu.numel()
        cut = [n * k // chunks for k in range(chunks + 1)]
        sh.wait_stream(cur)
        with torch.cuda.stream(sh):
            fu.copy_(fh, non_blocking=True)
        step = self.rk54_step if rk54 else self.rk_step
        for i in range(nsteps):
            cur.wait_stream(sh)
            step(U, dt, 1)
            sd.wait_stream(cur)
            for k in range(chunks):
                a, b = cut[k], cut[k + 1]
                with torch.cuda.stream(sd):
                    fh[a:b].copy_(fu[a:b], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(sd)
                if i + 1 < nsteps:
                    sh.wait_event(ev)
                    with torch.cuda.stream(sh):
                        fu[a:b].copy_(fh[a:b], non_blocking=True)
        cur.wait_stream(sd)
        return H

    def diagnostics(self, U, degree=10):
        """TGV ensemble averages (<E*>, eps2, eps3), PAPER.md l.2052-2080 (3-D NS), by the
        quadrature exact to `degree` (the paper's 10, l.2075; 0 = solution points)."""
        if degree != getattr(self, "_diag_degree", 10):
            sdrt.diagnostics_rule(self.ctx, degree)
        self._diag_degree = degree
        out = torch.empty(3, dtype=torch.float64, device=self.device)
        sdrt.diagnostics(self.ctx, U.data_ptr(), out.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
        return out.cpu().numpy()

    def set_timing(self, enable):
        sdrt.ctx_set_timing(self.ctx, enable)

    def set_graph(self, mode):
        """CUDA-graph replay of repeated K-step calls: -1 auto (small meshes), 0 off, 1 on."""
        sdrt.ctx_set_graph(self.ctx, mode)

    def kernel_times(self):
        return sdrt.ctx_kernel_times(self.ctx)

    def last_launches(self):
        return sdrt.ctx_last_launches(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            sdrt.ctx_destroy(self.ctx)
            self.ctx = None
        if getattr(self, "mesh", None):
            sdrt.mesh_destroy(self.mesh)
            self.mesh = None
        if getattr(self, "ops", None):
            sdrt.operators_destroy(self.ops)
            self.ops = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def from_config(cfg, device="cuda", N=None):
    return Solver(cfg.etype, cfg.p, cfg.N if N is None else N, cfg.lo, cfg.hi, cfg.eq, device=device,
                  **cfg.physics_kwargs())
