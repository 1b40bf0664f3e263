"""Out-of-bounds write checks with guard regions (compute-sanitizer is closed on this
GPU pool, so the library's device writes are bounded by our own canaries): the
workspace, the state and the residual output are carved out of larger device buffers
whose leading and trailing guard bands hold a bit pattern; after residual, RK4, RK54,
face-flux and diagnostics calls on every element path (fused tensor, fused simplex,
generic incl. prisms, far-field ghosts, the NCCL halo path) every guard byte must be
intact.  Also checks the workspace size query is exactly sufficient: the last used
byte can lie anywhere inside, but nothing may land past it."""
import numpy as np
import pytest

from sdrt_inputs import CONFIGS, initial_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GUARD = 1 << 20          # bytes per guard band
PAT = 0x5A               # guard byte


def _guarded(nbytes, dev):
    buf = torch.full((GUARD + nbytes + 256 + GUARD,), PAT, dtype=torch.uint8, device=dev)
    base = buf.data_ptr() + GUARD
    start = (base + 255) // 256 * 256
    return buf, start


def _check(buf, start, nbytes):
    host = buf.cpu().numpy()
    off = start - buf.data_ptr()
    assert (host[:off] == PAT).all(), "write before the region"
    assert (host[off + nbytes:] == PAT).all(), "write past the region"


CASES = [("c1", "quad", 2, (5, 4), None, {}), ("c2", "tri", 3, (4, 5), None, {}), ("c3", "hex", 4, (3, 3, 4), None, {}),
         ("c4", "hex", 3, (3, 4, 3), None, {}), ("c5", "tet", 3, (3, 3, 3), None, {}),
         ("c4", "pri", 3, (3, 3, 3), None, {}), ("c4", "hex", 3, (4, 3, 3), (0, 1, 1), {}),
         ("c5", "tet", 2, (3, 3, 3), None, {"loopback": True})]


@pytest.mark.parametrize("name,etype,p,N,per,opt", CASES)
def test_no_writes_outside_buffers(name, etype, p, N, per, opt):
    from paper_2105_08632_b200 import sdrt
    cfg = CONFIGS[name]
    dev = torch.device("cuda")
    st = torch.cuda.current_stream().cuda_stream
    m = sdrt.mesh_create(etype, p, list(N), cfg.lo, cfg.hi, periodic=per)
    if opt.get("loopback"):
        sdrt.mesh_set_halo(m, True)
    o = sdrt.operators_build(etype, p)
    ph = sdrt.physics(cfg.eq, **cfg.physics_kwargs())
    nbytes = sdrt.ctx_workspace_bytes(m, o, ph)
    wbuf, ws = _guarded(nbytes, dev)
    ctx = sdrt.ctx_create(m, o, ph, ws, nbytes, st)
    info = sdrt.mesh_info(m)
    nv = cfg.nvars
    if per is not None:
        ff = np.zeros(nv)
        ff[0] = 1.0
        if nv > 1:
            ff[-1] = 1.0 / (0.4 * 1.4 * 0.01)
        sdrt.ctx_set_farfield(ctx, ff, st)
    if opt.get("loopback"):
        sdrt.ctx_attach_comm(ctx, sdrt.comm_unique_id(), 0, 1)
    shape = (info["nsol"], nv, info["K_pad"])
    sbytes = int(np.prod(shape)) * 8
    ubuf, up = _guarded(sbytes, dev)
    rbuf, rp = _guarded(sbytes, dev)
    U = torch.zeros(shape, dtype=torch.float64)
    x = sdrt.mesh_sol_coords(m)
    U[:, :, :info["K"]] = torch.from_numpy(initial_state(cfg, x))
    torch.cuda.synchronize()
    host = U.numpy().view(np.uint8).reshape(-1)
    ubuf[up - ubuf.data_ptr(): up - ubuf.data_ptr() + sbytes].copy_(torch.from_numpy(host.copy()))
    sdrt.residual(ctx, up, rp, st)
    sdrt.rk_step(ctx, up, cfg.dt, 2, 0, st)
    if etype != "pri":
        sdrt.rk54_step(ctx, up, cfg.dt, 1, 0, st)
    if not opt.get("loopback"):
        fbytes = info["next"] * nv * info["K_pad"] * 8
        fbuf, fp = _guarded(fbytes, dev)
        sdrt.face_flux(ctx, up, rp, fp, st)
        torch.cuda.synchronize()
        _check(fbuf, fp, fbytes)
    if cfg.eq == "ns" and etype in ("hex", "tet") and per is None and not opt.get("loopback"):
        dbuf, dp = _guarded(24, dev)
        sdrt.diagnostics(ctx, up, dp, st)
        torch.cuda.synchronize()
        _check(dbuf, dp, 24)
    torch.cuda.synchronize()
    _check(wbuf, ws, nbytes)
    _check(ubuf, up, sbytes)
    _check(rbuf, rp, sbytes)
    sdrt.ctx_destroy(ctx)
    sdrt.operators_destroy(o)
    sdrt.mesh_destroy(m)
