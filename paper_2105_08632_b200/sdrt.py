"""Thin ctypes binding of libsdrt.so (include/sdrt.h): argument marshalling only.

Every function has the C name without the ``sdrt_`` prefix.  Device buffers are
passed as raw pointers (torch tensors' data_ptr()); streams as cudaStream_t
handles (``torch.cuda.current_stream().cuda_stream``).  There is no CPU fallback:
importing this module fails loudly if the shared library is missing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("SDRT_LIB") or os.path.join(_HERE, "libsdrt.so")
if not os.path.exists(_LIBPATH):
    raise ImportError(f"libsdrt.so not built ({_LIBPATH}); run __graft_entry__.build() or "
                      "python paper_2105_08632_b200/build.py")
lib = ctypes.CDLL(_LIBPATH)

ETYPES = {"quad": 0, "tri": 1, "hex": 2, "tet": 3, "pri": 4}
EQS = {"linadv": 0, "linadvdiff": 1, "euler": 2, "ns": 3}
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "UNSUPPORTED", -3: "ILL_CONDITIONED", -4: "CUDA",
          -5: "NCCL", -6: "WORKSPACE", -7: "DIVERGED", -8: "INTERNAL"}


class SdrtError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"sdrt {STATUS.get(code, code)}: {msg}")
        self.code = code


class MeshInfo(ctypes.Structure):
    _fields_ = [("etype", ctypes.c_int), ("p", ctypes.c_int), ("nd", ctypes.c_int),
                ("nsol", ctypes.c_int), ("next", ctypes.c_int), ("nint", ctypes.c_int),
                ("nu", ctypes.c_int), ("nfaces", ctypes.c_int), ("nfp", ctypes.c_int),
                ("nsub", ctypes.c_int), ("N", ctypes.c_int * 3), ("Nglobal", ctypes.c_int * 3),
                ("offset", ctypes.c_int * 3), ("K", ctypes.c_int64), ("K_pad", ctypes.c_int64),
                ("n_faces", ctypes.c_int64), ("K_trace", ctypes.c_int64)]


class PhysicsT(ctypes.Structure):
    _fields_ = [("eq", ctypes.c_int), ("c", ctypes.c_double * 3), ("mu", ctypes.c_double),
                ("gamma", ctypes.c_double), ("Pr", ctypes.c_double), ("beta", ctypes.c_double),
                ("eta", ctypes.c_double)]


_vp = ctypes.c_void_p
_i3 = ctypes.c_int * 3
_d3 = ctypes.c_double * 3
lib.sdrt_abi_version.restype = ctypes.c_int
lib.sdrt_last_error.restype = ctypes.c_char_p
lib.sdrt_mesh_create.argtypes = [ctypes.c_int, ctypes.c_int, _i3, _d3, _d3, _i3, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_vp)]
lib.sdrt_mesh_info.argtypes = [_vp, ctypes.POINTER(MeshInfo)]
lib.sdrt_mesh_export_maps.argtypes = [_vp, _vp, _vp, _vp, _vp]
lib.sdrt_mesh_sol_coords.argtypes = [_vp, _vp]
lib.sdrt_mesh_detj.argtypes = [_vp, _vp]
lib.sdrt_mesh_destroy.argtypes = [_vp]
lib.sdrt_mesh_destroy.restype = None
lib.sdrt_operators_build.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]
lib.sdrt_operators_get.argtypes = [_vp, ctypes.c_char_p, _vp, ctypes.POINTER(ctypes.c_int),
                                   ctypes.POINTER(ctypes.c_int)]
lib.sdrt_operators_destroy.argtypes = [_vp]
lib.sdrt_operators_destroy.restype = None
lib.sdrt_ctx_workspace_bytes.argtypes = [_vp, _vp, ctypes.POINTER(PhysicsT)]
lib.sdrt_ctx_workspace_bytes.restype = ctypes.c_size_t
lib.sdrt_ctx_create.argtypes = [_vp, _vp, ctypes.POINTER(PhysicsT), _vp, ctypes.c_size_t, _vp, ctypes.POINTER(_vp)]
lib.sdrt_residual.argtypes = [_vp, _vp, _vp, _vp]
lib.sdrt_face_flux.argtypes = [_vp, _vp, _vp, _vp, _vp]
lib.sdrt_rk_step.argtypes = [_vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int, _vp]
lib.sdrt_rk54_step.argtypes = [_vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int, _vp]
lib.sdrt_diagnostics.argtypes = [_vp, _vp, _vp, _vp]
lib.sdrt_diagnostics_rule.argtypes = [_vp, ctypes.c_int]
lib.sdrt_mesh_set_halo.argtypes = [_vp, ctypes.c_int]
lib.sdrt_mesh_halo_lists.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
lib.sdrt_mesh_neighbor.argtypes = [_vp, ctypes.c_int64, ctypes.c_int, _vp, _vp]
lib.sdrt_halo_info.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
lib.sdrt_halo_pack.argtypes = [_vp, ctypes.c_int, _vp, _vp]
lib.sdrt_halo_unpack.argtypes = [_vp, ctypes.c_int, _vp, _vp]
lib.sdrt_stage_traces.argtypes = [_vp, _vp, _vp]
lib.sdrt_stage_grad.argtypes = [_vp, _vp, ctypes.c_int, _vp]
lib.sdrt_stage_flux.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_double, _vp, _vp]
lib.sdrt_stage_grad_part.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp]
lib.sdrt_stage_flux_part.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_double, _vp, ctypes.c_int, _vp]
lib.sdrt_ctx_set_timing.argtypes = [_vp, ctypes.c_int]
lib.sdrt_ctx_set_graph.argtypes = [_vp, ctypes.c_int]
lib.sdrt_ctx_kernel_times.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.POINTER(ctypes.c_int)]
lib.sdrt_ctx_last_launches.argtypes = [_vp]
lib.sdrt_ctx_last_launches.restype = ctypes.c_int64
lib.sdrt_comm_unique_id.argtypes = [_vp]
lib.sdrt_ctx_set_farfield.argtypes = [_vp, _vp, _vp]
lib.sdrt_ctx_attach_comm.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int]
lib.sdrt_ctx_destroy.argtypes = [_vp]
lib.sdrt_ctx_destroy.restype = None

EXPORTED = ["sdrt_abi_version", "sdrt_last_error", "sdrt_mesh_create", "sdrt_mesh_info",
            "sdrt_mesh_export_maps", "sdrt_mesh_sol_coords", "sdrt_mesh_detj", "sdrt_mesh_destroy",
            "sdrt_operators_build", "sdrt_operators_get", "sdrt_operators_destroy",
            "sdrt_ctx_workspace_bytes", "sdrt_ctx_create", "sdrt_residual", "sdrt_face_flux", "sdrt_rk_step",
            "sdrt_ctx_last_launches", "sdrt_ctx_destroy", "sdrt_ctx_set_timing", "sdrt_ctx_set_graph",
            "sdrt_ctx_kernel_times",
            "sdrt_mesh_set_halo", "sdrt_mesh_halo_lists", "sdrt_mesh_neighbor", "sdrt_halo_info",
            "sdrt_halo_pack", "sdrt_halo_unpack", "sdrt_stage_traces", "sdrt_stage_grad", "sdrt_stage_flux",
            "sdrt_comm_unique_id", "sdrt_ctx_attach_comm", "sdrt_ctx_set_farfield"]


def _check(code):
    if code != 0:
        raise SdrtError(code, lib.sdrt_last_error().decode())


def abi_version():
    return lib.sdrt_abi_version()


def last_error():
    return lib.sdrt_last_error().decode()


# ------------------------------------------------------------------ meshes
def mesh_create(etype, p, N, lo, hi, rank=0, nranks=1, pgrid=None, periodic=None):
    et = ETYPES[etype] if isinstance(etype, str) else int(etype)
    N3 = list(N) + [1] * (3 - len(N))
    lo3 = list(lo) + [0.0] * (3 - len(lo))
    hi3 = list(hi) + [1.0] * (3 - len(hi))
    per = [1, 1, 1] if periodic is None else [int(bool(x)) for x in periodic] + [1] * (3 - len(periodic))
    pg = None
    if pgrid is not None:
        pg = (ctypes.c_int * 3)(*(list(pgrid) + [1] * (3 - len(pgrid))))
    out = _vp()
    _check(lib.sdrt_mesh_create(et, p, _i3(*N3), _d3(*lo3), _d3(*hi3), _i3(*per), rank, nranks, pg,
                                ctypes.byref(out)))
    return out


def mesh_info(m):
    info = MeshInfo()
    _check(lib.sdrt_mesh_info(m, ctypes.byref(info)))
    d = {k: getattr(info, k) for k, _ in MeshInfo._fields_}
    for k in ("N", "Nglobal", "offset"):
        d[k] = list(d[k])
    return d


def mesh_export_maps(m):
    info = mesh_info(m)
    F, K, nf, nfp = info["n_faces"], info["K"], info["nfaces"], info["nfp"]
    fe = np.zeros((F, 2), dtype=np.int32)
    fl = np.zeros((F, 2), dtype=np.int8)
    fp = np.zeros((F, nfp), dtype=np.int16)
    il = np.zeros((K, nf), dtype=np.uint8)
    _check(lib.sdrt_mesh_export_maps(m, fe.ctypes.data, fl.ctypes.data, fp.ctypes.data, il.ctypes.data))
    return fe, fl, fp, il


def mesh_sol_coords(m):
    info = mesh_info(m)
    x = np.zeros((info["nsol"], info["nd"], info["K"]))
    _check(lib.sdrt_mesh_sol_coords(m, x.ctypes.data))
    return x


def mesh_detj(m):
    info = mesh_info(m)
    x = np.zeros(info["K"])
    _check(lib.sdrt_mesh_detj(m, x.ctypes.data))
    return x


def mesh_set_halo(m, force_self_halo):
    _check(lib.sdrt_mesh_set_halo(m, int(bool(force_self_halo))))


def mesh_halo_lists(m):
    """[(peer, d, side, send_row, send_col, recv_row, recv_col)] per slab (numpy int32)."""
    cnt = ctypes.c_int64()
    _check(lib.sdrt_mesh_halo_lists(m, -1, None, None, None, ctypes.byref(cnt), None, None, None, None))
    out = []
    for i in range(cnt.value):
        peer, d, side, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check(lib.sdrt_mesh_halo_lists(m, i, ctypes.byref(peer), ctypes.byref(d), ctypes.byref(side),
                                        ctypes.byref(n), None, None, None, None))
        a = [np.zeros(n.value, dtype=np.int32) for _ in range(4)]
        _check(lib.sdrt_mesh_halo_lists(m, i, None, None, None, ctypes.byref(n), *[x.ctypes.data for x in a]))
        out.append((peer.value, d.value, side.value, *a))
    return out


def mesh_neighbor(m, e, f):
    """(trace column, neighbour local face) the kernels use across face f of local element e."""
    col, face = ctypes.c_int64(), ctypes.c_int()
    _check(lib.sdrt_mesh_neighbor(m, int(e), int(f), ctypes.byref(col), ctypes.byref(face)))
    return col.value, face.value


def mesh_destroy(m):
    lib.sdrt_mesh_destroy(m)


# ------------------------------------------------------------------ operators
SCHEMES = {"sdrt": 0, "frsdrt": 1, "frdg": 2}


def operators_build(etype, p, scheme=0):
    scheme = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
    et = ETYPES[etype] if isinstance(etype, str) else int(etype)
    out = _vp()
    _check(lib.sdrt_operators_build(et, p, scheme, ctypes.byref(out)))
    return out


def operators_get(o, name):
    r, c = ctypes.c_int(), ctypes.c_int()
    _check(lib.sdrt_operators_get(o, name.encode(), None, ctypes.byref(r), ctypes.byref(c)))
    a = np.zeros((r.value, c.value))
    _check(lib.sdrt_operators_get(o, name.encode(), a.ctypes.data, ctypes.byref(r), ctypes.byref(c)))
    return a


def operators_destroy(o):
    lib.sdrt_operators_destroy(o)


# ------------------------------------------------------------------ contexts
def physics(eq, c=(0.0, 0.0, 0.0), mu=0.0, gamma=1.4, Pr=0.71, beta=0.0, eta=0.0):
    cc = list(c) + [0.0] * (3 - len(c))
    return PhysicsT(EQS[eq] if isinstance(eq, str) else int(eq), _d3(*cc), mu, gamma, Pr, beta, eta)


def ctx_workspace_bytes(m, o, ph):
    return lib.sdrt_ctx_workspace_bytes(m, o, ctypes.byref(ph))


def ctx_create(m, o, ph, ws_ptr, ws_bytes, stream):
    out = _vp()
    _check(lib.sdrt_ctx_create(m, o, ctypes.byref(ph), _vp(ws_ptr), ws_bytes, _vp(stream), ctypes.byref(out)))
    return out


def residual(ctx, U_ptr, dUdt_ptr, stream):
    _check(lib.sdrt_residual(ctx, _vp(U_ptr), _vp(dUdt_ptr), _vp(stream)))


def ctx_set_farfield(ctx, state, stream):
    """Far-field exterior state (N_V conserved values, host) of the non-periodic axes."""
    st = np.ascontiguousarray(np.asarray(state, dtype=np.float64))
    _check(lib.sdrt_ctx_set_farfield(ctx, st.ctypes.data, _vp(stream)))


def comm_unique_id():
    """128-byte NCCL unique id (rank 0; broadcast it to the other ranks)."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.sdrt_comm_unique_id(buf))
    return bytes(buf)


def ctx_attach_comm(ctx, uid, rank, nranks):
    buf = (ctypes.c_uint8 * 128)(*uid)
    _check(lib.sdrt_ctx_attach_comm(ctx, buf, int(rank), int(nranks)))


def face_flux(ctx, U_ptr, dUdt_ptr, F_ptr, stream):
    _check(lib.sdrt_face_flux(ctx, _vp(U_ptr), _vp(dUdt_ptr), _vp(F_ptr), _vp(stream)))


def rk_step(ctx, U_ptr, dt, nsteps, check_every=0, stream=0):
    _check(lib.sdrt_rk_step(ctx, _vp(U_ptr), float(dt), int(nsteps), int(check_every), _vp(stream)))


def ctx_set_timing(ctx, enable):
    _check(lib.sdrt_ctx_set_timing(ctx, int(bool(enable))))


def ctx_set_graph(ctx, mode):
    _check(lib.sdrt_ctx_set_graph(ctx, int(mode)))


def ctx_kernel_times(ctx, max_tags=32):
    """{kernel name: (total device ms, launches)} since timing was enabled / last read."""
    names = ctypes.create_string_buffer(64 * max_tags)
    ms = np.zeros(max_tags)
    cnt = np.zeros(max_tags, dtype=np.int64)
    n = ctypes.c_int()
    _check(lib.sdrt_ctx_kernel_times(ctx, max_tags, names, ms.ctypes.data, cnt.ctypes.data, ctypes.byref(n)))
    raw = names.raw
    out = {}
    for t in range(n.value):
        nm = raw[64 * t: 64 * t + 64].split(b"\0", 1)[0].decode()
        if cnt[t]:
            out[nm] = (float(ms[t]), int(cnt[t]))
    return out


def halo_info(ctx):
    n = ctypes.c_int()
    peer, d, side = (ctypes.c_int * 6)(), (ctypes.c_int * 6)(), (ctypes.c_int * 6)()
    off = (ctypes.c_int64 * 7)()
    _check(lib.sdrt_halo_info(ctx, ctypes.byref(n), peer, d, side, off))
    k = n.value
    return list(peer[:k]), list(d[:k]), list(side[:k]), list(off[:k + 1])


def halo_pack(ctx, which, send_ptr, stream):
    _check(lib.sdrt_halo_pack(ctx, int(which), _vp(send_ptr), _vp(stream)))


def halo_unpack(ctx, which, recv_ptr, stream):
    _check(lib.sdrt_halo_unpack(ctx, int(which), _vp(recv_ptr), _vp(stream)))


def stage_traces(ctx, U_ptr, stream):
    _check(lib.sdrt_stage_traces(ctx, _vp(U_ptr), _vp(stream)))


def rk54_step(ctx, U_ptr, dt, nsteps, check_every, stream):
    _check(lib.sdrt_rk54_step(ctx, _vp(U_ptr), float(dt), int(nsteps), int(check_every), _vp(stream)))


RK54_STAGE0 = 10  # staged-API stage code of RK54 stage 0 (include/sdrt.h)


def diagnostics(ctx, U_ptr, out_ptr, stream):
    _check(lib.sdrt_diagnostics(ctx, _vp(U_ptr), _vp(out_ptr), _vp(stream)))


def diagnostics_rule(ctx, degree):
    _check(lib.sdrt_diagnostics_rule(ctx, int(degree)))


def stage_grad(ctx, U_ptr, stage, stream):
    _check(lib.sdrt_stage_grad(ctx, _vp(U_ptr), int(stage), _vp(stream)))


def stage_flux(ctx, U_ptr, stage, dt, out_ptr, stream):
    _check(lib.sdrt_stage_flux(ctx, _vp(U_ptr), int(stage), float(dt), _vp(out_ptr), _vp(stream)))


def stage_grad_part(ctx, U_ptr, stage, part, stream):
    _check(lib.sdrt_stage_grad_part(ctx, _vp(U_ptr), int(stage), int(part), _vp(stream)))


def stage_flux_part(ctx, U_ptr, stage, dt, out_ptr, part, stream):
    _check(lib.sdrt_stage_flux_part(ctx, _vp(U_ptr), int(stage), float(dt), _vp(out_ptr), int(part),
                                    _vp(stream)))


def ctx_last_launches(ctx):
    return lib.sdrt_ctx_last_launches(ctx)


def ctx_destroy(ctx):
    lib.sdrt_ctx_destroy(ctx)
