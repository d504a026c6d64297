"""Thin ctypes binding of include/chordal_sdp.h (argument marshalling only).

Every step of the ADMM iteration and of the PSD projection runs in the CUDA
library libchordal_sdp.so.  There is no Python or CPU fallback: if the library
is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libchordal_sdp.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_1609_06068_b200.build` "
        "(or __graft_entry__.build()); there is no CPU fallback")

def _torch_nccl():
    """Path of the NCCL bundled with torch (nvidia-nccl wheel), without importing torch."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


if "SDP_NCCL_LIB" not in os.environ and _torch_nccl():
    os.environ["SDP_NCCL_LIB"] = _torch_nccl()
lib = C.CDLL(LIB_PATH)

SDP_OK, SDP_MAX_ITER = 0, 1
SDP_E = {-1: "SDP_E_INVALID_ARG", -2: "SDP_E_RANK_DEFICIENT", -3: "SDP_E_CUDA", -4: "SDP_E_NCCL",
         -5: "SDP_E_OOM", -6: "SDP_E_NUMERICAL", -7: "SDP_E_STATE"}
FORM = {"primal": 0, "dual": 1}
SDP_A_COO, SDP_A_DENSE = 0, 1
VEC_X, VEC_Y, VEC_XMAT, VEC_SDP_X, VEC_SDP_Y = 0, 1, 2, 3, 4
BLK_XK, BLK_LAMBDA, BLK_VK, BLK_SDP_Z = 0, 1, 2, 3
SDP_MAX_K = 1024


class SdpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{SDP_E.get(code, code)}: {msg}")
        self.code = code


class sdp_problem(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32),
                ("c_nnz", C.c_int64), ("c_row", C.c_void_p), ("c_col", C.c_void_p), ("c_val", C.c_void_p),
                ("a_fmt", C.c_int32), ("a_nnz", C.c_int64), ("a_con", C.c_void_p), ("a_row", C.c_void_p),
                ("a_col", C.c_void_p), ("a_val", C.c_void_p), ("b", C.c_void_p),
                ("e_nnz", C.c_int64), ("e_row", C.c_void_p), ("e_col", C.c_void_p)]


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_int32)


class sdp_allocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", C.c_void_p)]


class sdp_options(C.Structure):
    _fields_ = [("form", C.c_int32), ("rho", C.c_double), ("device", C.c_int32), ("stream", C.c_void_p),
                ("check_every", C.c_int32), ("use_graph", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_id", C.c_void_p), ("adapt_rho", C.c_int32), ("adapt_mu", C.c_double),
                ("adapt_tau", C.c_double), ("allocator", C.POINTER(sdp_allocator)), ("comm", C.c_void_p)]


class sdp_info(C.Structure):
    _fields_ = [("iters", C.c_int64), ("eps_p", C.c_double), ("eps_d", C.c_double), ("objective", C.c_double),
                ("setup_s", C.c_double), ("n", C.c_int64), ("m", C.c_int64), ("N", C.c_int64), ("p", C.c_int64),
                ("kmin", C.c_int64), ("kmax", C.c_int64), ("stot", C.c_int64), ("form", C.c_int32),
                ("s_diagonal", C.c_int32), ("jacobi_capped", C.c_int64),
                ("launches_per_iter", C.c_int32), ("jacobi_sweeps", C.c_int64), ("rho", C.c_double),
                ("pipelined", C.c_int32), ("s_factor", C.c_int32), ("nnz_l", C.c_int64),
                ("fused", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_sig = {
    "sdp_default_options": (None, [C.POINTER(sdp_options)]),
    "sdp_setup": (_i32, [C.POINTER(sdp_problem), C.POINTER(sdp_options), C.POINTER(_vp)]),
    "sdp_step": (_i32, [_vp, _i32]),
    "sdp_solve": (_i32, [_vp, _i32, _d, C.POINTER(sdp_info)]),
    "sdp_reset": (_i32, [_vp]),
    "sdp_set_rho": (_i32, [_vp, _d]),
    "sdp_get_info": (_i32, [_vp, C.POINTER(sdp_info)]),
    "sdp_get_vector": (_i32, [_vp, _i32, _vp]),
    "sdp_get_blocks": (_i32, [_vp, _i32, _vp]),
    "sdp_get_pattern": (_i32, [_vp, _vp, _vp]),
    "sdp_get_cliques": (_i32, [_vp, _vp, _vp]),
    "sdp_get_history": (_i32, [_vp, _vp, _i64, C.POINTER(_i64)]),
    "sdp_complete_x": (_i32, [_vp, _d, _vp]),
    "sdp_get_elimination_order": (_i32, [_vp, _vp]),
    "sdp_destroy": (_i32, [_vp]),
    "sdp_workspace_bytes": (_i32, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    "sdp_loopback_create": (_i32, [_i32, _i32, C.POINTER(_vp)]),
    "sdp_loopback_destroy": (_i32, [_vp]),
    "sdp_psd_plan_create_ex": (_i32, [_i64, _vp, _i32, C.POINTER(sdp_allocator), C.POINTER(_vp)]),
    "sdp_state_bytes": (_i32, [_vp, C.POINTER(_i64)]),
    "sdp_save_state": (_i32, [_vp, _vp, _i64]),
    "sdp_load_state": (_i32, [_vp, _vp, _i64]),
    "sdp_profile_phases": (_i32, [_vp, _i32, _vp]),
    "sdp_chordal_cliques": (_i32, [_i32, _i64, _vp, _vp, C.POINTER(_i32), _vp, _i64, _vp, C.POINTER(_i64),
                                   C.POINTER(_i64)]),
    "sdp_psd_plan_create": (_i32, [_i64, _vp, _i32, C.POINTER(_vp)]),
    "sdp_project_psd_batch": (_i32, [_vp, _vp, _vp, _vp]),
    "sdp_project_psd_batch_host": (_i32, [_vp, _vp, _vp, _vp]),
    "sdp_psd_plan_values": (_i64, [_vp]),
    "sdp_psd_plan_launches": (_i32, [_vp]),
    "sdp_psd_plan_destroy": (_i32, [_vp]),
    "sdp_nccl_unique_id": (_i32, [_vp]),
    "sdp_shard_plan": (_i32, [_i32, _i64, _vp, _vp, _i32, _i32, _vp, C.POINTER(_i64), _vp, _vp, C.POINTER(_i64), _vp,
                              _i64]),
    "sdp_schur_inverse_host": (_i32, [_i32, _vp, _vp, _vp, _i32, _vp, C.POINTER(_i64)]),
    "sdp_last_error": (C.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


def _check(rc):
    if rc < 0:
        raise SdpError(rc, lib.sdp_last_error().decode())
    return rc


def _arr(a, dtype):
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)  # torch.cuda.Stream


def chordal_cliques(n, row, col):
    """sdp_chordal_cliques: (list of clique vertex arrays, fill edge count)."""
    row = _arr(row, np.int32)
    col = _arr(col, np.int32)
    p = C.c_int32()
    nv = C.c_int64()
    fill = C.c_int64()
    sizes = np.zeros(n, np.int32)
    cap = int(n) * 64
    while True:
        verts = np.zeros(cap, np.int32)
        rc = lib.sdp_chordal_cliques(n, row.size, _ptr(row), _ptr(col), C.byref(p), _ptr(sizes), cap,
                                     _ptr(verts), C.byref(nv), C.byref(fill))
        if rc < 0 and nv.value > cap:
            cap = int(nv.value)
            continue
        _check(rc)
        break
    out, e = [], 0
    for k in sizes[:p.value]:
        out.append(verts[e:e + k].copy())
        e += k
    return out, int(fill.value)


def schur_inverse_host(S, force_sparse=True):
    """sdp_schur_inverse_host: S^-1 of a sparse SPD matrix (scipy sparse or dense) through the
    library's sparse Cholesky; returns (S^-1 dense, nnz of the factor)."""
    import scipy.sparse as sp
    A = sp.csr_matrix(S)
    A.sort_indices()
    m = A.shape[0]
    ptr = _arr(A.indptr, np.int64)
    idx = _arr(A.indices, np.int32)
    val = _arr(A.data, np.float64)
    out = np.empty((m, m))
    nnz = C.c_int64()
    _check(lib.sdp_schur_inverse_host(m, _ptr(ptr), _ptr(idx), _ptr(val), int(bool(force_sparse)), _ptr(out),
                                      C.byref(nnz)))
    return out, int(nnz.value)


def nccl_unique_id():
    """128-byte NCCL id (bytes) for sharded handles (call on rank 0, broadcast)."""
    buf = C.create_string_buffer(128)
    _check(lib.sdp_nccl_unique_id(buf))
    return buf.raw


def shard_plan(n, row, col, world, rank):
    """sdp_shard_plan: dict(clique_rank, cliques (this rank's, ascending), local_coords, owned,
    shared_coords)."""
    row = _arr(row, np.int32)
    col = _arr(col, np.int32)
    cap = max(16, int(n) * int(n))
    cap = min(cap, 1 << 26)
    crank = np.zeros(cap, np.int32)
    loc = np.zeros(cap, np.int32)
    own = np.zeros(cap, np.uint8)
    shr = np.zeros(cap, np.int32)
    nl = C.c_int64()
    ns = C.c_int64()
    _check(lib.sdp_shard_plan(n, row.size, _ptr(row), _ptr(col), world, rank, _ptr(crank), C.byref(nl), _ptr(loc),
                              _ptr(own), C.byref(ns), _ptr(shr), cap))
    p = len(chordal_cliques(n, row, col)[0])
    cr = crank[:p].copy()
    return {"clique_rank": cr, "cliques": np.flatnonzero(cr == rank), "local_coords": loc[:nl.value].copy(),
            "owned": own[:nl.value].astype(bool), "shared_coords": shr[:ns.value].copy()}


class TorchAllocator:
    """sdp_allocator backed by torch uint8 tensors: PyTorch's caching allocator owns every
    device byte of the handles / plans that use it (include/chordal_sdp.h, sdp_allocator)."""

    def __init__(self):
        import torch
        self._torch = torch
        self.live = {}

        def _alloc(ctx, nbytes, device):
            try:
                t = self._torch.empty(int(nbytes), dtype=self._torch.uint8, device=f"cuda:{int(device)}")
            except Exception:  # noqa: BLE001  (OOM -> NULL -> SDP_E_OOM)
                return None
            self.live[t.data_ptr()] = t
            return t.data_ptr()

        def _free(ctx, ptr, device):
            self.live.pop(int(ptr), None)

        self._cb = (_ALLOC_FN(_alloc), _FREE_FN(_free))
        self.struct = sdp_allocator(self._cb[0], self._cb[1], None)

    def bytes_held(self):
        return sum(t.numel() for t in self.live.values())


class LoopbackGroup:
    """sdp_loopback_create: an in-process group of `world` sharded handles (one host thread
    per rank, collective calls) -- runs the clique-sharded device path on one GPU."""

    def __init__(self, world, device=0):
        h = C.c_void_p()
        _check(lib.sdp_loopback_create(int(world), int(device), C.byref(h)))
        self.h, self.world = h, int(world)

    def close(self):
        if getattr(self, "h", None):
            lib.sdp_loopback_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """Handle of sdp_setup().  `prob` needs the attributes n, m, c_row, c_col,
    c_val, b, a_fmt ("coo" | "dense"), a_con, a_row, a_col, a_val (optional e_row,
    e_col: the user pattern E).  allocator: None (cudaMalloc), "torch" or a
    TorchAllocator.  comm: a LoopbackGroup for world > 1 inside one process."""

    def __init__(self, prob, form="primal", rho=1.0, device=0, stream=None, use_graph=True, check_every=10,
                 rank=0, world=1, nccl_id=None, adapt_rho=False, adapt_mu=10.0, adapt_tau=2.0, allocator=None,
                 comm=None):
        self.form = form
        self.allocator = TorchAllocator() if allocator == "torch" else allocator
        self.comm = comm
        keep = []

        def k(a, dt):
            a = _arr(a, dt)
            keep.append(a)
            return a

        P = sdp_problem()
        P.n, P.m = int(prob.n), int(prob.m)
        cr, cc, cv = k(prob.c_row, np.int32), k(prob.c_col, np.int32), k(prob.c_val, np.float64)
        P.c_nnz, P.c_row, P.c_col, P.c_val = cr.size, _ptr(cr), _ptr(cc), _ptr(cv)
        ar, ac, av = k(prob.a_row, np.int32), k(prob.a_col, np.int32), k(prob.a_val, np.float64)
        if prob.a_fmt == "dense":
            P.a_fmt, P.a_nnz, P.a_con = SDP_A_DENSE, ar.size, None
        else:
            acon = k(prob.a_con, np.int32)
            P.a_fmt, P.a_nnz, P.a_con = SDP_A_COO, ar.size, _ptr(acon)
        P.a_row, P.a_col, P.a_val = _ptr(ar), _ptr(ac), _ptr(av)
        bb = k(prob.b, np.float64)
        P.b = _ptr(bb)
        if getattr(prob, "e_row", None) is not None:
            er, ec = k(prob.e_row, np.int32), k(prob.e_col, np.int32)
            P.e_nnz, P.e_row, P.e_col = er.size, _ptr(er), _ptr(ec)
        else:
            P.e_nnz, P.e_row, P.e_col = 0, None, None
        O = sdp_options()
        lib.sdp_default_options(C.byref(O))
        O.form, O.rho, O.device = FORM[form], float(rho), int(device)
        O.stream = _stream_ptr(stream)
        O.use_graph = int(bool(use_graph))
        O.check_every = int(check_every)
        O.adapt_rho = 1 if adapt_rho else 0
        O.adapt_mu, O.adapt_tau = float(adapt_mu), float(adapt_tau)
        O.rank, O.world = int(rank), int(world)
        self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        O.nccl_id = C.cast(self._nccl_id, C.c_void_p) if self._nccl_id is not None else None
        if self.allocator is not None:
            O.allocator = C.pointer(self.allocator.struct)
        O.comm = comm.h if comm is not None else None
        h = C.c_void_p()
        _check(lib.sdp_setup(C.byref(P), C.byref(O), C.byref(h)))
        self.h = h
        self._info = self.info()

    # --- iteration -------------------------------------------------------
    def step(self, iters):
        _check(lib.sdp_step(self.h, int(iters)))

    def solve(self, max_iters, tol):
        info = sdp_info()
        rc = _check(lib.sdp_solve(self.h, int(max_iters), float(tol), C.byref(info)))
        return ("solved" if rc == SDP_OK else "max_iter"), info.as_dict()

    def reset(self):
        _check(lib.sdp_reset(self.h))

    def set_rho(self, rho):
        _check(lib.sdp_set_rho(self.h, float(rho)))

    def save_state(self) -> bytes:
        """Checkpoint of the device-resident ADMM state (sdp_save_state)."""
        n = C.c_int64()
        _check(lib.sdp_state_bytes(self.h, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(lib.sdp_save_state(self.h, buf, n.value))
        return buf.raw

    def load_state(self, blob: bytes):
        """Resume from a save_state() blob of the same problem, form and sharding."""
        buf = C.create_string_buffer(bytes(blob), len(blob))
        _check(lib.sdp_load_state(self.h, buf, len(blob)))

    def info(self):
        info = sdp_info()
        _check(lib.sdp_get_info(self.h, C.byref(info)))
        return info.as_dict()

    # --- getters ----------------------------------------------------------
    @property
    def N(self):
        return self._info["N"]

    def _vec(self, which, n):
        out = np.empty(n)
        _check(lib.sdp_get_vector(self.h, which, _ptr(out)))
        return out

    def x(self):
        return self._vec(VEC_X, self._info["N"])

    def x_mat(self):
        return self._vec(VEC_XMAT, self._info["N"])

    def y(self):
        return self._vec(VEC_Y, self._info["m"])

    # the primal-dual SDP pair carried by the iterates (Remark 1; header: SDP_VEC_SDP_X)
    def sdp_x(self):
        """Unscaled entries X_ij of the SDP primal X on the pattern (canonical order)."""
        return self._vec(VEC_SDP_X, self._info["N"])

    def sdp_y(self):
        """The SDP dual multipliers yhat."""
        return self._vec(VEC_SDP_Y, self._info["m"])

    def sdp_z(self):
        """Stacked svec Agler blocks Z_k of the SDP dual slack (Theorem 2)."""
        return self.blocks("sdp_z")

    def workspace_bytes(self):
        live, peak = C.c_int64(), C.c_int64()
        _check(lib.sdp_workspace_bytes(self.h, C.byref(live), C.byref(peak)))
        return int(live.value), int(peak.value)

    def blocks(self, which):
        idx = {"xk": BLK_XK, "zk": BLK_XK, "lambda": BLK_LAMBDA, "vk": BLK_VK, "sdp_z": BLK_SDP_Z}[which]
        out = np.empty(self._info["stot"])
        _check(lib.sdp_get_blocks(self.h, idx, _ptr(out)))
        return out

    def pattern(self):
        r = np.empty(self._info["N"], np.int32)
        c = np.empty(self._info["N"], np.int32)
        _check(lib.sdp_get_pattern(self.h, _ptr(r), _ptr(c)))
        return r, c

    def cliques(self):
        p = self._info["p"]
        sizes = np.empty(p, np.int32)
        # total vertices = sum of sizes; sizes unknown before the call: query twice
        verts = np.empty(int(self._info["kmax"]) * p, np.int32)
        _check(lib.sdp_get_cliques(self.h, _ptr(sizes), _ptr(verts)))
        out, e = [], 0
        for k in sizes:
            out.append(verts[e:e + k].copy())
            e += k
        return out

    def complete_x(self, rtol=1e-8):
        """PSD completion of X = smat(x) off the chordal pattern (sdp_complete_x), n x n."""
        n = self._info["n"]
        out = np.empty((n, n))
        _check(lib.sdp_complete_x(self.h, float(rtol), _ptr(out)))
        return out

    def elimination_order(self):
        n = self._info["n"]
        out = np.empty(n, dtype=np.int32)
        _check(lib.sdp_get_elimination_order(self.h, _ptr(out)))
        return out

    def history(self, cap=1 << 20):
        out = np.empty(3 * cap)
        rows = C.c_int64()
        _check(lib.sdp_get_history(self.h, _ptr(out), cap, C.byref(rows)))
        return out[:3 * rows.value].reshape(rows.value, 3)

    PHASES = ("gemv", "kkt_small", "gemvT", "projection", "scatter", "dual_update", "finalize")

    def profile_phases(self, iters):
        out = np.zeros(len(self.PHASES))
        _check(lib.sdp_profile_phases(self.h, int(iters), _ptr(out)))
        return dict(zip(self.PHASES, out.tolist()))

    def close(self):
        if getattr(self, "h", None):
            lib.sdp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PsdPlan:
    """sdp_psd_plan_create / sdp_project_psd_batch (packed upper, unscaled)."""

    def __init__(self, sizes, device=0, allocator=None):
        self.sizes = _arr(sizes, np.int32)
        self.device = int(device)
        self.allocator = TorchAllocator() if allocator == "torch" else allocator
        h = C.c_void_p()
        al = C.pointer(self.allocator.struct) if self.allocator is not None else None
        _check(lib.sdp_psd_plan_create_ex(self.sizes.size, _ptr(self.sizes), self.device, al, C.byref(h)))
        self.h = h
        self.values = int(lib.sdp_psd_plan_values(h))
        self.launches = int(lib.sdp_psd_plan_launches(h))

    def _dev(self, t, name):
        """Device pointer of an int (trusted) or a torch tensor (checked: CUDA, float64, contiguous,
        at least plan.values elements)."""
        if isinstance(t, int):
            return t
        if not (t.is_cuda and t.dtype.is_floating_point and t.element_size() == 8 and t.is_contiguous()):
            raise ValueError(f"{name}: need a contiguous float64 CUDA tensor")
        if t.numel() < self.values:
            raise ValueError(f"{name}: {t.numel()} elements < plan.values = {self.values}")
        return int(t.data_ptr())

    def project(self, d_in, d_out, stream=None):
        """d_in, d_out: device pointers (int) or torch CUDA float64 tensors."""
        pin, pout = self._dev(d_in, "d_in"), self._dev(d_out, "d_out")
        _check(lib.sdp_project_psd_batch(self.h, pin, pout, _stream_ptr(stream)))

    def project_host(self, h_in, h_out=None, stream=None):
        h_in = _arr(h_in, np.float64).reshape(-1)
        if h_in.size != self.values:
            raise ValueError(f"h_in has {h_in.size} values, the plan needs {self.values}")
        if h_out is None:
            h_out = np.empty_like(h_in)
        if not (isinstance(h_out, np.ndarray) and h_out.dtype == np.float64 and h_out.flags.c_contiguous
                and h_out.size == self.values):
            raise ValueError("h_out must be a C-contiguous float64 array of plan.values elements")
        _check(lib.sdp_project_psd_batch_host(self.h, _ptr(h_in), h_out.ctypes.data_as(C.c_void_p),
                                              _stream_ptr(stream)))
        return h_out

    def close(self):
        if getattr(self, "h", None):
            lib.sdp_psd_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
