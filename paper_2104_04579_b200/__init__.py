"""libboris Python binding: argument marshalling over the C ABI (include/libboris.h).

B200-native relativistic Boris particle pusher (arXiv 2104.04579).  Every step
of the push runs in the CUDA kernels of ``libboris.so``; this module only
converts Python/numpy/torch arguments to the C ABI's plain pointers and sizes,
and raises :class:`BorisError` on a non-OK status.  Function names are the C
names.  There is no CPU fallback: importing this package fails loudly if
``libboris.so`` has not been built (``python -m paper_2104_04579_b200._build``).

Pointers are passed as Python ints (``tensor.data_ptr()``); streams as ints
(``torch.cuda.current_stream().cuda_stream``) or ``None`` for the default stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libboris.so")

BORIS_OK = 0
BORIS_E_INVALID_ARG = 1
BORIS_E_OUT_OF_MEMORY = 2
BORIS_E_CUDA = 3
BORIS_E_TYPE_OUT_OF_RANGE = 4
BORIS_E_MISMATCH = 5
BORIS_E_UNSUPPORTED = 6
BORIS_E_NO_DEVICE = 7

BORIS_LAYOUT_AOS = 0
BORIS_LAYOUT_SOA = 1
BORIS_FP32 = 0
BORIS_FP64 = 1
BORIS_MEMORY_DEVICE = 0
BORIS_MEMORY_HOST = 1
BORIS_MAX_TYPES = 256
BORIS_MAX_PARTICLES = 1 << 40
BORIS_PUSH_AUTO = 0
BORIS_PUSH_STREAM_EACH_STEP = 1
BORIS_PUSH_PUSHER_BORIS = 0x00
BORIS_PUSH_PUSHER_VAY = 0x10
BORIS_PUSH_PUSHER_HIGUERA_CARY = 0x20
BORIS_PUSH_PUSHER_MASK = 0x30
BORIS_OPT_FUSED_GENERIC = 1
BORIS_OPT_MD_ORDER = 3
BORIS_OPT_HOST_CHUNK = 2
BORIS_AOS_RECORD_BYTES = {BORIS_FP32: 36, BORIS_FP64: 72}
BORIS_AOS_FIELD_BYTES = {BORIS_FP32: 24, BORIS_FP64: 48}

# Every symbol include/libboris.h declares (checked by tests/test_abi_cpu.py).
EXPORTED = (
    "boris_abi_version", "boris_status_string", "boris_last_error",
    "boris_set_option", "boris_get_option",
    "boris_ensemble_create", "boris_ensemble_wrap_soa", "boris_ensemble_wrap_aos",
    "boris_ensemble_destroy", "boris_ensemble_upload", "boris_ensemble_download",
    "boris_ensemble_validate_types", "boris_ensemble_get_info", "boris_ensemble_get_time",
    "boris_ensemble_set_time", "boris_field_create_arrays_soa", "boris_field_create_arrays_aos",
    "boris_field_create_uniform", "boris_field_create_plane_wave", "boris_field_create_mdipole",
    "boris_field_create_grid", "boris_ensemble_sort_by_cell", "boris_deposit_current",
    "boris_push_deposit",
    "boris_field_destroy", "boris_field_evaluate", "boris_push", "boris_push_diag", "boris_push_ex",
    "boris_kinetic_energy",
)


class BorisError(RuntimeError):
    def __init__(self, status: int, func: str, detail: str):
        self.status = status
        super().__init__(f"{func}: {_status_name(status)}: {detail}")


class boris_particle_type(ctypes.Structure):
    _fields_ = [("charge", ctypes.c_double), ("mass", ctypes.c_double)]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_d = ctypes.c_double
_dp = ctypes.POINTER(ctypes.c_double)
_i16p = ctypes.POINTER(ctypes.c_int16)
_tp = ctypes.POINTER(boris_particle_type)
_hp = ctypes.POINTER(ctypes.c_void_p)

_SIGNATURES = {
    "boris_abi_version": ([], _i32),
    "boris_status_string": ([_i32], ctypes.c_char_p),
    "boris_last_error": ([], ctypes.c_char_p),
    "boris_set_option": ([_i32, _i64], _i32),
    "boris_get_option": ([_i32, ctypes.POINTER(_i64)], _i32),
    "boris_ensemble_create": ([_i32, _i32, _i32, _i64, _tp, _i32, _d, _hp], _i32),
    "boris_ensemble_wrap_soa": ([_i32, _i32, _i32, _i64] + [_vp] * 9 + [_tp, _i32, _d, _hp], _i32),
    "boris_ensemble_wrap_aos": ([_i32, _i32, _i32, _i64, _vp, _tp, _i32, _d, _hp], _i32),
    "boris_ensemble_destroy": ([_vp], _i32),
    "boris_ensemble_upload": ([_vp, _i64, _i64, _dp, _dp, _dp, _i16p, _dp, _vp], _i32),
    "boris_ensemble_download": ([_vp, _i64, _i64, _dp, _dp, _dp, _dp, _i16p, _vp], _i32),
    "boris_ensemble_validate_types": ([_vp, _vp], _i32),
    "boris_ensemble_get_info": ([_vp] + [ctypes.POINTER(_i32)] * 2 + [ctypes.POINTER(_i64)]
                                + [ctypes.POINTER(_i32)] * 3, _i32),
    "boris_ensemble_get_time": ([_vp, _dp], _i32),
    "boris_ensemble_set_time": ([_vp, _d], _i32),
    "boris_field_create_arrays_soa": ([_vp] + [_vp] * 6 + [_hp], _i32),
    "boris_field_create_arrays_aos": ([_vp, _vp, _hp], _i32),
    "boris_field_create_uniform": ([_dp, _dp, _hp], _i32),
    "boris_field_create_plane_wave": ([_d, _dp, _dp, _d, _d, _d, _hp], _i32),
    "boris_field_create_mdipole": ([_d, _d, _d, _hp], _i32),
    "boris_field_destroy": ([_vp], _i32),
    "boris_field_create_grid": ([_i32, _i32, _i32, _i32, _i32, _dp, _dp] + [_vp] * 6 + [_hp], _i32),
    "boris_ensemble_sort_by_cell": ([_vp, _vp, _vp], _i32),
    "boris_deposit_current": ([_vp, _vp, _d, _vp, _vp, _vp, _vp], _i32),
    "boris_push_deposit": ([_vp, _vp, _d, _vp, _vp, _vp, _vp, _vp], _i32),
    "boris_field_evaluate": ([_vp, _vp, _d, _vp, _vp], _i32),
    "boris_push": ([_vp, _vp, _d, _i64, _vp], _i32),
    "boris_push_diag": ([_vp, _vp, _d, _i64, _vp, _vp], _i32),
    "boris_push_ex": ([_vp, _vp, _d, _i64, ctypes.c_uint32, _vp, _vp], _i32),
    "boris_kinetic_energy": ([_vp, _vp, _vp], _i32),
}

_lib = None


def load_library(path: str | None = None):
    """Load libboris.so (raises ImportError if it is missing: no fallback exists).
    LIBBORIS_PATH may point at a tuning variant built by `_build --tag`."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("LIBBORIS_PATH") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"libboris.so not found at {path}; build it with "
            "`python -m paper_2104_04579_b200._build` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _status_name(s: int) -> str:
    return load_library().boris_status_string(s).decode()


def _check(status: int, func: str):
    if status != BORIS_OK:
        raise BorisError(status, func, load_library().boris_last_error().decode())


def _types(types):
    arr = (boris_particle_type * len(types))()
    for i, (q, m) in enumerate(types):
        arr[i].charge = float(q)
        arr[i].mass = float(m)
    return arr, len(types)


def _stream(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return int(stream.cuda_stream)
    return int(stream)


def _dptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _f64(a, n3=None):
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------------------
# Library
# ---------------------------------------------------------------------------

def boris_abi_version() -> int:
    return int(load_library().boris_abi_version())


def boris_status_string(status: int) -> str:
    return _status_name(status)


def boris_last_error() -> str:
    return load_library().boris_last_error().decode()


def boris_set_option(option: int, value: int):
    _check(load_library().boris_set_option(option, value), "boris_set_option")


def boris_get_option(option: int) -> int:
    v = _i64()
    _check(load_library().boris_get_option(option, ctypes.byref(v)), "boris_get_option")
    return int(v.value)


# ---------------------------------------------------------------------------
# Ensembles
# ---------------------------------------------------------------------------

def boris_ensemble_create(device, layout, precision, n, types, light_velocity):
    t, nt = _types(types)
    h = ctypes.c_void_p()
    _check(load_library().boris_ensemble_create(device, layout, precision, n, t, nt,
                                                light_velocity, ctypes.byref(h)),
           "boris_ensemble_create")
    return h.value


def boris_ensemble_wrap_soa(device, memory, precision, n, x, y, z, px, py, pz, weight, gamma,
                            type_, types, light_velocity):
    t, nt = _types(types)
    h = ctypes.c_void_p()
    _check(load_library().boris_ensemble_wrap_soa(device, memory, precision, n, x, y, z, px, py,
                                                  pz, weight, gamma, type_, t, nt,
                                                  light_velocity, ctypes.byref(h)),
           "boris_ensemble_wrap_soa")
    return h.value


def boris_ensemble_wrap_aos(device, memory, precision, n, records, types, light_velocity):
    t, nt = _types(types)
    h = ctypes.c_void_p()
    _check(load_library().boris_ensemble_wrap_aos(device, memory, precision, n, records, t, nt,
                                                  light_velocity, ctypes.byref(h)),
           "boris_ensemble_wrap_aos")
    return h.value


def boris_ensemble_destroy(ens):
    _check(load_library().boris_ensemble_destroy(ens), "boris_ensemble_destroy")


def boris_ensemble_upload(ens, first, count, pos3, mom3, weight=None, type_=None, gamma=None,
                          stream=None):
    pos3, mom3, weight, gamma = _f64(pos3), _f64(mom3), _f64(weight), _f64(gamma)
    tp = None
    if type_ is not None:
        type_ = np.ascontiguousarray(np.asarray(type_, dtype=np.int16))
        tp = type_.ctypes.data_as(_i16p)
    _check(load_library().boris_ensemble_upload(ens, first, count, _dptr(pos3), _dptr(mom3),
                                                _dptr(weight), tp, _dptr(gamma),
                                                _stream(stream)),
           "boris_ensemble_upload")


def boris_ensemble_download(ens, first, count, stream=None):
    """Returns dict(pos (count,3), mom (count,3), weight, gamma, type) as numpy arrays."""
    pos = np.empty((count, 3))
    mom = np.empty((count, 3))
    w = np.empty(count)
    g = np.empty(count)
    ty = np.empty(count, np.int16)
    _check(load_library().boris_ensemble_download(ens, first, count, _dptr(pos), _dptr(mom),
                                                  _dptr(w), _dptr(g),
                                                  ty.ctypes.data_as(_i16p), _stream(stream)),
           "boris_ensemble_download")
    return {"pos": pos, "mom": mom, "weight": w, "gamma": g, "type": ty}


def boris_ensemble_validate_types(ens, stream=None):
    _check(load_library().boris_ensemble_validate_types(ens, _stream(stream)),
           "boris_ensemble_validate_types")


def boris_ensemble_get_info(ens):
    lay, prec, nt, dev, mem = (_i32() for _ in range(5))
    n = _i64()
    _check(load_library().boris_ensemble_get_info(ens, ctypes.byref(lay), ctypes.byref(prec),
                                                  ctypes.byref(n), ctypes.byref(nt),
                                                  ctypes.byref(dev), ctypes.byref(mem)),
           "boris_ensemble_get_info")
    return {"layout": lay.value, "precision": prec.value, "n": n.value, "n_types": nt.value,
            "device": dev.value, "memory": mem.value}


def boris_ensemble_get_time(ens) -> float:
    t = _d()
    _check(load_library().boris_ensemble_get_time(ens, ctypes.byref(t)), "boris_ensemble_get_time")
    return t.value


def boris_ensemble_set_time(ens, t):
    _check(load_library().boris_ensemble_set_time(ens, t), "boris_ensemble_set_time")


# ---------------------------------------------------------------------------
# Fields
# ---------------------------------------------------------------------------

def boris_field_create_arrays_soa(like, Ex, Ey, Ez, Bx, By, Bz):
    h = ctypes.c_void_p()
    _check(load_library().boris_field_create_arrays_soa(like, Ex, Ey, Ez, Bx, By, Bz,
                                                        ctypes.byref(h)),
           "boris_field_create_arrays_soa")
    return h.value


def boris_field_create_arrays_aos(like, records):
    h = ctypes.c_void_p()
    _check(load_library().boris_field_create_arrays_aos(like, records, ctypes.byref(h)),
           "boris_field_create_arrays_aos")
    return h.value


def boris_field_create_uniform(E, B):
    E = (ctypes.c_double * 3)(*[float(v) for v in E])
    B = (ctypes.c_double * 3)(*[float(v) for v in B])
    h = ctypes.c_void_p()
    _check(load_library().boris_field_create_uniform(E, B, ctypes.byref(h)),
           "boris_field_create_uniform")
    return h.value


def boris_field_create_plane_wave(E0, k_hat, e_hat, omega, k, phase0=0.0):
    kh = (ctypes.c_double * 3)(*[float(v) for v in k_hat])
    eh = (ctypes.c_double * 3)(*[float(v) for v in e_hat])
    h = ctypes.c_void_p()
    _check(load_library().boris_field_create_plane_wave(E0, kh, eh, omega, k, phase0,
                                                        ctypes.byref(h)),
           "boris_field_create_plane_wave")
    return h.value


def boris_field_create_mdipole(A0, omega0, k):
    h = ctypes.c_void_p()
    _check(load_library().boris_field_create_mdipole(A0, omega0, k, ctypes.byref(h)),
           "boris_field_create_mdipole")
    return h.value


def boris_field_create_grid(device, precision, nx, ny, nz, origin, spacing, Ex, Ey, Ez, Bx, By,
                            Bz):
    """Grid field (CIC gather); Ex..Bz are device pointers of nx*ny*nz FP (x fastest)."""
    org = (ctypes.c_double * 3)(*[float(v) for v in origin])
    sp = (ctypes.c_double * 3)(*[float(v) for v in spacing])
    h = ctypes.c_void_p()
    _check(load_library().boris_field_create_grid(device, precision, nx, ny, nz, org, sp, Ex, Ey,
                                                  Ez, Bx, By, Bz, ctypes.byref(h)),
           "boris_field_create_grid")
    return h.value


def boris_ensemble_sort_by_cell(ens, grid, stream=None):
    _check(load_library().boris_ensemble_sort_by_cell(ens, grid, _stream(stream)),
           "boris_ensemble_sort_by_cell")


def boris_deposit_current(ens, grid, dt, Jx, Jy, Jz, stream=None):
    """CIC current deposition at the half-step position into device arrays Jx..Jz."""
    _check(load_library().boris_deposit_current(ens, grid, dt, Jx, Jy, Jz, _stream(stream)),
           "boris_deposit_current")


def boris_push_deposit(ens, grid, dt, Jx, Jy, Jz, d_diag=None, stream=None):
    """One grid-gather push followed by the current deposition of the new state (fused)."""
    _check(load_library().boris_push_deposit(ens, grid, dt, Jx, Jy, Jz, d_diag, _stream(stream)),
           "boris_push_deposit")


def boris_field_destroy(field):
    _check(load_library().boris_field_destroy(field), "boris_field_destroy")


def boris_field_evaluate(analytic, ens, t, out, stream=None):
    _check(load_library().boris_field_evaluate(analytic, ens, t, out, _stream(stream)),
           "boris_field_evaluate")


# ---------------------------------------------------------------------------
# Push
# ---------------------------------------------------------------------------

def boris_push(ens, field, dt, n_steps, stream=None):
    _check(load_library().boris_push(ens, field, dt, n_steps, _stream(stream)), "boris_push")


def boris_push_diag(ens, field, dt, n_steps, d_diag, stream=None):
    _check(load_library().boris_push_diag(ens, field, dt, n_steps, d_diag, _stream(stream)),
           "boris_push_diag")


def boris_push_ex(ens, field, dt, n_steps, flags=BORIS_PUSH_AUTO, d_diag=None, stream=None):
    _check(load_library().boris_push_ex(ens, field, dt, n_steps, flags, d_diag, _stream(stream)),
           "boris_push_ex")


def boris_kinetic_energy(ens, d_diag, stream=None):
    _check(load_library().boris_kinetic_energy(ens, d_diag, _stream(stream)),
           "boris_kinetic_energy")
