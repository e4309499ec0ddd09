"""ctypes binding of libpfcs.so (include/pfcs.h) and the device plumbing.

This module is the only place that touches the C ABI.  It fails loudly:
there is no CPU fallback anywhere in the product path — if the library is
missing or no CUDA device is present every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PFCS_LIB_PATH", str(_HERE / "libpfcs.so")))

PFCS_OK = 0
PFCS_E_ARG = 1
PFCS_E_CUDA = 2
PFCS_E_UNSUPPORTED = 3
PFCS_E_NONFINITE = 4
DIAG_SLOTS = 64
DIAG_VALS = 4

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_p = ctypes.c_void_p
_c_d = ctypes.c_double

# symbol -> argtypes (every function returns int unless listed in _RESTYPE)
_SIGS = {
    "pfcs_version": [],
    "pfcs_last_error": [],
    "pfcs_device_count": [ctypes.POINTER(_c_int)],
    "pfcs_fft_axis_c2c": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_p],
    "pfcs_fft_axis_c2c_pro": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_int, _c_p, _c_int, _c_p],
    "pfcs_plan_create": [_c_i64, _c_i64, _c_i64, _c_p],
    "pfcs_plan_destroy": [_c_p],
    "pfcs_plan_fwd": [_c_p, _c_p, _c_p, _c_p],
    "pfcs_plan_inv": [_c_p, _c_p, _c_p, _c_p, _c_p],
    "pfcs_plan_pfc_steps": [_c_p, _c_p, _c_p, _c_p, _c_p, _c_d, _c_d, _c_i64, _c_p, _c_p, _c_p],
    "pfcs_plan_spectral_elems": [_c_p],
    "pfcs_fft_zlines": [_c_p, _c_p, _c_i64, _c_i64, _c_int, _c_int, _c_int, _c_p],
    "pfcs_fft_lines": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_int, _c_p],
    "pfcs_fft_zlines_to": [_c_p, _c_p, _c_i64, _c_i64, _c_int, _c_int, _c_int, _c_p],
    "pfcs_fft_lines_scatter": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_int, _c_p],
    "pfcs_pfc_update_z_to": [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_p, _c_p, _c_p,
                             _c_d, _c_d, _c_p, _c_p],
    "pfcs_enable_peer_access": [_c_int],
    "pfcs_malloc": [_c_i64, ctypes.POINTER(_c_p)],
    "pfcs_free": [_c_p],
    "pfcs_ipc_get_handle": [_c_p, _c_p],
    "pfcs_ipc_open_handle": [_c_p, ctypes.POINTER(_c_p)],
    "pfcs_ipc_close": [_c_p],
    "pfcs_stream_sync": [_c_p],
    "pfcs_ipc_event_create": [ctypes.POINTER(_c_p), _c_p],
    "pfcs_ipc_event_open": [_c_p, ctypes.POINTER(_c_p)],
    "pfcs_event_record": [_c_p, _c_p],
    "pfcs_stream_wait_event": [_c_p, _c_p],
    "pfcs_event_destroy": [_c_p],
    "pfcs_rfft_x": [_c_p, _c_p, _c_i64, _c_i64, _c_p],
    "pfcs_irfft_x": [_c_p, _c_p, _c_i64, _c_i64, _c_p],
    "pfcs_rfft_x_pro": [_c_p, _c_p, _c_i64, _c_i64, _c_int, _c_p, _c_d, _c_p],
    "pfcs_xmul_x": [_c_p, _c_p, _c_i64, _c_i64, _c_p],
    "pfcs_xdot3_supported": [_c_i64, _c_i64],
    "pfcs_hydro_mu_z": [_c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_p],
    "pfcs_hydro_mu_zgrad": [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d,
                            _c_p],
    "pfcs_xdot3_x": [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_p, _c_p],
    "pfcs_pfc_cube_x": [_c_p, _c_i64, _c_i64, _c_int, _c_p, _c_p],
    "pfcs_pfc_update_z": [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_int,
                          _c_p, _c_p, _c_p, _c_d, _c_d, _c_p, _c_p],
    "pfcs_pfc_cube": [_c_p, _c_i64, _c_int, _c_p, _c_p],
    "pfcs_pfc_update": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d, _c_p, _c_p],
    "pfcs_mul_deriv": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_int, _c_p],
    "pfcs_cmul": [_c_p, _c_p, _c_p, _c_i64, _c_p],
    "pfcs_hydro_advect": [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p],
    "pfcs_hydro_psi_update": [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d,
                              _c_p, _c_p],
    "pfcs_hydro_mu": [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_p],
    "pfcs_hydro_vel_update": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                              _c_p, _c_p],
    "pfcs_ch_nonlin": [_c_p, _c_p, _c_i64, _c_d, _c_p],
    "pfcs_ch_update": [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                       _c_p, _c_p],
    "pfcs_ch_mu": [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_p],
    "pfcs_hydro_psi_update_to": [_c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d,
                                 _c_p, _c_p],
    "pfcs_hydro_vel_update_to": [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                                 _c_p, _c_p],
    "pfcs_ch_update_to": [_c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_d, _c_d,
                          _c_p, _c_p],
    "pfcs_add3": [_c_p, _c_p, _c_p, _c_p, _c_i64, _c_p],
    "pfcs_real_pointwise": [_c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_d, _c_p],
    "pfcs_update_zinv": [_c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p,
                         _c_d, _c_d, _c_d, _c_p, _c_p],
    "pfcs_update_zzinv": [_c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p,
                          _c_d, _c_d, _c_d, _c_int, _c_p, _c_p],
    "pfcs_axpy": [_c_p, _c_p, _c_p, _c_i64, _c_d, _c_p],
    "pfcs_energy_sum": [_c_p, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p],
    "pfcs_energy_scratch_bytes": [_c_i64],
    "pfcs_absmax": [_c_p, _c_i64, _c_i64, _c_p, _c_p],
    "pfcs_apply_op": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_d, _c_p],
}
_RESTYPE = {"pfcs_last_error": ctypes.c_char_p, "pfcs_energy_scratch_bytes": _c_i64,
            "pfcs_plan_spectral_elems": _c_i64}

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A libpfcs call failed (CUDA error or unsupported size)."""


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load(require_cuda: bool = True):
    """Load libpfcs.so (once).  Raises if it is absent or, by default, if
    no CUDA device is visible — there is no host fallback."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise NativeError(
                        f"{LIB_PATH} is missing: run __graft_entry__.build() "
                        "(nvcc, sm_100a) before using the CUDA path")
                lib = ctypes.CDLL(str(LIB_PATH))
                for name, args in _SIGS.items():
                    fn = getattr(lib, name)
                    fn.argtypes = args
                    fn.restype = _RESTYPE.get(name, _c_int)
                _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise NativeError("no CUDA device visible: the pfcspectral B200 path has no CPU fallback")
    return _lib


def last_error() -> str:
    msg = load(require_cuda=False).pfcs_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc == PFCS_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == PFCS_E_ARG:
        raise ValueError(msg)
    raise NativeError(msg)


# Launch accounting for bench.py: `launches` counts every kernel-launching
# call; when `trace` is a list, each call appends (name, start, end) CUDA
# events recorded on the current stream around the launch.
launches = 0
trace: list | None = None
_NO_LAUNCH = {"pfcs_version", "pfcs_last_error", "pfcs_device_count", "pfcs_energy_scratch_bytes",
              "pfcs_plan_create", "pfcs_plan_destroy", "pfcs_plan_spectral_elems", "pfcs_ipc_event_create",
              "pfcs_ipc_event_open", "pfcs_event_record", "pfcs_stream_wait_event", "pfcs_event_destroy",
              "pfcs_xdot3_supported"}


def call(name: str, *args) -> None:
    global launches
    fn = getattr(load(), name)
    if trace is not None and name not in _NO_LAUNCH:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        rc = fn(*args)
        b.record()
        trace.append((name, args, a, b))
    else:
        rc = fn(*args)
    if name not in _NO_LAUNCH:
        launches += 1
    check(rc, name)


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return t.data_ptr()
