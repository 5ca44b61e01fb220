"""ctypes binding of libsplat_b200.so (include/splat_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every entry point raises `RuntimeError` naming what is absent.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from .errors import ShapeMismatchError, ValidationError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsplat_b200.so")
# A/B experiments only: load another build of the same library (tools/ab.sh)
if os.environ.get("SB_LIB_VARIANT"):
    LIB_PATH = os.path.abspath(os.environ["SB_LIB_VARIANT"])

SB_OK, SB_EINVAL, SB_ECUDA, SB_EWORKSPACE, SB_ENODEVICE = 0, -1, -2, -3, -4

# exported symbols and their argtypes (all pointers are c_void_p)
VP, I64, I32, SZ = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
SIGNATURES = {
    "sb_last_error": ([], C.c_char_p),
    "sb_version": ([], C.c_int),
    "sb_record_bytes": ([], C.c_int),
    "sb_raster_row_bytes": ([], C.c_int),
    "sb_screen_grad_bytes": ([], C.c_int),
    "sb_morton_keys_workspace_bytes": ([I64], SZ),
    "sb_morton_keys": ([VP, I64, VP, VP, VP, VP, VP, SZ, VP], C.c_int),
    "sb_morton_encode": ([VP, I64, VP, VP, VP, VP], C.c_int),
    "sb_sort_workspace_bytes": ([I64], SZ),
    "sb_radix_sort_pairs_u64": ([VP, VP, VP, VP, I64, C.c_int, VP, VP, SZ, VP], C.c_int),
    "sb_permute_rows": ([VP, I64, C.c_int, VP, VP, VP, VP], C.c_int),
    "sb_project_workspace_bytes": ([I64], SZ),
    "sb_project_cull_compact": ([VP, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, SZ, VP], C.c_int),
    "sb_build_clusters": ([VP, I64, I32, VP, VP], C.c_int),
    "sb_cull_clusters": ([VP, I64, I32, I64, VP, VP, VP, VP, VP], C.c_int),
    "sb_bin_state_workspace_bytes": ([I64, I32], SZ),
    "sb_bin_prepare": ([VP, VP, I64, VP, VP, VP, VP, VP, SZ, VP], C.c_int),
    "sb_host_mapped_pointer": ([VP, C.POINTER(C.c_void_p)], C.c_int),
    "sb_bin_finish_workspace_bytes": ([I64, I32], SZ),
    "sb_bin_finish": ([VP, VP, I64, VP, I64, I64, VP, VP, VP, VP, SZ, VP], C.c_int),
    "sb_raster_workspace_bytes": ([], SZ),
    "sb_raster_fwd": ([VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, SZ, VP], C.c_int),
    "sb_raster_bwd_workspace_bytes": ([I32, I64, I64], SZ),
    "sb_raster_bwd": ([VP, VP, VP, VP, VP, VP, VP, VP, VP, VP, I64, I64, I64, VP, SZ, VP], C.c_int),
    "sb_chain_projection_bwd": ([VP, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP], C.c_int),
    "sb_chain_projection_bwd_accumulate": ([VP, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP], C.c_int),
    "sb_adam_sparse": ([VP, VP, VP, VP, VP, VP, I64, VP, VP], C.c_int),
    "sb_variance_score": ([VP, VP, VP, I64, VP, VP], C.c_int),
    "sb_densify_workspace_bytes": ([I64, I64], SZ),
    "sb_densify_select": ([VP, VP, I64, I64, C.c_double, VP, VP, VP, VP, VP, SZ, VP], C.c_int),
    "sb_densify_apply": ([VP, I64, VP, VP, I64, VP, I64, C.c_double, I32, VP, VP, VP, VP, VP, VP, SZ, VP], C.c_int),
    "sb_lane_reduce": ([VP, I64, C.c_int, VP, VP, VP], C.c_int),
    "sb_loss_workspace_bytes": ([I32, I32], SZ),
    "sb_loss_fwd_bwd": ([VP, VP, VP, I32, I32, C.c_float, VP, VP, VP, VP], C.c_int),
}


class SbCamera(C.Structure):
    _fields_ = [("w2c", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("near_plane", C.c_double),
                ("far_plane", C.c_double), ("planes", C.c_double * 24),
                ("width", C.c_int32), ("height", C.c_int32), ("pad_", C.c_int32 * 2)]


class SbRasterCfg(C.Structure):
    _fields_ = [("alpha_min", C.c_float), ("alpha_max", C.c_float), ("t_stop", C.c_float),
                ("background", C.c_float * 3), ("low_pass", C.c_float),
                ("use_culling", C.c_int32), ("conic_reduce", C.c_int32), ("half_state", C.c_int32),
                ("deterministic", C.c_int32)]


_lib = None
_lock = threading.Lock()


def load():
    """Load the library (raises RuntimeError if it is not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"libsplat_b200.so not found at {LIB_PATH}: build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
                lib = C.CDLL(LIB_PATH)
                for name, (args, res) in SIGNATURES.items():
                    f = getattr(lib, name)
                    f.argtypes = args
                    f.restype = res
                _lib = lib
    return _lib


def exported_symbols():
    return sorted(SIGNATURES)


_have_cuda = False


def require_cuda(t: torch.Tensor | None = None):
    global _have_cuda
    if not _have_cuda:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2503_01199_b200 needs a CUDA device (B200, sm_100a); none is available")
        _have_cuda = True
    if t is not None and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")


# stream handle -> device index, so call() can make that device current
# (the C-ABI launches on the current device; include/splat_b200.h)
_stream_device: dict = {}


def device_index(device=None) -> int:
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, int):
        return device
    return device_index(torch.device(device))


_cuda_ready = False


_raw_current = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def raw_stream(device=None) -> tuple:
    """(device index, current stream handle) without constructing a
    torch.cuda.Stream (the per-call host cost of torch.cuda.current_stream
    is a visible share of a small-scene iteration); torch builds without the
    raw accessor take the public path."""
    global _cuda_ready
    if not _cuda_ready:
        torch.cuda.init()
        _cuda_ready = True
    idx = device_index(device)
    if _raw_current is None:
        return idx, torch.cuda.current_stream(idx).cuda_stream
    return idx, _raw_current(idx)


def stream_ptr(device=None) -> int:
    idx, s = raw_stream(device)
    _stream_device[s] = idx
    return s


def ptr(t: torch.Tensor | None):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


# kernel launches issued by each entry point (for bench.py's gpu_launches);
# the radix sort issues 3 per 8-bit pass and is counted by the caller.
KERNELS_PER_CALL = {
    "sb_morton_keys": 3, "sb_morton_encode": 1, "sb_permute_rows": 1, "sb_project_cull_compact": 1, "sb_bin_prepare": 3,
    "sb_bin_finish": 2, "sb_raster_fwd": 1, "sb_raster_bwd": 1, "sb_radix_sort_pairs_u64": 10,
    "sb_chain_projection_bwd": 1, "sb_chain_projection_bwd_accumulate": 1, "sb_adam_sparse": 1, "sb_build_clusters": 1, "sb_cull_clusters": 1, "sb_variance_score": 1, "sb_lane_reduce": 1,
    "sb_densify_select": 14, "sb_densify_apply": 3,
    "sb_loss_fwd_bwd": 1,
}
launch_count = {"n": 0}
# optional per-call CUDA-event timing: {name: [(start_event, end_event), ...]}
_timing: dict | None = None


def enable_call_timing(on: bool = True):
    """Record CUDA events around every sb_* call on the current stream."""
    global _timing
    _timing = {} if on else None


def call_timings() -> dict:
    """{name: [ms, ...]} for the calls recorded since enable_call_timing()."""
    if _timing is None:
        return {}
    return {k: [a.elapsed_time(b) for a, b in v] for k, v in _timing.items()}


# entry points whose last argument tuple is kept for replay_time()
_keep_args: dict | None = None


def keep_last_args(names):
    """Remember the arguments of the last call of each named entry point
    (bench.py replays the raster kernels to time them back to back)."""
    global _keep_args
    _keep_args = {n: None for n in names} if names else None


def replay_time(name: str, k: int) -> float:
    """Average device time (ms) of `name` re-issued k times back to back on
    its recorded stream with the arguments of its last call: CUDA events on
    that stream around the k launches, after one untimed launch.  The calls
    are pure functions of their buffers (the raster tile queues reset
    themselves; a replayed backward adds its gradients again, same work)."""
    lib = load()
    args = (_keep_args or {}).get(name)
    if args is None:
        raise RuntimeError(f"replay_time: no recorded call of {name}")
    sv = args[-1].value if isinstance(args[-1], C.c_void_p) else args[-1]
    stream = torch.cuda.ExternalStream(sv) if sv else torch.cuda.default_stream()
    f = getattr(lib, name)
    with torch.cuda.stream(stream):
        f(*args)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            rc = f(*args)
        b.record()
    b.synchronize()
    if rc != SB_OK:
        raise RuntimeError(f"{name} replay failed ({rc})")
    launch_count["n"] += (k + 1) * KERNELS_PER_CALL.get(name, 0)
    return a.elapsed_time(b) / k


def call(name: str, *args):
    """Call an sb_* entry point and map its status to the reference's
    exception conventions (errors.py:6-32)."""
    lib = load()
    launch_count["n"] += KERNELS_PER_CALL.get(name, 0)
    dev = None
    if args and isinstance(args[-1], C.c_void_p) and args[-1].value in _stream_device:
        dev = _stream_device[args[-1].value]
        if dev == torch.cuda.current_device():
            dev = None
    if dev is not None:     # the stream belongs to another device: launch there
        with torch.cuda.device(dev):
            return _call(lib, name, args)
    return _call(lib, name, args)


def _call(lib, name, args):
    if _keep_args is not None and name in _keep_args:
        _keep_args[name] = args
    if _timing is not None:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        rc = getattr(lib, name)(*args)
        b.record()
        _timing.setdefault(name, []).append((a, b))
    else:
        rc = getattr(lib, name)(*args)
    if rc != SB_OK:
        msg = (lib.sb_last_error() or b"").decode()
        if rc == SB_EINVAL:
            raise ValueError(f"{name}: {msg}")
        raise RuntimeError(f"{name} failed ({rc}): {msg}")
    return rc


# ---------------------------------------------------------------------------
# workspace arena: one growable byte buffer per (purpose, device, stream)
_arena: dict = {}


def workspace(purpose: str, nbytes: int, device) -> torch.Tensor:
    """Per (purpose, device, current stream): the self-resetting workspaces
    (tile queues, look-back words, bin counts, loss ticket, screen-gradient
    rows) must not be shared by work in flight on two streams at once."""
    key = (purpose,) + raw_stream(device)
    buf = _arena.get(key)
    if buf is None or buf.numel() < nbytes:
        # zero-filled once: the raster tile queues expect a zeroed workspace
        # on first use and leave it zeroed (include/splat_b200.h)
        buf = torch.zeros(max(int(nbytes * 1.25), 256), dtype=torch.uint8, device=device)
        _arena[key] = buf
    return buf


__all__ = ["load", "call", "ptr", "stream_ptr", "workspace", "SbCamera", "SbRasterCfg", "require_cuda",
           "ShapeMismatchError", "ValidationError", "exported_symbols"]
