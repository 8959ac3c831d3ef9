"""ctypes binding of libhadis_b200.so (the C ABI in include/hadis_b200.h).

The CUDA library is the only compute path: if it is missing or no CUDA device
is visible, every call raises -- there is no CPU fallback.  PyTorch supplies
device memory and the current stream; the ABI itself sees plain pointers.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhadis_b200.so")
if os.environ.get("HADIS_LIB_VARIANT"):      # A/B builds of the same library (tools/ only)
    LIB_PATH = os.path.join(_HERE, f"libhadis_b200_{os.environ['HADIS_LIB_VARIANT']}.so")

_c_int, _c_i32, _c_i64, _c_sz, _c_dbl, _c_vp = (ctypes.c_int, ctypes.c_int32, ctypes.c_int64,
                                               ctypes.c_size_t, ctypes.c_double, ctypes.c_void_p)

# status codes (hadis_status)
OK, ERR_ARG, ERR_RECORDS, ERR_CAPACITY, ERR_CUDA, ERR_NO_ROWS, ERR_NEG_DEMAND, ERR_UNSUPPORTED = range(8)
# stats layout (hadis_frontier_stat)
ST_ROWS, ST_CANDIDATES, ST_UNCERTAIN, ST_EXACT_CELLS, ST_OVERFLOW, ST_PAIR0 = 0, 1, 2, 3, 4, 8
PAIR_PARAMS = 6

_SIGNATURES = {
    "hadis_abi_version": (_c_int, []),
    "hadis_status_string": (ctypes.c_char_p, [_c_int]),
    "hadis_last_cuda_error": (ctypes.c_char_p, []),
    "hadis_kernel_launches": (_c_i64, []),
    "hadis_hfix_shift": (_c_int, [_c_i64]),
    "hadis_bin_hist": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_i32, _c_i32, _c_vp, _c_vp,
                                _c_vp, _c_vp]),
    "hadis_hist_scan": (_c_int, [_c_vp, _c_vp, _c_i32, _c_i32, _c_vp, _c_vp]),
    "hadis_row_plan_bytes": (_c_sz, [_c_i32]),
    "hadis_bs_store_elems": (_c_i64, [_c_i64, _c_i32]),
    "hadis_records_bucket": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_i32, _c_i32, _c_vp,
                                      _c_vp, _c_vp, _c_vp, _c_sz, _c_vp]),
    "hadis_records_plan": (_c_int, [_c_vp, _c_i64, _c_vp, _c_i32, _c_i32, _c_vp, _c_vp, _c_sz,
                                    _c_vp]),
    "hadis_records_scatter": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_i32, _c_i32, _c_vp,
                                       _c_vp, _c_vp, _c_sz, _c_vp]),
    "hadis_bin_hist_rows": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_vp, _c_vp, _c_vp,
                                     _c_vp, _c_vp]),
    "hadis_frontier_workspace_bytes": (_c_sz, [_c_i32, _c_i32, _c_i64, _c_i64, _c_i64]),
    "hadis_pair_frontiers": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_vp, _c_vp,
                                      _c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_i32, _c_vp, _c_sz,
                                      _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp,
                                      _c_vp, _c_vp, _c_vp, _c_vp]),
    "hadis_pair_frontiers_compact": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_vp,
                                              _c_vp, _c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_i32,
                                              _c_vp, _c_sz, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp,
                                              _c_vp, _c_vp, _c_vp, _c_vp, _c_vp]),
    "hadis_fid_exact": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp,
                                 _c_vp]),
    "hadis_cascade_workspace_bytes": (_c_sz, [_c_i32, _c_i32]),
    "hadis_cascade_points": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp, _c_i32, _c_i32,
                                      _c_vp, _c_vp, _c_vp, _c_vp, _c_sz, _c_vp]),
    "hadis_shard_slab_bytes": (_c_sz, [_c_i32, _c_i64]),
    "hadis_shard_merge_workspace_bytes": (_c_sz, [_c_i32]),
    "hadis_shard_merge": (_c_int, [_c_vp, _c_i32, _c_sz, _c_i64, _c_i32, _c_vp, _c_vp, _c_vp,
                                   _c_i32, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp,
                                   _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_sz, _c_vp]),
    "hadis_lexicon_bytes": (_c_sz, []),
    "hadis_text_workspace_bytes": (_c_sz, [_c_i64]),
    "hadis_text_records": (_c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_i32, _c_vp,
                                    _c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp,
                                    _c_sz, _c_vp]),
    "hadis_text_features": (_c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp,
                                     _c_vp, _c_vp]),
    "hadis_text_keys": (_c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_vp]),
    "hadis_keyed_normal_host": (_c_int, [_c_vp, _c_vp, _c_i64, _c_dbl, _c_vp, _c_i32]),
    "hadis_tune_weights": (_c_int, [_c_vp, _c_vp, _c_i32, _c_i32, _c_vp, _c_i32, _c_i32, _c_vp,
                                    _c_vp, _c_vp]),
    "hadis_pareto_workspace_bytes": (_c_sz, [_c_i64]),
    "hadis_pareto_prune": (_c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_sz, _c_vp]),
    "hadis_solve_workspace_bytes": (_c_sz, [_c_i32, _c_i32]),
    "hadis_solve_many": (_c_int, [_c_i32, _c_vp, _c_vp, _c_vp, _c_i32, _c_i32, _c_vp, _c_vp, _c_vp,
                                  _c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_dbl, _c_vp, _c_vp,
                                  _c_vp, _c_vp, _c_vp, _c_vp, _c_sz, _c_vp]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


class HadisError(RuntimeError):
    """A libhadis_b200 call failed (status code and message attached)."""

    def __init__(self, status, where):
        self.status = status
        msg = load().hadis_status_string(status).decode()
        if status == ERR_CUDA:
            msg += ": " + load().hadis_last_cuda_error().decode()
        super().__init__(f"{where}: {msg} (status {status})")


def load():
    """Load the shared library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; "
                "g.build()\"` (or `make -C paper_2509_00642_b200/csrc`). There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.hadis_abi_version() != 1:
            raise RuntimeError("libhadis_b200.so ABI version mismatch")
        _lib = lib
    return _lib


def check(status, where):
    if status != OK:
        raise HadisError(status, where)


def torch_cuda():
    """torch with a visible CUDA device, else a loud error (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the HADIS B200 path needs a CUDA device (sm_100a); "
                           "no CPU fallback exists")
    return torch


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def stream_handle(stream=None, device=None):
    """cudaStream_t of ``stream``, else of the current stream of ``device``."""
    torch = torch_cuda()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def pareto_prune_indices(lat, qual):
    """Indices kept by pareto_prune, in its output order (GPU)."""
    torch = torch_cuda()
    lat = np.asarray(lat, dtype=np.float64)
    qual = np.asarray(qual, dtype=np.float64)
    if np.isnan(lat).any() or np.isnan(qual).any():
        raise ValueError("pareto_prune: NaN keys are not ordered")
    n = int(lat.shape[0])
    dev = torch.device("cuda")
    d_lat = torch.from_numpy(lat).to(dev)
    d_qual = torch.from_numpy(qual).to(dev)
    out_idx = torch.empty(n, dtype=torch.int64, device=dev)
    out_cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lib = load()
    ws_bytes = lib.hadis_pareto_workspace_bytes(n)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=dev)
    check(lib.hadis_pareto_prune(ptr(d_lat), ptr(d_qual), n, ptr(out_idx), ptr(out_cnt), ptr(ws),
                                 ws_bytes, stream_handle()), "hadis_pareto_prune")
    k = int(out_cnt.item())
    return out_idx[:k].cpu().tolist()
