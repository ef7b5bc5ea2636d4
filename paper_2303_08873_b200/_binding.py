"""Thin ctypes binding of libadapt.so (include/adapt.h).

Argument marshalling only: every step of record -> label -> train -> select
runs in the library's sm_100a kernels.  Same names as the C ABI.  Arrays may
be numpy arrays (host) or torch tensors (host or CUDA); a CUDA stream may be a
torch.cuda.Stream, an int handle or None (legacy default stream).

There is no fallback: if libadapt.so is missing the import fails, and with no
usable B200 every compute call raises AdaptError(ADAPT_E_CUDA).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libadapt.so")

ADAPT_OK = 0
ADAPT_E_INVALID_ARG = -1
ADAPT_E_USAGE = -2
ADAPT_E_ARITY = -3
ADAPT_E_INSUFFICIENT_DATA = -4
ADAPT_E_SPEC_MISMATCH = -5
ADAPT_E_BAD_VALUE = -6
ADAPT_E_TOO_MANY_DISTINCT = -7
ADAPT_E_NOT_TRAINED = -8
ADAPT_E_CUDA = -9
ADAPT_E_NCCL = -10
ADAPT_E_OOM = -11

# the exported symbols of include/adapt.h (checked by tests/test_boundary.py)
SYMBOLS = [
    "adapt_init", "adapt_nccl_unique_id", "adapt_init_host_comm", "adapt_finalize",
    "adapt_last_error", "adapt_version",
    "adapt_region_create", "adapt_region_destroy", "adapt_region_info", "adapt_record",
    "adapt_record_batch", "adapt_get_wide_table", "adapt_record_table", "adapt_distinct_pairs", "adapt_train", "adapt_train_many",
    "adapt_select", "adapt_select_batch", "adapt_select_batch_host", "adapt_select_table", "adapt_get_tree",
    "adapt_forest_size", "adapt_get_forest_tree", "adapt_kfold", "adapt_get_kfold_tree",
    "adapt_set_tree", "adapt_get_labels", "adapt_get_value_table", "adapt_get_bins",
    "adapt_profile_enable", "adapt_profile_reset", "adapt_profile_get", "adapt_train_stats",
    "__adapt_region_create", "__adapt_region_begin", "__adapt_region_end",
    "__adapt_region_set_feature", "__adapt_region_get_policy", "__adapt_region_train",
]

NODE_DTYPE = np.dtype([
    ("feature", np.int32), ("left", np.int32), ("right", np.int32), ("label", np.int32),
    ("depth", np.int32), ("pad_", np.int32), ("threshold", np.float64), ("n", np.int64),
    ("gini", np.float64),
])
assert NODE_DTYPE.itemsize == 48

KFOLD_DTYPE = np.dtype([  # adapt_kfold_result_t
    ("shuffle", np.int32), ("fold", np.int32), ("n_nodes", np.int32), ("pad_", np.int32),
    ("n_train", np.int64), ("n_test", np.int64), ("n_correct", np.int64),
    ("t_selected", np.float64), ("t_best", np.float64),
])
assert KFOLD_DTYPE.itemsize == 56


class adapt_phase_t(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64),
                ("ms", ctypes.c_double), ("bytes", ctypes.c_double)]


_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_void_p)
_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t,
                                 ctypes.c_void_p)


class adapt_host_comm_t(ctypes.Structure):
    _fields_ = [("all_gather", _ALLGATHER_FN), ("all_reduce_u64", _ALLREDUCE_FN),
                ("user", ctypes.c_void_p)]


class AdaptError(RuntimeError):
    def __init__(self, code: int, call: str, msg: str):
        super().__init__(f"{call} -> {code}: {msg}")
        self.code = code


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
_L = ctypes.CDLL(LIB_PATH)
_P, _I, _I64, _U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
_sigs = {
    "adapt_init": [_I, _I, _I, _P],
    "adapt_nccl_unique_id": [_P],
    "adapt_init_host_comm": [_I, _I, _I, ctypes.POINTER(adapt_host_comm_t)],
    "adapt_finalize": [],
    "adapt_region_create": [ctypes.c_char_p, _I, _I, ctypes.c_char_p, _I, _P],
    "adapt_region_destroy": [_P],
    "adapt_region_info": [_P, _P, _P, _P, _P, _P, _P],
    "adapt_record": [_P, _P, _I, _U64],
    "adapt_record_table": [_P, _P, _P, _I64, _I, _P],
    "adapt_record_batch": [_P, _P, _P, _P, _I64, _I, _P],
    "adapt_get_wide_table": [_P, _P, _P, _I64, _P],
    "adapt_distinct_pairs": [_P, _P],
    "adapt_train": [_P, _P],
    "adapt_train_many": [_P, _I, _P],
    "adapt_select": [_P, _P, _P],
    "adapt_select_batch": [_P, _P, _I64, _P, _P],
    "adapt_select_batch_host": [_P, _P, _I64, _P, _P],
    "adapt_select_table": [_P, _P, _I, _P],
    "adapt_get_tree": [_P, _P, ctypes.c_int32, _P],
    "adapt_forest_size": [_P, _P],
    "adapt_get_forest_tree": [_P, ctypes.c_int32, _P, ctypes.c_int32, _P],
    "adapt_kfold": [_P, _I, _I, _I, _U64, _P, _P],
    "adapt_get_kfold_tree": [_P, ctypes.c_int32, _P, ctypes.c_int32, _P],
    "adapt_set_tree": [_P, _P, ctypes.c_int32],
    "adapt_get_labels": [_P, _P, _I64],
    "adapt_get_value_table": [_P, _I, _P, _P],
    "adapt_get_bins": [_P, _P, _I64],
    "adapt_profile_enable": [_I],
    "adapt_profile_reset": [],
    "adapt_profile_get": [_P, _I, _P],
    "adapt_train_stats": [_P, _P, _I, _P],
}
for _name, _args in _sigs.items():
    getattr(_L, _name).argtypes = _args
    getattr(_L, _name).restype = _I
_L.adapt_last_error.restype = ctypes.c_char_p
_L.adapt_version.restype = ctypes.c_char_p
_L.__adapt_region_create.argtypes = [ctypes.c_char_p, _I, _I, ctypes.c_char_p, _I]
_L.__adapt_region_create.restype = _P
for _name in ("__adapt_region_begin", "__adapt_region_end", "__adapt_region_train"):
    getattr(_L, _name).argtypes = [_P]
    getattr(_L, _name).restype = None
_L.__adapt_region_set_feature.argtypes = [_P, ctypes.c_float]
_L.__adapt_region_set_feature.restype = None
_L.__adapt_region_get_policy.argtypes = [_P]
_L.__adapt_region_get_policy.restype = _I


def lib() -> ctypes.CDLL:
    return _L


def _check(rc: int, call: str) -> None:
    if rc != ADAPT_OK:
        raise AdaptError(rc, call, adapt_last_error())


def _ptr(a) -> int:
    """Address of a numpy array or torch tensor (host or device)."""
    if a is None:
        return 0
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _check_array(a, name: str, dtype, cols: int | None, rows: int, on_device: bool | None):
    """Validate an operand before its pointer crosses the C ABI: element type,
    contiguity, [rows][cols] shape (at least `rows` rows) and its device."""
    if a is None or isinstance(a, int):
        return  # raw addresses: the caller vouches for them
    if isinstance(a, np.ndarray):
        if on_device:
            raise ValueError(f"{name}: a numpy array is host memory but on_device=True")
        dts = (dtype,) if isinstance(dtype, str) else dtype
        if a.dtype not in [np.dtype(d) for d in dts]:
            raise TypeError(f"{name}: dtype {a.dtype}, expected {dtype}")
        shape = a.shape
    elif hasattr(a, "data_ptr"):
        import torch

        dts = (dtype,) if isinstance(dtype, str) else dtype
        if a.dtype not in [getattr(torch, d) for d in dts if hasattr(torch, d)]:
            raise TypeError(f"{name}: dtype {a.dtype}, expected torch.{dtype}")
        if on_device is not None and bool(a.is_cuda) != bool(on_device):
            raise ValueError(f"{name}: tensor on {a.device} but on_device={bool(on_device)}")
        shape = tuple(a.shape)
    else:
        raise TypeError(f"{name}: unsupported array type {type(a)}")
    if cols is None:
        ok = (len(shape) == 1 and shape[0] >= rows) or (rows == 0)
    elif len(shape) == 2:
        ok = shape[1] == cols and shape[0] >= rows
    else:
        ok = len(shape) == 1 and shape[0] >= rows * cols
    if not ok:
        want = f"[>= {rows}]" if cols is None else f"[>= {rows}][{cols}]"
        raise ValueError(f"{name}: shape {shape}, expected {want}")
    _ptr(a)  # contiguity


# Device tables passed with on_device=1 are BORROWED until the next train
# (adapt.h adapt_record_table): hold a reference per region so the caching
# allocator cannot recycle them in between.  Replaced by the next record_table,
# dropped by adapt_region_destroy.
_borrowed: dict = {}


def _stream(s) -> int:
    if s is None:
        return 0
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ------------------------------------------------------------------- C ABI --
def adapt_last_error() -> str:
    return (_L.adapt_last_error() or b"").decode()


def adapt_version() -> str:
    return _L.adapt_version().decode()


def adapt_init(device: int = 0, rank: int = 0, world: int = 1, nccl_unique_id: bytes | None = None):
    buf = None
    if nccl_unique_id is not None:
        buf = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
    _check(_L.adapt_init(device, rank, world, ctypes.cast(buf, _P) if buf else None), "adapt_init")


_host_comm_keepalive = None


def adapt_init_host_comm(device: int, rank: int, world: int, all_gather, all_reduce_u64):
    """Host-staged collectives (adapt.h adapt_init_host_comm).

    all_gather(send: np.ndarray[uint8]) -> np.ndarray[uint8] of world*len(send)
    bytes in rank order; all_reduce_u64(buf: np.ndarray[uint64]) -> the element-wise
    sum over ranks (np.ndarray[uint64], same length).
    Exceptions in a hook become a non-zero return (-> ADAPT_E_NCCL)."""
    global _host_comm_keepalive

    def _ag(send, recv, nbytes, _user):
        try:
            snd = np.ctypeslib.as_array(ctypes.cast(send, ctypes.POINTER(ctypes.c_uint8)), (nbytes,))
            out = np.asarray(all_gather(snd.copy()), dtype=np.uint8).reshape(-1)
            if out.size != world * nbytes:
                return 2
            ctypes.memmove(recv, out.ctypes.data, out.size)
            return 0
        except Exception:  # noqa: BLE001  (reported through the return code)
            return 1

    def _ar(buf, count, _user):
        try:
            a = np.ctypeslib.as_array(buf, (count,))
            r = np.asarray(all_reduce_u64(a.copy()), dtype=np.uint64).reshape(-1)
            if r.size != count:
                return 2
            a[:] = r
            return 0
        except Exception:  # noqa: BLE001
            return 1

    hooks = adapt_host_comm_t(_ALLGATHER_FN(_ag), _ALLREDUCE_FN(_ar), None)
    _host_comm_keepalive = hooks  # the library keeps the function pointers
    _check(_L.adapt_init_host_comm(device, rank, world, ctypes.byref(hooks)), "adapt_init_host_comm")


def adapt_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_L.adapt_nccl_unique_id(ctypes.cast(buf, _P)), "adapt_nccl_unique_id")
    return buf.raw


def adapt_finalize():
    _check(_L.adapt_finalize(), "adapt_finalize")


def adapt_region_create(id: str, num_features: int, num_variants: int,
                        model_params: str | None = None, min_train_data: int = 0) -> int:
    out = ctypes.c_void_p()
    _check(_L.adapt_region_create(id.encode(), num_features, num_variants,
                                  model_params.encode() if model_params is not None else None,
                                  min_train_data, ctypes.byref(out)), "adapt_region_create")
    return out.value


def adapt_region_destroy(h: int):
    _check(_L.adapt_region_destroy(h), "adapt_region_destroy")
    _borrowed.pop(h, None)


def adapt_region_info(h: int) -> dict:
    F, V, D, M, T = (ctypes.c_int() for _ in range(5))
    rows = ctypes.c_int64()
    _check(_L.adapt_region_info(h, ctypes.byref(F), ctypes.byref(V), ctypes.byref(D),
                                ctypes.byref(M), ctypes.byref(rows), ctypes.byref(T)),
           "adapt_region_info")
    return dict(num_features=F.value, num_variants=V.value, max_depth=D.value,
                min_train_data=M.value, num_rows=rows.value, trained=bool(T.value))


def adapt_record(h: int, features, variant: int, elapsed_ns: int):
    x = np.ascontiguousarray(features, dtype=np.float32)
    _check(_L.adapt_record(h, x.ctypes.data, int(variant), int(elapsed_ns)), "adapt_record")


def adapt_record_table(h: int, features, times, n: int | None = None, on_device: bool | None = None,
                       stream=None):
    if n is None:
        n = int(features.shape[0])
    if on_device is None:
        on_device = bool(getattr(features, "is_cuda", False))
    info = adapt_region_info(h)
    _check_array(features, "features", "float32", info["num_features"], int(n), on_device)
    _check_array(times, "times", "float32", info["num_variants"], int(n), on_device)
    _check(_L.adapt_record_table(h, _ptr(features), _ptr(times), int(n), int(on_device),
                                 _stream(stream)), "adapt_record_table")
    if on_device:
        _borrowed[h] = (features, times)
    else:
        _borrowed.pop(h, None)


def adapt_record_batch(h: int, features, variants, elapsed_ns, m: int | None = None,
                       on_device: bool | None = None, stream=None):
    """m long-format records (features [m][F] f32, variants [m] i32, elapsed_ns [m] u64)."""
    if m is None:
        m = int(features.shape[0])
    if on_device is None:
        on_device = bool(getattr(features, "is_cuda", False))
    F = adapt_region_info(h)["num_features"]
    _check_array(features, "features", "float32", F, int(m), on_device)
    _check_array(variants, "variants", "int32", None, int(m), on_device)
    _check_array(elapsed_ns, "elapsed_ns", ("uint64", "int64"), None, int(m), on_device)
    _check(_L.adapt_record_batch(h, _ptr(features), _ptr(variants), _ptr(elapsed_ns), int(m),
                                 int(on_device), _stream(stream)), "adapt_record_batch")


def adapt_get_wide_table(h: int):
    """(features [n][F] f32, times [n][V] f32) the last train aggregated from records."""
    n = ctypes.c_int64()
    _check(_L.adapt_get_wide_table(h, None, None, 0, ctypes.byref(n)), "adapt_get_wide_table")
    info = adapt_region_info(h)
    F, V = info["num_features"], info["num_variants"]
    feat = np.empty((n.value, F), np.float32)
    times = np.empty((n.value, V), np.float32)
    _check(_L.adapt_get_wide_table(h, _ptr(feat), _ptr(times), n.value, ctypes.byref(n)),
           "adapt_get_wide_table")
    return feat, times


def adapt_distinct_pairs(h: int) -> int:
    c = ctypes.c_int64()
    _check(_L.adapt_distinct_pairs(h, ctypes.byref(c)), "adapt_distinct_pairs")
    return c.value


def adapt_train(h: int, stream=None):
    _check(_L.adapt_train(h, _stream(stream)), "adapt_train")


def adapt_train_many(hs, stream=None):
    arr = (ctypes.c_void_p * len(hs))(*hs)
    _check(_L.adapt_train_many(ctypes.cast(arr, _P), len(hs), _stream(stream)), "adapt_train_many")


def adapt_select(h: int, features) -> int:
    x = np.ascontiguousarray(features, dtype=np.float32)
    v = ctypes.c_int32()
    _check(_L.adapt_select(h, x.ctypes.data, ctypes.byref(v)), "adapt_select")
    return v.value


def adapt_select_batch(h: int, d_X, m: int, d_out, stream=None):
    F = adapt_region_info(h)["num_features"]
    _check_array(d_X, "X", "float32", F, int(m), True)
    _check_array(d_out, "out", "int32", None, int(m), True)
    _check(_L.adapt_select_batch(h, _ptr(d_X), int(m), _ptr(d_out), _stream(stream)),
           "adapt_select_batch")


def adapt_select_batch_host(h: int, X, m: int, out, stream=None):
    F = adapt_region_info(h)["num_features"]
    _check_array(X, "X", "float32", F, int(m), False)
    _check_array(out, "out", "int32", None, int(m), False)
    _check(_L.adapt_select_batch_host(h, _ptr(X), int(m), _ptr(out), _stream(stream)),
           "adapt_select_batch_host")


def adapt_select_table(h: int, out, stream=None):
    """Selections of every row of the recorded (host) wide table into out [n]
    int32 (a numpy array or a host / CUDA tensor)."""
    on_dev = bool(getattr(out, "is_cuda", False))
    _check_array(out, "out", "int32", None, adapt_region_info(h)["num_rows"], on_dev)
    _check(_L.adapt_select_table(h, _ptr(out), int(on_dev), _stream(stream)), "adapt_select_table")


def adapt_get_tree(h: int) -> np.ndarray:
    n = ctypes.c_int32()
    rc = _L.adapt_get_tree(h, None, 0, ctypes.byref(n))
    if rc not in (ADAPT_OK, ADAPT_E_INVALID_ARG) or n.value <= 0:
        _check(rc, "adapt_get_tree")
    out = np.zeros(n.value, NODE_DTYPE)
    _check(_L.adapt_get_tree(h, out.ctypes.data, n.value, ctypes.byref(n)), "adapt_get_tree")
    return out


def adapt_forest_size(h: int) -> int:
    t = ctypes.c_int32()
    _check(_L.adapt_forest_size(h, ctypes.byref(t)), "adapt_forest_size")
    return t.value


def adapt_get_forest_tree(h: int, t: int) -> np.ndarray:
    """Tree t of a forest (tree 0 of a decision-tree region), NODE_DTYPE records."""
    n = ctypes.c_int32()
    _L.adapt_get_forest_tree(h, int(t), None, 0, ctypes.byref(n))  # size query (cap 0)
    out = np.zeros(max(n.value, 1), NODE_DTYPE)
    _check(_L.adapt_get_forest_tree(h, int(t), out.ctypes.data, len(out), ctypes.byref(n)),
           "adapt_get_forest_tree")
    return out[:n.value]


def adapt_kfold(h: int, K: int, train_groups: int, shuffles: int, seed: int = 0,
                stream=None) -> np.ndarray:
    """The paper's K-fold harness: shuffles * K models, KFOLD_DTYPE records
    in (shuffle, fold) order.  Collective over ranks; the table is the recorded one."""
    out = np.zeros(shuffles * K if shuffles > 0 and K > 0 else 1, KFOLD_DTYPE)
    _check(_L.adapt_kfold(h, int(K), int(train_groups), int(shuffles), ctypes.c_uint64(seed),
                          out.ctypes.data, _stream(stream)), "adapt_kfold")
    return out


def adapt_get_kfold_tree(h: int, model: int) -> np.ndarray:
    """Tree of K-fold model `model` (= shuffle * K + fold) of the last adapt_kfold."""
    n = ctypes.c_int32()
    _L.adapt_get_kfold_tree(h, int(model), None, 0, ctypes.byref(n))  # size query (cap 0)
    out = np.zeros(max(n.value, 1), NODE_DTYPE)
    _check(_L.adapt_get_kfold_tree(h, int(model), out.ctypes.data, len(out), ctypes.byref(n)),
           "adapt_get_kfold_tree")
    return out[:n.value]


def adapt_set_tree(h: int, nodes: np.ndarray):
    nodes = np.ascontiguousarray(nodes, dtype=NODE_DTYPE)
    _check(_L.adapt_set_tree(h, nodes.ctypes.data, len(nodes)), "adapt_set_tree")


def adapt_get_labels(h: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint8)
    _check(_L.adapt_get_labels(h, out.ctypes.data, n), "adapt_get_labels")
    return out


def adapt_get_value_table(h: int, f: int) -> np.ndarray:
    vals = np.zeros(256, np.float32)
    c = ctypes.c_int()
    _check(_L.adapt_get_value_table(h, f, vals.ctypes.data, ctypes.byref(c)), "adapt_get_value_table")
    return vals[: c.value].copy()


def adapt_get_bins(h: int, n: int, F: int) -> np.ndarray:
    out = np.empty((n, F), np.uint8)
    _check(_L.adapt_get_bins(h, out.ctypes.data, n), "adapt_get_bins")
    return out


def adapt_profile_enable(enable: bool = True):
    _check(_L.adapt_profile_enable(int(enable)), "adapt_profile_enable")


def adapt_profile_reset():
    _check(_L.adapt_profile_reset(), "adapt_profile_reset")


def adapt_profile_get() -> dict:
    arr = (adapt_phase_t * 64)()
    n = ctypes.c_int()
    _check(_L.adapt_profile_get(ctypes.cast(arr, _P), 64, ctypes.byref(n)), "adapt_profile_get")
    return {arr[i].name.decode(): dict(launches=arr[i].launches, ms=arr[i].ms, bytes=arr[i].bytes)
            for i in range(min(n.value, 64))}


def adapt_train_stats(h: int) -> list:
    lv = ctypes.c_int()
    _check(_L.adapt_train_stats(h, None, 0, ctypes.byref(lv)), "adapt_train_stats")
    K = 6  # values per level (adapt.h)
    buf = np.zeros(K * max(lv.value, 1), np.int64)
    _check(_L.adapt_train_stats(h, buf.ctypes.data, buf.size, ctypes.byref(lv)), "adapt_train_stats")
    return [dict(nodes=int(buf[K * d]), rows_hist=int(buf[K * d + 1]), rows_part=int(buf[K * d + 2]),
                 hist_bytes=int(buf[K * d + 3]), comm_bytes=int(buf[K * d + 4]),
                 direct_hist_bytes=int(buf[K * d + 5]))
            for d in range(lv.value)]


# ------------------------------------------------------ Apollo Table-1 shim --
def __adapt_region_create(id: str, num_features: int, num_policies: int,
                          model_type_params: str | None = None, min_train_data: int = 0):
    return _L.__adapt_region_create(id.encode(), num_features, num_policies,
                                    model_type_params.encode() if model_type_params else None,
                                    min_train_data)


def __adapt_region_begin(r):
    _L.__adapt_region_begin(r)


def __adapt_region_end(r):
    _L.__adapt_region_end(r)


def __adapt_region_set_feature(r, v: float):
    _L.__adapt_region_set_feature(r, ctypes.c_float(v))


def __adapt_region_get_policy(r) -> int:
    return _L.__adapt_region_get_policy(r)


def __adapt_region_train(r):
    _L.__adapt_region_train(r)
