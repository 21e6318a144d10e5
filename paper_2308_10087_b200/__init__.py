"""B200-native chunk-pipelined full-graph GCN/GCNII training (GNNPipe, arXiv 2308.10087).

Python mirror of the reference's public API for the hot path (proj/include/gnnsim/*.hpp),
implemented over the in-tree C-ABI libraries:

* ``lib/libgnnsim_b200.so`` — host C++ (bit-exact CSR / chunking / schedule / init) and
  the trainers, exported as ``gs_*``;
* ``lib/libgpcuda.so`` — the sm_100a stage engine, exported as ``gp_*``.

Nothing here computes on the CPU: training goes through the CUDA engine and fails loudly
(``GpuEngineError``) when the extension or a device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "GP_OK", "GP_EINVAL", "GP_ENUMERIC", "GP_EFABRIC", "GP_ECUDA", "GP_ERUNTIME",
    "GnnsimError", "InvalidArgument", "NumericError", "FabricError", "GpuEngineError",
    "LayerKind", "ModelKind", "stage_footprint", "ModelConfig", "TrainOptions", "TrainResult", "LayerSpec",
    "Dataset", "make_chunks", "partition_vertices", "shuffle_chunk_order", "make_stage_assignment",
    "save_assignment", "load_assignment",
    "build_layer_specs", "init_params", "train_pipeline", "train_sequential", "train_hybrid", "StageEngine",
    "nccl_unique_id", "device_count", "lib_paths", "PROFILE_CLASSES",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBDIR = os.environ.get("GP_LIBDIR") or os.path.join(_HERE, "lib")

# Eager CUDA module loading (read by the driver at initialisation, so set before the
# engine library makes its first CUDA call). With lazy loading, the first launch of a
# kernel synchronises the context; two stages of one process linked by in-stream
# waits (gp_link_ipc between threads) then deadlock on a first launch.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

GP_OK, GP_EINVAL, GP_ENUMERIC, GP_EFABRIC, GP_ECUDA, GP_ERUNTIME = 0, 1, 2, 3, 4, 5
PROFILE_CLASSES = ["remask", "fwd_agg", "fwd_dense", "bwd_agg", "bwd_dense", "xent", "pgrad", "optim", "xfer"]
IPC_BLOB_BYTES = 256  # GP_IPC_BLOB_BYTES
GP_BUF = {"h": 0, "pre": 1, "dz": 2, "dagg": 3, "dh0": 4, "hsnap": 5, "in": 6, "dh_in": 7, "gather": 8,
          "hist_h": 9, "hist_in": 10, "hist_dagg": 11}


class GnnsimError(RuntimeError):
    """Base error (std::runtime_error in the reference)."""


class InvalidArgument(GnnsimError, ValueError):
    """std::invalid_argument."""


class NumericError(GnnsimError):
    """gnnsim::NumericError (engines.hpp:48-51)."""


class FabricError(GnnsimError):
    """gnnsim::FabricError (fabric.hpp:139-142)."""


class GpuEngineError(GnnsimError):
    """CUDA / NCCL failure or missing device / extension."""


_ERR = {GP_EINVAL: InvalidArgument, GP_ENUMERIC: NumericError, GP_EFABRIC: FabricError, GP_ECUDA: GpuEngineError}


class LayerKind:
    DENSE, GCNCONV, SAGECONV, GCN2CONV = 0, 1, 2, 3


class ModelKind:
    GCN, SAGE, GCNII = 0, 1, 2


# ----------------------------------------------------------------------------- ctypes
class gp_layer_spec(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("in_dim", C.c_uint32), ("out_dim", C.c_uint32), ("relu", C.c_uint32),
                ("alpha", C.c_double), ("beta", C.c_double)]


class gp_stage_config(C.Structure):
    _fields_ = [("device", C.c_int32), ("num_vertices", C.c_uint32), ("num_chunks", C.c_uint32),
                ("num_stages", C.c_uint32), ("stage", C.c_uint32), ("layer_begin", C.c_uint32),
                ("layer_end", C.c_uint32), ("num_layers", C.c_uint32), ("specs", C.POINTER(gp_layer_spec)),
                ("hidden", C.c_uint32), ("num_classes", C.c_uint32), ("dropout", C.c_double),
                ("seed", C.c_uint64), ("optimizer", C.c_uint32), ("lr", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("fix_alpha", C.c_uint32),
                ("historical_gradients", C.c_uint32), ("synchronous_mode", C.c_uint32),
                ("group_size", C.c_uint32), ("group_rank", C.c_uint32)]


class gp_epoch_stats(C.Structure):
    _fields_ = [("epoch", C.c_uint32), ("has_quality", C.c_uint32), ("loss_sum", C.c_double),
                ("correct", C.c_uint64 * 3), ("bytes_sent", C.c_uint64 * 6), ("msgs_sent", C.c_uint64 * 6),
                ("epoch_ms", C.c_float), ("busy_ms", C.c_float), ("kernel_launches", C.c_uint64)]


class gp_profile(C.Structure):
    _fields_ = [("ms", C.c_double * 9), ("launches", C.c_uint64 * 9), ("alg_bytes", C.c_double * 9),
                ("flops", C.c_double * 9), ("gather_bytes", C.c_double * 9),
                ("span_ms", C.c_double * 9)]


class gs_model_config(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("layers", C.c_uint32), ("hidden", C.c_uint32), ("dropout", C.c_double),
                ("gcnii_alpha", C.c_double), ("gcnii_lambda", C.c_double), ("self_loops", C.c_uint32)]


class gs_train_options(C.Structure):
    _fields_ = [("model", gs_model_config), ("optimizer", C.c_uint32), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("epochs", C.c_uint32),
                ("seed", C.c_uint64), ("shuffle_chunks", C.c_uint32), ("fix_alpha", C.c_uint32),
                ("historical_gradients", C.c_uint32), ("synchronous_mode", C.c_uint32), ("device", C.c_int32),
                ("profile", C.c_uint32), ("collect_trace", C.c_uint32), ("resume_path", C.c_char_p),
                ("save_state_path", C.c_char_p)]


class gs_trace_event(C.Structure):
    _fields_ = [("worker", C.c_uint32), ("kind", C.c_uint32), ("chunk", C.c_int32), ("layer_lo", C.c_int32),
                ("layer_hi", C.c_int32), ("reserved", C.c_uint32), ("t_start", C.c_double), ("t_end", C.c_double)]


class gs_bubble_report(C.Structure):
    _fields_ = [("measured_bubble", C.c_double), ("ideal_bubble", C.c_double), ("stages", C.c_uint32),
                ("chunks", C.c_uint32), ("span", C.c_double)]


class gs_comm_model_input(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("n", "layers", "hidden", "stages", "ways", "alpha", "vecs",
                                          "bytes_per_value")]


# TraceEvent (fabric.hpp) as a numpy record; kind: 0 compute, 1 send, 2 recv, 3 idle
TRACE_DTYPE = np.dtype([("worker", np.uint32), ("kind", np.uint32), ("chunk", np.int32), ("layer_lo", np.int32),
                        ("layer_hi", np.int32), ("reserved", np.uint32), ("t_start", np.float64),
                        ("t_end", np.float64)])
TRACE_KINDS = ("compute", "send", "recv", "idle")


_lib = None


def lib_paths() -> List[str]:
    return [os.path.join(_LIBDIR, "libgnnsim_b200.so"), os.path.join(_LIBDIR, "libgpcuda.so")]


def _L():
    """Load the in-tree libraries (fails loudly: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_paths()[0]
    if not os.path.exists(path):
        raise GpuEngineError(f"{path} is missing: run __graft_entry__.build() (make -C paper_2308_10087_b200/csrc)")
    lib = C.CDLL(path, mode=C.RTLD_LOCAL)  # never interpose symbols of torch / other libraries
    P = C.POINTER
    u32p, u64p, f32p, u8p, f64p = P(C.c_uint32), P(C.c_uint64), P(C.c_float), P(C.c_uint8), P(C.c_double)
    vp = C.c_void_p
    sig = {
        "gs_last_error": (C.c_char_p, []),
        "gs_dataset_from_edges": (C.c_int, [C.c_uint32, u32p, C.c_uint64, f32p, C.c_uint32, u32p, C.c_uint32, u8p, P(vp)]),
        "gs_dataset_synthetic_er": (C.c_int, [C.c_uint32, C.c_double, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, P(vp)]),
        "gs_dataset_load": (C.c_int, [C.c_char_p, P(vp)]),
        "gs_dataset_save": (C.c_int, [vp, C.c_char_p]),
        "gs_dataset_free": (None, [vp]),
        "gs_dataset_shape": (C.c_int, [vp, u32p, u64p, u32p, u32p]),
        "gs_dataset_graph": (C.c_int, [vp, u64p, u32p, u32p]),
        "gs_dataset_arrays": (C.c_int, [vp, f32p, u32p, u8p]),
        "gs_normalize_adjacency": (C.c_int, [vp, C.c_int, u64p, u32p, f32p]),
        "gs_make_chunks": (C.c_int, [vp, C.c_uint32, C.c_uint64, u32p]),
        "gs_partition_vertices": (C.c_int, [vp, C.c_uint32, C.c_uint64, u32p, u64p, u64p]),
        "gs_shuffle_chunk_order": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, u32p]),
        "gs_save_assignment": (C.c_int, [C.c_char_p, C.c_uint32, u32p, C.c_uint64]),
        "gs_load_assignment": (C.c_int, [C.c_char_p, P(C.c_uint32), u32p, C.c_uint64, P(C.c_uint64)]),
        "gs_make_stage_assignment": (C.c_int, [C.c_uint32, C.c_uint32, u32p]),
        "gs_num_layers": (C.c_int, [P(gs_model_config), u32p]),
        "gs_build_layer_specs": (C.c_int, [P(gs_model_config), C.c_uint32, C.c_uint32, P(gp_layer_spec)]),
        "gs_init_params": (C.c_int, [P(gs_model_config), C.c_uint32, C.c_uint32, C.c_uint64, f32p]),
        "gs_checkpoint_names_bytes": (C.c_int, [C.c_char_p, P(C.c_uint64)]),
        "gs_train_pipeline": (C.c_int, [vp, u32p, C.c_uint32, C.c_uint32, P(gs_train_options), P(vp)]),
        "gs_train_sequential": (C.c_int, [vp, P(gs_train_options), P(vp)]),
        "gs_train_hybrid": (C.c_int, [vp, u32p, u32p, C.c_uint32, C.c_uint32, P(gs_train_options), P(vp)]),
        "gs_train_graph_parallel": (C.c_int, [vp, u32p, P(gs_train_options), P(vp)]),
        "gp_upload_partition": (C.c_int, [vp, u32p]),
        "gp_link_group": (C.c_int, [P(vp), C.c_uint32]),
        "gs_result_metrics": (C.c_int, [vp, u32p, f64p, u64p]),
        "gs_result_params": (C.c_int, [vp, f32p]),
        "gs_result_profile": (C.c_int, [vp, P(gp_profile)]),
        "gs_result_peak_bytes": (C.c_int, [vp, u64p]),
        "gs_result_trace": (C.c_int, [vp, vp, C.c_uint64, u64p]),
        "gs_result_ledger": (C.c_int, [vp, u64p]),
        "gs_write_metrics_csv": (C.c_int, [C.c_char_p, f64p, u64p, C.c_uint32]),
        "gs_write_trace_jsonl": (C.c_int, [C.c_char_p, vp, C.c_uint64]),
        "gs_write_comm_report_csv": (C.c_int, [C.c_char_p, u64p, C.c_uint32]),
        "gs_bubble_analysis": (C.c_int, [vp, C.c_uint64, P(gs_bubble_report)]),
        "gs_comm_volumes": (C.c_int, [P(gs_comm_model_input), f64p, f64p, f64p]),
        "gs_save_stage_checkpoint": (C.c_int, [C.c_char_p, P(gs_model_config), C.c_uint32, C.c_uint32, f32p,
                                               C.c_uint32, C.c_uint32]),
        "gs_load_checkpoint": (C.c_int, [C.c_char_p, P(C.c_char), C.c_uint64, u64p, f32p, u64p, u64p]),
        "gp_get_optimizer_state": (C.c_int, [vp, C.c_uint32, f32p, f32p, f32p, f32p, u64p]),
        "gp_set_optimizer_state": (C.c_int, [vp, C.c_uint32, f32p, f32p, f32p, f32p, C.c_uint64]),
        "gs_crossover_report": (C.c_int, [P(gs_comm_model_input), P(gs_comm_model_input), P(gs_comm_model_input),
                                          f64p, P(C.c_char), C.c_uint64]),
        "gs_write_compare_csv": (C.c_int, [C.c_char_p, C.c_char_p, f64p, u64p, C.c_uint64]),
        "gp_set_trace": (C.c_int, [vp, C.c_int]),
        "gp_get_trace": (C.c_int, [vp, vp, C.c_uint64, u64p]),
        "gp_clear_trace": (C.c_int, [vp]),
        "gs_result_free": (None, [vp]),
        "gp_abi_version": (C.c_uint32, []),
        "gp_device_count": (C.c_int, [P(C.c_int)]),
        "gp_create": (C.c_int, [P(gp_stage_config), P(vp)]),
        "gp_destroy": (None, [vp]),
        "gp_last_error": (C.c_char_p, [vp]),
        "gp_upload_graph": (C.c_int, [vp, u64p, u32p, f32p, C.c_uint64, u32p]),
        "gp_upload_graph_raw": (C.c_int, [vp, u64p, u32p, C.c_uint64, C.c_int, u32p]),
        "gp_share_graph": (C.c_int, [vp, vp]),
        "gp_upload_features": (C.c_int, [vp, f32p, C.c_uint32]),
        "gp_upload_labels": (C.c_int, [vp, u32p, u8p]),
        "gp_set_layer_params": (C.c_int, [vp, C.c_uint32, f32p, f32p]),
        "gp_get_layer_params": (C.c_int, [vp, C.c_uint32, f32p, f32p]),
        "gp_get_layer_grads": (C.c_int, [vp, C.c_uint32, f32p, f32p]),
        "gp_link_local": (C.c_int, [vp, vp]),
        "gp_nccl_unique_id": (C.c_int, [P(C.c_uint8)]),
        "gp_link_nccl": (C.c_int, [vp, P(C.c_uint8), P(C.c_uint8)]),
        "gp_ipc_export": (C.c_int, [vp, P(C.c_uint8), P(C.c_uint8)]),
        "gp_group_export": (C.c_int, [vp, P(C.c_uint8), C.c_uint64, P(C.c_uint64)]),
        "gp_link_group_ipc": (C.c_int, [vp, P(P(C.c_uint8)), P(C.c_uint64)]),
        "gp_link_ipc": (C.c_int, [vp, P(C.c_uint8), P(C.c_uint8)]),
        "gp_abort": (None, [vp]),
        "gp_run_epoch": (C.c_int, [vp, C.c_uint32, u32p, P(gp_epoch_stats)]),
        "gp_download": (C.c_int, [vp, C.c_uint32, C.c_uint32, f32p, C.c_uint64]),
        "gp_upload_history": (C.c_int, [vp, C.c_uint32, C.c_uint32, f32p, C.c_uint64, C.c_uint32]),
        "gp_stage_footprint": (C.c_int, [P(gp_stage_config), C.c_uint64, C.c_uint32, u64p]),
        "gp_set_profiling": (C.c_int, [vp, C.c_int]),
        "gp_set_live_timing": (C.c_int, [vp, C.c_int]),
        "gp_get_profile": (C.c_int, [vp, P(gp_profile)]),
        "gp_reset_profile": (C.c_int, [vp]),
        "gp_device_bytes": (C.c_int, [vp, u64p]),
        "gp_mark": (C.c_int, [vp, C.c_uint32]),
        "gp_elapsed": (C.c_int, [vp, C.c_uint32, C.c_uint32, P(C.c_float)]),
        "gp_synchronize": (C.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _gs(rc: int) -> None:
    if rc != GP_OK:
        msg = (_L().gs_last_error() or b"").decode()
        raise _ERR.get(rc, GnnsimError)(msg)


def _gp(rc: int, ctx=None) -> None:
    if rc != GP_OK:
        msg = (_L().gp_last_error(ctx) or b"").decode()
        raise _ERR.get(rc, GnnsimError)(msg)


def device_count() -> int:
    n = C.c_int(0)
    _L().gp_device_count(C.byref(n))
    return n.value


# ----------------------------------------------------------------------------- model
@dataclass
class ModelConfig:
    """ModelConfig (nn.hpp:22-30)."""
    kind: int = ModelKind.GCN
    layers: int = 2
    hidden: int = 16
    dropout: float = 0.5
    gcnii_alpha: float = 0.1
    gcnii_lambda: float = 0.5
    self_loops: bool = True

    def c(self) -> gs_model_config:
        return gs_model_config(self.kind, self.layers, self.hidden, self.dropout, self.gcnii_alpha,
                               self.gcnii_lambda, int(self.self_loops))


@dataclass
class TrainOptions:
    """TrainOptions (engines.hpp:69-77) + StalenessConfig (:28-33) + OptimizerConfig (nn.hpp:432-438)."""
    model: ModelConfig = field(default_factory=ModelConfig)
    optimizer: str = "adam"
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    epochs: int = 1
    seed: int = 1
    shuffle_chunks: bool = True
    fix_alpha: int = 10
    historical_gradients: bool = False
    synchronous_mode: bool = False
    device: int = 0
    profile: bool = False
    collect_trace: bool = False  # FabricOptions::collect_trace: measured per-chunk trace (chunks run serially)
    resume_path: str = ""        # continue from a state written by save_state_path (epochs continue)
    save_state_path: str = ""    # write parameters + optimizer state after the last epoch

    def c(self) -> gs_train_options:
        return gs_train_options(self.model.c(), 1 if self.optimizer == "sgd" else 0, self.lr, self.beta1,
                                self.beta2, self.eps, self.epochs, self.seed, int(self.shuffle_chunks),
                                self.fix_alpha, int(self.historical_gradients), int(self.synchronous_mode),
                                self.device, int(self.profile), int(self.collect_trace),
                                self.resume_path.encode() or None, self.save_state_path.encode() or None)


@dataclass
class LayerSpec:
    kind: int
    in_dim: int
    out_dim: int
    relu: bool
    alpha: float
    beta: float

    @property
    def has_bias(self) -> bool:
        return self.kind != LayerKind.GCN2CONV

    @property
    def aggregates(self) -> bool:
        return self.kind != LayerKind.DENSE

    @property
    def k_in(self) -> int:
        """Rows of W (nn.hpp:42): SageConv concatenates [own | mean], so 2 in_dim."""
        return 2 * self.in_dim if self.kind == LayerKind.SAGECONV else self.in_dim


def build_layer_specs(model: ModelConfig, in_features: int, num_classes: int) -> List[LayerSpec]:
    """build_layer_specs (nn.cpp:28-64)."""
    L = C.c_uint32()
    _gs(_L().gs_num_layers(C.byref(model.c()), C.byref(L)))
    arr = (gp_layer_spec * L.value)()
    _gs(_L().gs_build_layer_specs(C.byref(model.c()), in_features, num_classes, arr))
    return [LayerSpec(s.kind, s.in_dim, s.out_dim, bool(s.relu), s.alpha, s.beta) for s in arr]


def _split_params(specs: Sequence[LayerSpec], flat: np.ndarray):
    out, at = [], 0
    for s in specs:
        w = flat[at:at + s.k_in * s.out_dim].reshape(s.k_in, s.out_dim).copy()
        at += s.k_in * s.out_dim
        b = flat[at:at + s.out_dim].copy() if s.has_bias else np.zeros(0, np.float32)
        at += s.out_dim if s.has_bias else 0
        out.append((w, b))
    return out


def _param_count(specs) -> int:
    return sum(s.k_in * s.out_dim + (s.out_dim if s.has_bias else 0) for s in specs)


def init_params(model: ModelConfig, in_features: int, num_classes: int, seed: int):
    """init_params (nn.hpp:60-72): list of (W [k_in x out], b) float32, bit-exact Glorot."""
    specs = build_layer_specs(model, in_features, num_classes)
    flat = np.zeros(_param_count(specs), np.float32)
    _gs(_L().gs_init_params(C.byref(model.c()), in_features, num_classes, seed, _ptr(flat, C.c_float)))
    return _split_params(specs, flat)


# ----------------------------------------------------------------------------- dataset
class Dataset:
    """Dataset (dataset.hpp:15-29) held by the host library."""

    def __init__(self, handle):
        self._h = handle
        n, m, F, Cc = C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_uint32()
        _gs(_L().gs_dataset_shape(handle, C.byref(n), C.byref(m), C.byref(F), C.byref(Cc)))
        self.num_vertices, self.num_edges, self.num_features, self.num_classes = n.value, m.value, F.value, Cc.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gs_dataset_free(self._h)
            self._h = None

    @staticmethod
    def from_edges(n: int, edges: np.ndarray, features: np.ndarray, labels: np.ndarray, num_classes: int,
                   split: np.ndarray) -> "Dataset":
        """build_graph (graph.cpp:33-66) over an arbitrary edge list + node data."""
        e = np.ascontiguousarray(np.asarray(edges, np.uint32).reshape(-1, 2))
        x = np.ascontiguousarray(features, np.float32).reshape(n, -1)
        lab = np.ascontiguousarray(labels, np.uint32)
        sp = np.ascontiguousarray(split, np.uint8)
        h = C.c_void_p()
        _gs(_L().gs_dataset_from_edges(n, _ptr(e, C.c_uint32), e.shape[0], _ptr(x, C.c_float), x.shape[1],
                                       _ptr(lab, C.c_uint32), num_classes, _ptr(sp, C.c_uint8), C.byref(h)))
        return Dataset(h)

    @staticmethod
    def synthetic_er(n: int, p: float, graph_seed: int, num_features: int, num_classes: int,
                     feature_seed: int) -> "Dataset":
        """generate_er (graph.cpp:119-156) + hashed features."""
        h = C.c_void_p()
        _gs(_L().gs_dataset_synthetic_er(n, p, graph_seed, num_features, num_classes, feature_seed, C.byref(h)))
        return Dataset(h)

    @staticmethod
    def load(path: str) -> "Dataset":
        """load_dataset (dataset.cpp:64-119)."""
        h = C.c_void_p()
        _gs(_L().gs_dataset_load(str(path).encode(), C.byref(h)))
        return Dataset(h)

    def save(self, path: str) -> None:
        """save_dataset (dataset.cpp:121-145)."""
        _gs(_L().gs_dataset_save(self._h, str(path).encode()))

    def graph(self):
        """(csr_offsets u64[N+1], csr_neighbors u32[2E], degrees u32[N])."""
        off = np.zeros(self.num_vertices + 1, np.uint64)
        nb = np.zeros(2 * self.num_edges, np.uint32)
        dg = np.zeros(self.num_vertices, np.uint32)
        _gs(_L().gs_dataset_graph(self._h, _ptr(off, C.c_uint64), _ptr(nb, C.c_uint32), _ptr(dg, C.c_uint32)))
        return off, nb, dg

    def arrays(self):
        """(features f32[N,F], labels u32[N], split u8[N])."""
        x = np.zeros((self.num_vertices, self.num_features), np.float32)
        lab = np.zeros(self.num_vertices, np.uint32)
        sp = np.zeros(self.num_vertices, np.uint8)
        _gs(_L().gs_dataset_arrays(self._h, _ptr(x, C.c_float), _ptr(lab, C.c_uint32), _ptr(sp, C.c_uint8)))
        return x, lab, sp

    def normalize_adjacency(self, self_loops: bool = True):
        """normalize_adjacency<float> (graph.cpp:68-98): (offsets u64, cols u32, vals f32)."""
        nnz = 2 * self.num_edges + (self.num_vertices if self_loops else 0)
        off = np.zeros(self.num_vertices + 1, np.uint64)
        cols = np.zeros(nnz, np.uint32)
        vals = np.zeros(nnz, np.float32)
        _gs(_L().gs_normalize_adjacency(self._h, int(self_loops), _ptr(off, C.c_uint64), _ptr(cols, C.c_uint32),
                                        _ptr(vals, C.c_float)))
        return off, cols, vals


def make_chunks(ds: Dataset, num_chunks: int, seed: int) -> np.ndarray:
    """make_chunks (partition.cpp:213-224): chunk_of u32[N]."""
    out = np.zeros(ds.num_vertices, np.uint32)
    _gs(_L().gs_make_chunks(ds._h, num_chunks, seed, _ptr(out, C.c_uint32)))
    return out


def partition_vertices(ds: Dataset, num_parts: int, seed: int):
    """partition_vertices (partition.cpp:191-198): (assignment, edge_cut, boundary_total)."""
    out = np.zeros(ds.num_vertices, np.uint32)
    cut, bt = C.c_uint64(), C.c_uint64()
    _gs(_L().gs_partition_vertices(ds._h, num_parts, seed, _ptr(out, C.c_uint32), C.byref(cut), C.byref(bt)))
    return out, cut.value, bt.value


def shuffle_chunk_order(num_chunks: int, epoch: int, seed: int) -> np.ndarray:
    """shuffle_chunk_order (partition.cpp:239-248)."""
    out = np.zeros(num_chunks, np.uint32)
    _gs(_L().gs_shuffle_chunk_order(num_chunks, epoch, seed, _ptr(out, C.c_uint32)))
    return out


def save_assignment(path: str, num_parts: int, assignment) -> None:
    """save_assignment (partition.cpp:250-256): chunks.txt / parts.txt."""
    a = np.ascontiguousarray(assignment, np.uint32)
    _gs(_L().gs_save_assignment(path.encode(), num_parts, _ptr(a, C.c_uint32), a.size))


def load_assignment(path: str):
    """load_assignment (partition.cpp:258-267): (num_parts, assignment)."""
    parts, n = C.c_uint32(), C.c_uint64()
    _gs(_L().gs_load_assignment(path.encode(), C.byref(parts), None, 0, C.byref(n)))
    a = np.zeros(n.value, np.uint32)
    _gs(_L().gs_load_assignment(path.encode(), C.byref(parts), _ptr(a, C.c_uint32), a.size, C.byref(n)))
    return int(parts.value), a


def make_stage_assignment(layers: int, stages: int):
    """make_stage_assignment (engines.cpp:8-21): list of [begin, end)."""
    out = np.zeros(2 * stages, np.uint32)
    _gs(_L().gs_make_stage_assignment(layers, stages, _ptr(out, C.c_uint32)))
    return [(int(out[2 * s]), int(out[2 * s + 1])) for s in range(stages)]


# ----------------------------------------------------------------------------- trainers
@dataclass
class TrainResult:
    """TrainResult (engines.hpp:59-67)."""
    metrics: np.ndarray          # T x [epoch, train_loss, train_acc, val_acc, test_acc, wall_time_s, bubble]
    comm: np.ndarray             # T x [graph, pipeline, weightsync] bytes
    params: list                 # [(W, b)]
    profile: dict
    peak_buffer_bytes: int
    trace: np.ndarray = field(default_factory=lambda: np.zeros(0, TRACE_DTYPE))  # TRACE_DTYPE records
    ledger: np.ndarray = field(default_factory=lambda: np.zeros((0, 6, 2), np.uint64))  # T x tag x link bytes

    @property
    def train_loss(self) -> np.ndarray:
        return self.metrics[:, 1]


def bubble_analysis(trace: np.ndarray) -> dict:
    """bubble_analysis (analytics.cpp:59-86) over a measured trace."""
    tr = np.ascontiguousarray(trace, TRACE_DTYPE)
    out = gs_bubble_report()
    _gs(_L().gs_bubble_analysis(tr.ctypes.data_as(C.c_void_p), tr.size, C.byref(out)))
    return {"measured_bubble": out.measured_bubble, "ideal_bubble": out.ideal_bubble, "stages": out.stages,
            "chunks": out.chunks, "span": out.span}


def comm_volumes(n, layers, hidden, stages=1, ways=1, alpha=0.0, vecs=1, bytes_per_value=4) -> dict:
    """volume_graph / volume_pipeline / volume_hybrid (analytics.cpp:12-24), bytes per epoch."""
    c = gs_comm_model_input(n, layers, hidden, stages, ways, alpha, vecs, bytes_per_value)
    g, p, h = C.c_double(), C.c_double(), C.c_double()
    _gs(_L().gs_comm_volumes(C.byref(c), C.byref(g), C.byref(p), C.byref(h)))
    return {"graph": g.value, "pipeline": p.value, "hybrid": h.value}


def save_stage_checkpoint(path: str, model: "ModelConfig", in_features: int, num_classes: int, params,
                          lo: int, hi: int) -> None:
    """save_stage_checkpoint (nn.hpp:511-531): layers [lo, hi) in the reference's checkpoint format."""
    flat = np.concatenate([np.concatenate([np.ascontiguousarray(W, np.float32).ravel(),
                                           np.ascontiguousarray(b if b is not None else [], np.float32).ravel()])
                           for W, b in params]).astype(np.float32)
    _gs(_L().gs_save_stage_checkpoint(path.encode(), C.byref(model.c()), in_features, num_classes,
                                      _ptr(flat, C.c_float), lo, hi))


def load_checkpoint(path: str):
    """load_checkpoint (nn.cpp:104-124): [(name, float32 array of shape (rows, cols))]."""
    lib = _L()
    nt, nf = C.c_uint64(), C.c_uint64()
    _gs(lib.gs_load_checkpoint(path.encode(), None, 0, None, None, C.byref(nt), C.byref(nf)))
    shapes = np.zeros(2 * nt.value, np.uint64)
    data = np.zeros(nf.value, np.float32)
    nb = C.c_uint64()
    _gs(lib.gs_checkpoint_names_bytes(path.encode(), C.byref(nb)))
    names = C.create_string_buffer(int(nb.value))
    _gs(lib.gs_load_checkpoint(path.encode(), names, len(names), _ptr(shapes, C.c_uint64), _ptr(data, C.c_float),
                               C.byref(nt), C.byref(nf)))
    out, at = [], 0
    for i, name in enumerate(names.value.decode().split("\n") if nt.value else []):
        r, c = int(shapes[2 * i]), int(shapes[2 * i + 1])
        out.append((name, data[at:at + r * c].reshape(r, c).copy()))
        at += r * c
    return out


@dataclass
class CommModelInput:
    """CommModelInput (analytics.hpp:14-24)."""
    n: float = 0
    layers: float = 0
    hidden: float = 0
    stages: float = 1
    ways: float = 1
    alpha: float = 0
    vecs: float = 1
    bytes_per_value: float = 4

    def c(self) -> gs_comm_model_input:
        return gs_comm_model_input(self.n, self.layers, self.hidden, self.stages, self.ways, self.alpha, self.vecs,
                                   self.bytes_per_value)


def crossover_report(graph_in: CommModelInput, pipe_in: CommModelInput, hybrid_in: CommModelInput) -> dict:
    """crossover_report (analytics.cpp:26-56): predicted bytes, ordering, winner, inequalities."""
    b = np.zeros(3, np.float64)
    buf = C.create_string_buffer(4096)
    _gs(_L().gs_crossover_report(C.byref(graph_in.c()), C.byref(pipe_in.c()), C.byref(hybrid_in.c()),
                                 _ptr(b, C.c_double), buf, len(buf)))
    lines = buf.value.decode().split("\n")
    return {"bytes_graph": b[0], "bytes_pipeline": b[1], "bytes_hybrid": b[2], "winner": lines[0],
            "ordering": lines[1].split(","), "tie": lines[2] == "1", "inequalities": lines[3:]}


def write_compare_csv(path: str, rows) -> None:
    """write_compare_csv (analytics.cpp:88-103); rows: dicts with mode, n, layers, hidden, stages, ways,
    alpha, vecs, predicted_bytes, measured_bytes, rel_error."""
    keys = ("n", "layers", "hidden", "stages", "ways", "alpha", "vecs", "predicted_bytes", "rel_error")
    vals = np.array([[float(r[k]) for k in keys] for r in rows], np.float64).reshape(-1, 9)
    meas = np.array([int(r["measured_bytes"]) for r in rows], np.uint64)
    modes = "\n".join(r["mode"] for r in rows).encode()
    _gs(_L().gs_write_compare_csv(path.encode(), modes, _ptr(vals, C.c_double), _ptr(meas, C.c_uint64), len(rows)))


def write_run_outputs(res: "TrainResult", out_dir: str) -> None:
    """metrics.csv, trace.jsonl and comm_report.csv of a run (gnnsim.cpp:242-258 formats)."""
    os.makedirs(out_dir, exist_ok=True)
    lib = _L()
    met = np.ascontiguousarray(res.metrics, np.float64)
    comm = np.ascontiguousarray(res.comm, np.uint64)
    _gs(lib.gs_write_metrics_csv(os.path.join(out_dir, "metrics.csv").encode(), _ptr(met, C.c_double),
                                 _ptr(comm, C.c_uint64), met.shape[0]))
    tr = np.ascontiguousarray(res.trace, TRACE_DTYPE)
    _gs(lib.gs_write_trace_jsonl(os.path.join(out_dir, "trace.jsonl").encode(), tr.ctypes.data_as(C.c_void_p),
                                 tr.size))
    led = np.ascontiguousarray(res.ledger, np.uint64)
    _gs(lib.gs_write_comm_report_csv(os.path.join(out_dir, "comm_report.csv").encode(), _ptr(led, C.c_uint64),
                                     led.shape[0]))


def _result(h, specs) -> TrainResult:
    lib = _L()
    try:
        T = C.c_uint32()
        _gs(lib.gs_result_metrics(h, C.byref(T), None, None))
        met = np.zeros((T.value, 7), np.float64)
        comm = np.zeros((T.value, 3), np.uint64)
        _gs(lib.gs_result_metrics(h, C.byref(T), _ptr(met, C.c_double), _ptr(comm, C.c_uint64)))
        flat = np.zeros(_param_count(specs), np.float32)
        _gs(lib.gs_result_params(h, _ptr(flat, C.c_float)))
        pr = gp_profile()
        _gs(lib.gs_result_profile(h, C.byref(pr)))
        peak = C.c_uint64()
        _gs(lib.gs_result_peak_bytes(h, C.byref(peak)))
        prof = {name: {"ms": pr.ms[i], "launches": pr.launches[i], "alg_bytes": pr.alg_bytes[i],
                       "flops": pr.flops[i], "gather_bytes": pr.gather_bytes[i],
                       "span_ms": pr.span_ms[i]}
                for i, name in enumerate(PROFILE_CLASSES)}
        n = C.c_uint64()
        _gs(lib.gs_result_trace(h, None, 0, C.byref(n)))
        trace = np.zeros(n.value, TRACE_DTYPE)
        if n.value:
            _gs(lib.gs_result_trace(h, trace.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
        ledger = np.zeros((T.value, 6, 2), np.uint64)
        _gs(lib.gs_result_ledger(h, _ptr(ledger, C.c_uint64)))
        return TrainResult(met, comm, _split_params(specs, flat), prof, peak.value, trace, ledger)
    finally:
        lib.gs_result_free(h)


def train_pipeline(ds: Dataset, chunk_of: np.ndarray, num_stages: int, opt: TrainOptions) -> TrainResult:
    """train_pipeline<float> (engines.hpp:89-92) on the GPU engine."""
    co = np.ascontiguousarray(chunk_of, np.uint32)
    K = int(co.max()) + 1 if co.size else 0
    h = C.c_void_p()
    _gs(_L().gs_train_pipeline(ds._h, _ptr(co, C.c_uint32), K, num_stages, C.byref(opt.c()), C.byref(h)))
    return _result(h, build_layer_specs(opt.model, ds.num_features, ds.num_classes))


def train_hybrid(ds: Dataset, part_of: np.ndarray, chunk_of: np.ndarray, num_stages: int,
                 opt: TrainOptions) -> TrainResult:
    """train_hybrid<float> (engines.hpp:96-99): S pipeline stages x G graph partitions."""
    po = np.ascontiguousarray(part_of, np.uint32)
    co = np.ascontiguousarray(chunk_of, np.uint32)
    K = int(co.max()) + 1 if co.size else 0
    h = C.c_void_p()
    _gs(_L().gs_train_hybrid(ds._h, _ptr(po, C.c_uint32), _ptr(co, C.c_uint32), K, num_stages, C.byref(opt.c()),
                             C.byref(h)))
    return _result(h, build_layer_specs(opt.model, ds.num_features, ds.num_classes))


def train_graph_parallel(ds: Dataset, part_of: np.ndarray, opt: TrainOptions) -> TrainResult:
    """train_graph_parallel<float> (engines.hpp:83-87): hybrid at S = 1, K = 1."""
    po = np.ascontiguousarray(part_of, np.uint32)
    h = C.c_void_p()
    _gs(_L().gs_train_graph_parallel(ds._h, _ptr(po, C.c_uint32), C.byref(opt.c()), C.byref(h)))
    return _result(h, build_layer_specs(opt.model, ds.num_features, ds.num_classes))


def train_sequential(ds: Dataset, opt: TrainOptions) -> TrainResult:
    """train_sequential<float> (engines.hpp:79-81): the S=1, K=1 pipeline on the GPU."""
    h = C.c_void_p()
    _gs(_L().gs_train_sequential(ds._h, C.byref(opt.c()), C.byref(h)))
    return _result(h, build_layer_specs(opt.model, ds.num_features, ds.num_classes))


# ----------------------------------------------------------------------------- stage engine
def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _gp(_L().gp_nccl_unique_id(buf))
    return bytes(buf)


def _stage_config(specs_c, *, num_vertices, num_chunks, specs, stage, num_stages, layer_range, hidden,
                  num_classes, dropout, seed, lr=1e-3, optimizer="adam", fix_alpha=10, historical_gradients=False,
                  synchronous_mode=False, device=0, beta1=0.9, beta2=0.999, eps=1e-8, group_size=1, group_rank=0):
    cfg = gp_stage_config()
    cfg.device = device
    cfg.num_vertices = num_vertices
    cfg.num_chunks = num_chunks
    cfg.num_stages = num_stages
    cfg.stage = stage
    cfg.layer_begin, cfg.layer_end = layer_range
    cfg.num_layers = len(specs)
    cfg.specs = specs_c
    cfg.hidden = hidden
    cfg.num_classes = num_classes
    cfg.dropout = dropout
    cfg.seed = seed
    cfg.optimizer = 1 if optimizer == "sgd" else 0
    cfg.lr, cfg.beta1, cfg.beta2, cfg.eps = lr, beta1, beta2, eps
    cfg.fix_alpha = fix_alpha
    cfg.historical_gradients = int(historical_gradients)
    cfg.synchronous_mode = int(synchronous_mode)
    cfg.group_size = group_size
    cfg.group_rank = group_rank
    return cfg


def _specs_c(specs):
    return (gp_layer_spec * len(specs))(*[gp_layer_spec(s.kind, s.in_dim, s.out_dim, int(s.relu), s.alpha, s.beta)
                                          for s in specs])


def stage_footprint(*, nnz_norm: int, num_features: int = 0, **stage_kw) -> int:
    """Device bytes one stage (or hybrid worker) would allocate: gp_stage_footprint, the
    engine's own stash layout pass plus graph / features / labels. Needs no GPU. Takes the
    StageEngine keyword arguments (specs, num_vertices, num_chunks, stage, ...)."""
    sc = _specs_c(stage_kw["specs"])
    cfg = _stage_config(sc, **stage_kw)
    out = C.c_uint64()
    rc = _L().gp_stage_footprint(C.byref(cfg), nnz_norm, num_features, C.byref(out))
    if rc != GP_OK:
        raise _ERR.get(rc, GnnsimError)((_L().gp_last_error(None) or b"").decode())
    return int(out.value)


class StageEngine:
    """One pipeline stage on one GPU, driven directly through the gp_* C-ABI."""

    def __init__(self, *, num_vertices: int, num_chunks: int, specs: Sequence[LayerSpec], stage: int,
                 num_stages: int, layer_range, hidden: int, num_classes: int, dropout: float, seed: int,
                 lr: float = 1e-3, optimizer: str = "adam", fix_alpha: int = 10,
                 historical_gradients: bool = False, synchronous_mode: bool = False, device: int = 0,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, group_size: int = 1,
                 group_rank: int = 0):
        self.specs = list(specs)
        self._specs_c = _specs_c(specs)
        cfg = gp_stage_config()
        cfg.device = device
        cfg.num_vertices = num_vertices
        cfg.num_chunks = num_chunks
        cfg.num_stages = num_stages
        cfg.stage = stage
        cfg.layer_begin, cfg.layer_end = layer_range
        cfg.num_layers = len(specs)
        cfg.specs = self._specs_c
        cfg.hidden = hidden
        cfg.num_classes = num_classes
        cfg.dropout = dropout
        cfg.seed = seed
        cfg.optimizer = 1 if optimizer == "sgd" else 0
        cfg.lr, cfg.beta1, cfg.beta2, cfg.eps = lr, beta1, beta2, eps
        cfg.fix_alpha = fix_alpha
        cfg.historical_gradients = int(historical_gradients)
        cfg.synchronous_mode = int(synchronous_mode)
        cfg.group_size = group_size
        cfg.group_rank = group_rank
        self.n, self.K, self.stage, self.S = num_vertices, num_chunks, stage, num_stages
        self.G, self.grank = group_size, group_rank
        self.layer_range = tuple(layer_range)
        self.hidden = hidden
        h = C.c_void_p()
        rc = _L().gp_create(C.byref(cfg), C.byref(h))
        if rc != GP_OK:
            raise _ERR.get(rc, GnnsimError)((_L().gp_last_error(None) or b"").decode())
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _L().gp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload_partition(self, part_of):
        """Partition::assignment (hybrid, group_size > 1); call before upload_graph."""
        p = np.ascontiguousarray(part_of, np.uint32)
        _gp(_L().gp_upload_partition(self._h, _ptr(p, C.c_uint32)), self._h)

    def group_export(self) -> bytes:
        """This hybrid member's group blob (gp_group_export): share it with the other
        members of the stage group, then call link_group_ipc."""
        n = C.c_uint64()
        _gp(_L().gp_group_export(self._h, None, 0, C.byref(n)), self._h)
        buf = (C.c_uint8 * n.value)()
        _gp(_L().gp_group_export(self._h, buf, n.value, C.byref(n)), self._h)
        return bytes(buf)

    def link_group_ipc(self, blobs):
        """blobs[r] = group member r's blob (own entry ignored; may be None)."""
        G = len(blobs)
        arrs = [(C.c_uint8 * len(b)).from_buffer_copy(b) if b else None for b in blobs]
        ptrs = (C.POINTER(C.c_uint8) * G)(*[C.cast(a, C.POINTER(C.c_uint8)) if a is not None else None
                                          for a in arrs])
        lens = (C.c_uint64 * G)(*[len(b) if b else 0 for b in blobs])
        _gp(_L().gp_link_group_ipc(self._h, ptrs, lens), self._h)

    def upload_graph(self, offsets, cols, vals, chunk_of):
        off = np.ascontiguousarray(offsets, np.uint64)
        c = np.ascontiguousarray(cols, np.uint32)
        v = np.ascontiguousarray(vals, np.float32)
        co = np.ascontiguousarray(chunk_of, np.uint32)
        _gp(_L().gp_upload_graph(self._h, _ptr(off, C.c_uint64), _ptr(c, C.c_uint32), _ptr(v, C.c_float),
                                 c.size, _ptr(co, C.c_uint32)), self._h)

    def upload_graph_raw(self, offsets, neighbors, chunk_of, self_loops: bool = True):
        """gp_upload_graph_raw: the graph's own CSR (Dataset.graph()); normalize_adjacency<float>
        is applied while the packed CSR is built (on the device for large graphs)."""
        off = np.ascontiguousarray(offsets, np.uint64)
        nb = np.ascontiguousarray(neighbors, np.uint32)
        co = np.ascontiguousarray(chunk_of, np.uint32)
        _gp(_L().gp_upload_graph_raw(self._h, _ptr(off, C.c_uint64), _ptr(nb, C.c_uint32), nb.size,
                                     int(self_loops), _ptr(co, C.c_uint32)), self._h)

    def share_graph(self, owner: "StageEngine"):
        _gp(_L().gp_share_graph(self._h, owner._h), self._h)

    def upload_features(self, x):
        x = np.ascontiguousarray(x, np.float32)
        _gp(_L().gp_upload_features(self._h, _ptr(x, C.c_float), x.shape[1]), self._h)

    def upload_labels(self, labels, split):
        lab = np.ascontiguousarray(labels, np.uint32)
        sp = np.ascontiguousarray(split, np.uint8)
        _gp(_L().gp_upload_labels(self._h, _ptr(lab, C.c_uint32), _ptr(sp, C.c_uint8)), self._h)

    def set_params(self, layer: int, W, b=None):
        W = np.ascontiguousarray(W, np.float32)
        bp = None
        if b is not None and np.size(b):
            b = np.ascontiguousarray(b, np.float32)
            bp = _ptr(b, C.c_float)
        _gp(_L().gp_set_layer_params(self._h, layer, _ptr(W, C.c_float), bp), self._h)

    def get_params(self, layer: int):
        s = self.specs[layer]
        W = np.zeros((s.k_in, s.out_dim), np.float32)
        b = np.zeros(s.out_dim if s.has_bias else 0, np.float32)
        _gp(_L().gp_get_layer_params(self._h, layer, _ptr(W, C.c_float), _ptr(b, C.c_float) if b.size else None),
            self._h)
        return W, b

    def get_grads(self, layer: int):
        s = self.specs[layer]
        W = np.zeros((s.k_in, s.out_dim), np.float32)
        b = np.zeros(s.out_dim if s.has_bias else 0, np.float32)
        _gp(_L().gp_get_layer_grads(self._h, layer, _ptr(W, C.c_float), _ptr(b, C.c_float) if b.size else None),
            self._h)
        return W, b

    def link_local(self, downstream: "StageEngine"):
        _gp(_L().gp_link_local(self._h, downstream._h), downstream._h)

    def link_nccl(self, up_id: Optional[bytes], down_id: Optional[bytes]):
        up = (C.c_uint8 * 128).from_buffer_copy(up_id) if up_id else None
        down = (C.c_uint8 * 128).from_buffer_copy(down_id) if down_id else None
        _gp(_L().gp_link_nccl(self._h, up, down), self._h)

    def ipc_export(self):
        """Ring regions for the CUDA-IPC transport: (up_blob, down_blob), None for a
        missing side. Call after upload_graph; exchange the blobs out of band."""
        first, last = self.stage == 0, self.stage == self.S - 1
        up = (C.c_uint8 * IPC_BLOB_BYTES)() if not first else None
        down = (C.c_uint8 * IPC_BLOB_BYTES)() if not last else None
        _gp(_L().gp_ipc_export(self._h, up, down), self._h)
        return (bytes(up) if up is not None else None, bytes(down) if down is not None else None)

    def link_ipc(self, up_peer: Optional[bytes], down_peer: Optional[bytes]):
        """Link to the neighbour stages' exported blobs: `up_peer` is the `down` blob
        of stage s-1, `down_peer` the `up` blob of stage s+1."""
        up = (C.c_uint8 * IPC_BLOB_BYTES).from_buffer_copy(up_peer) if up_peer else None
        down = (C.c_uint8 * IPC_BLOB_BYTES).from_buffer_copy(down_peer) if down_peer else None
        _gp(_L().gp_link_ipc(self._h, up, down), self._h)

    def abort(self):
        _L().gp_abort(self._h)

    def run_epoch(self, t: int, order) -> gp_epoch_stats:
        o = np.ascontiguousarray(order, np.uint32)
        st = gp_epoch_stats()
        _gp(_L().gp_run_epoch(self._h, t, _ptr(o, C.c_uint32), C.byref(st)), self._h)
        return st

    def download(self, which: str, local_layer: int = 0) -> np.ndarray:
        lo, hi = self.layer_range
        if which in ("h", "dz", "hsnap"):
            width = self.specs[lo + local_layer].out_dim
        elif which in ("pre", "dagg"):
            width = self.specs[lo + local_layer].k_in
        elif which == "gather":
            width = self.specs[lo + local_layer].in_dim
        elif which == "dh0":
            width = self.hidden
        else:
            width = self.specs[lo].in_dim
        out = np.zeros((self.n, width), np.float32)
        _gp(_L().gp_download(self._h, GP_BUF[which], local_layer, _ptr(out, C.c_float), out.size), self._h)
        return out

    def set_profiling(self, on: bool = True):
        _L().gp_set_profiling(self._h, int(on))

    def set_live_timing(self, kernel_class: Optional[str]):
        """Events around every launch of one kernel class during normal epochs ("all": every
        class, None = off)."""
        cls = -1 if kernel_class is None else (len(PROFILE_CLASSES) if kernel_class == "all"
                                                else PROFILE_CLASSES.index(kernel_class))
        _gp(_L().gp_set_live_timing(self._h, cls), self._h)

    def reset_profile(self):
        _L().gp_reset_profile(self._h)

    def profile(self) -> dict:
        pr = gp_profile()
        _L().gp_get_profile(self._h, C.byref(pr))
        return {name: {"ms": pr.ms[i], "launches": pr.launches[i], "alg_bytes": pr.alg_bytes[i],
                       "flops": pr.flops[i], "gather_bytes": pr.gather_bytes[i],
                       "span_ms": pr.span_ms[i]}
                for i, name in enumerate(PROFILE_CLASSES)}

    def mark(self, slot: int):
        _gp(_L().gp_mark(self._h, slot), self._h)

    def elapsed_ms(self, a: int, b: int) -> float:
        v = C.c_float()
        _gp(_L().gp_elapsed(self._h, a, b, C.byref(v)), self._h)
        return v.value

    def synchronize(self):
        _gp(_L().gp_synchronize(self._h), self._h)

    def device_bytes(self) -> int:
        v = C.c_uint64()
        _L().gp_device_bytes(self._h, C.byref(v))
        return v.value
