"""ctypes front-end of the C restatement (oracle/gnnsim_oracle.c -> oracle/_ref/liboracle.so).

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py cpu_baseline)."""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: make -C oracle oracle-c")
        L = C.CDLL(LIB)
        P = C.POINTER
        vp, u32p, u64p, f32p, f64p, u8p = C.c_void_p, P(C.c_uint32), P(C.c_uint64), P(C.c_float), P(C.c_double), P(C.c_uint8)
        sig = {
            "or_synthetic_er": (vp, [C.c_uint32, C.c_double, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]),
            "or_from_edges": (vp, [C.c_uint32, u32p, C.c_uint64, f32p, C.c_uint32, u32p, C.c_uint32, u8p]),
            "or_free": (None, [vp]),
            "or_shape": (None, [vp, u32p, u64p]),
            "or_graph": (None, [vp, u64p, u32p, u32p]),
            "or_arrays": (None, [vp, f32p, u32p, u8p]),
            "or_normalize": (None, [vp, C.c_int, u64p, u32p, f32p]),
            "or_partition": (C.c_int, [vp, C.c_uint32, C.c_uint64, u32p]),
            "or_shuffle": (None, [C.c_uint32, C.c_uint64, C.c_uint64, u32p]),
            "or_stage_ranges": (None, [C.c_uint32, C.c_uint32, u32p]),
            "or_init_params": (None, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, f32p]),
            "or_dropmask_bits": (C.c_uint64, [C.c_double, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, u64p]),
            "or_train_data": (C.c_int, [vp, u32p, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32, C.c_uint32, C.c_double,
                                        C.c_uint64, C.c_uint32, C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                        C.c_double, f64p, u64p, f32p, f32p]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class OracleData:
    def __init__(self, h):
        self.h = h
        n, m = C.c_uint32(), C.c_uint64()
        lib().or_shape(h, C.byref(n), C.byref(m))
        self.n, self.m = n.value, m.value

    @staticmethod
    def synthetic_er(n, p, gseed, F, Cc, fseed):
        d = OracleData(lib().or_synthetic_er(n, p, gseed, F, Cc, fseed))
        d.F, d.C = F, Cc
        return d

    @staticmethod
    def from_edges(n, edges, x, lab, Cc, split):
        e = np.ascontiguousarray(np.asarray(edges, np.uint32).reshape(-1, 2))
        x = np.ascontiguousarray(x, np.float32).reshape(n, -1)
        lab = np.ascontiguousarray(lab, np.uint32)
        sp = np.ascontiguousarray(split, np.uint8)
        d = OracleData(lib().or_from_edges(n, _p(e, C.c_uint32), e.shape[0], _p(x, C.c_float), x.shape[1],
                                           _p(lab, C.c_uint32), Cc, _p(sp, C.c_uint8)))
        d.F, d.C = x.shape[1], Cc
        return d

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_free(self.h)
            self.h = None

    def graph(self):
        off = np.zeros(self.n + 1, np.uint64)
        nb = np.zeros(2 * self.m, np.uint32)
        dg = np.zeros(self.n, np.uint32)
        lib().or_graph(self.h, _p(off, C.c_uint64), _p(nb, C.c_uint32), _p(dg, C.c_uint32))
        return off, nb, dg

    def arrays(self):
        x = np.zeros((self.n, self.F), np.float32)
        lab = np.zeros(self.n, np.uint32)
        sp = np.zeros(self.n, np.uint8)
        lib().or_arrays(self.h, _p(x, C.c_float), _p(lab, C.c_uint32), _p(sp, C.c_uint8))
        return x, lab, sp

    def normalize(self, loops=True):
        nnz = 2 * self.m + (self.n if loops else 0)
        off = np.zeros(self.n + 1, np.uint64)
        col = np.zeros(nnz, np.uint32)
        val = np.zeros(nnz, np.float32)
        lib().or_normalize(self.h, int(loops), _p(off, C.c_uint64), _p(col, C.c_uint32), _p(val, C.c_float))
        return off, col, val

    def partition(self, parts, seed):
        out = np.zeros(self.n, np.uint32)
        if lib().or_partition(self.h, parts, seed, _p(out, C.c_uint32)) != 0:
            raise ValueError("partition: need 1 <= parts <= N")
        return out

    def train(self, chunk_of, K, S, model, layers, hidden, seed, epochs, dropout=0.5, shuffle=True, fix_alpha=10,
              hist=False, sync=False, sgd=False, lr=1e-3, want_h=False, num_params=None, h_size=None):
        co = np.ascontiguousarray(chunk_of, np.uint32)
        met = np.zeros((epochs, 5), np.float64)
        comm = np.zeros(epochs, np.uint64)
        params = np.zeros(num_params, np.float32)
        h = np.zeros(h_size, np.float32) if want_h else None
        rc = lib().or_train_data(self.h, _p(co, C.c_uint32), K, S, model, layers, hidden, dropout, seed, epochs,
                                 int(shuffle), fix_alpha, int(hist), int(sync), int(sgd), lr, _p(met, C.c_double),
                                 _p(comm, C.c_uint64), _p(params, C.c_float), _p(h, C.c_float) if want_h else None)
        if rc != 0:
            raise ValueError("oracle train: empty train mask")
        return met, comm, params, h


def shuffle(K, epoch, seed):
    out = np.zeros(K, np.uint32)
    lib().or_shuffle(K, epoch, seed, _p(out, C.c_uint32))
    return out


def stage_ranges(L, S):
    out = np.zeros(2 * S, np.uint32)
    lib().or_stage_ranges(L, S, _p(out, C.c_uint32))
    return [(int(out[2 * s]), int(out[2 * s + 1])) for s in range(S)]


def init_params(model, layers, hidden, F, Cc, seed, count):
    out = np.zeros(count, np.float32)
    lib().or_init_params(model, layers, hidden, F, Cc, seed, _p(out, C.c_float))
    return out


def dropmask(rate, seed, epoch, layer, n, cols):
    words = lib().or_dropmask_bits(rate, seed, epoch, layer, n, cols, None)
    out = np.zeros(words, np.uint64)
    lib().or_dropmask_bits(rate, seed, epoch, layer, n, cols, _p(out, C.c_uint64))
    return out
