"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two checkers.

* ``Oracle``: our plain-C restatement of the hot path (oracle/paillier_oracle.c,
  built into oracle/_build/libpaillier_oracle.so; rebuilt on demand with gcc,
  which exists on the GPU box too).
* ``Reference``: the unmodified reference library compiled by oracle/Makefile
  into oracle/_ref/ (only present when the dev container built it; the .so
  files travel to the GPU box with the repo snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg
import this module.  The product path (paper_2504_03909_b200) never does.

Numbers cross both boundaries as little-endian u32 limbs (numpy uint32).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libpaillier_oracle.so")
REF_CAPI_SO = os.path.join(HERE, "_ref", "libsfxb_refcapi.so")

_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


# ---------------------------------------------------------------- limbs


def to_words(x: int, words: int) -> np.ndarray:
    if x < 0 or x.bit_length() > 32 * words:
        raise ValueError("value does not fit")
    return np.frombuffer(x.to_bytes(4 * words, "little"), dtype=np.uint32).copy()


def from_words(w) -> int:
    return int.from_bytes(np.ascontiguousarray(w, dtype=np.uint32).tobytes(), "little")


def ints_to_words(xs, words: int) -> np.ndarray:
    out = np.zeros((len(xs), words), dtype=np.uint32)
    for i, x in enumerate(xs):
        out[i] = to_words(int(x), words)
    return out


def words_to_ints(arr) -> list[int]:
    arr = np.ascontiguousarray(arr, dtype=np.uint32)
    return [from_words(r) for r in arr.reshape(arr.shape[0], -1)]


# ---------------------------------------------------------------- oracle


def build_oracle() -> str:
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(
        os.path.join(HERE, "paillier_oracle.c")
    ):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    return ORACLE_SO


class OracleError(RuntimeError):
    pass


class Oracle:
    """Plain-C restatement (oracle/paillier_oracle.c)."""

    def __init__(self):
        lib = C.CDLL(build_oracle())
        self.lib = lib
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_key_id_of.restype = C.c_uint64
        lib.orc_key_id_of.argtypes = [_u32p, C.c_size_t]
        lib.orc_key_new.restype = C.c_void_p
        lib.orc_key_new.argtypes = [_u32p, C.c_void_p, C.c_void_p, C.c_size_t]
        lib.orc_key_free.argtypes = [C.c_void_p]
        lib.orc_key_id.restype = C.c_uint64
        lib.orc_key_id.argtypes = [C.c_void_p]
        lib.orc_rng_new.restype = C.c_void_p
        lib.orc_rng_new.argtypes = [C.c_uint64]
        lib.orc_rng_free.argtypes = [C.c_void_p]
        lib.orc_rng_draw.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, _u32p]
        lib.orc_encode_fixed.argtypes = [C.c_void_p, C.c_double, C.c_uint, _u32p, C.POINTER(C.c_int64)]
        lib.orc_decode_fixed.restype = C.c_double
        lib.orc_decode_fixed.argtypes = [C.c_void_p, _u32p, C.c_uint]
        lib.orc_encrypt_with_r.argtypes = [C.c_void_p, _u32p, _u32p, _u32p]
        lib.orc_encrypt_gh.argtypes = [C.c_void_p, C.c_void_p, _f64p, C.c_size_t, C.c_uint, _u32p,
                                       C.POINTER(C.c_uint64)]
        lib.orc_accumulate.argtypes = [C.c_void_p, _u32p, C.c_uint32, _u16p, C.c_uint32, _u32p,
                                       C.c_uint32, _u32p, C.c_uint32, _u32p, C.POINTER(C.c_uint64)]
        lib.orc_decrypt.argtypes = [C.c_void_p, _u32p, _u32p]
        lib.orc_decrypt_crt.argtypes = [C.c_void_p, _u32p, _u32p]
        lib.orc_decrypt_slots.argtypes = [C.c_void_p, _u32p, C.c_size_t, C.c_uint, _f64p,
                                          C.POINTER(C.c_uint64)]
        lib.orc_decode_int_sum.restype = C.c_double
        lib.orc_decode_int_sum.argtypes = [C.c_void_p, _i64p, C.c_size_t, C.c_uint]
        lib.orc_intsum_hist.argtypes = [C.c_void_p, _i64p, C.c_uint32, _u16p, C.c_uint32, _u32p, C.c_uint32,
                                        _u32p, C.c_uint32, C.c_uint, _f64p, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64)]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.orc_last_error().decode())


class OracleKey:
    """orc_key: n (and optionally p, q) — he.hpp:11-27."""

    def __init__(self, oracle: Oracle, n: int, p: int | None = None, q: int | None = None,
                 nw: int | None = None):
        self.o = oracle
        self.n, self.p, self.q = n, p, q
        self.nw = nw or max(1, (n.bit_length() + 31) // 32)
        self.n2 = n * n
        nwords = to_words(n, self.nw)
        if p is not None:
            pw, qw = to_words(p, self.nw), to_words(q, self.nw)
            self.h = oracle.lib.orc_key_new(nwords, pw.ctypes.data, qw.ctypes.data, self.nw)
        else:
            self.h = oracle.lib.orc_key_new(nwords, None, None, self.nw)
        if not self.h:
            raise OracleError(oracle.lib.orc_last_error().decode())
        self.key_id = oracle.lib.orc_key_id(self.h)

    def __del__(self):
        try:
            self.o.lib.orc_key_free(self.h)
        except Exception:
            pass

    def encode_fixed(self, x: float, scale: int = 40):
        out = np.zeros(self.nw, np.uint32)
        q = C.c_int64()
        self.o._check(self.o.lib.orc_encode_fixed(self.h, float(x), scale, out, C.byref(q)))
        return from_words(out), q.value

    def decode_fixed(self, m: int, scale: int = 40) -> float:
        return self.o.lib.orc_decode_fixed(self.h, to_words(m, self.nw), scale)

    def encrypt_with_r(self, m: int, r: int) -> int:
        out = np.zeros(2 * self.nw, np.uint32)
        self.o._check(self.o.lib.orc_encrypt_with_r(self.h, to_words(m, self.nw), to_words(r, self.nw), out))
        return from_words(out)

    def rng_draw(self, seed: int, count: int) -> np.ndarray:
        rng = self.o.lib.orc_rng_new(seed)
        out = np.zeros((count, self.nw), np.uint32)
        try:
            self.o._check(self.o.lib.orc_rng_draw(rng, self.h, count, out))
        finally:
            self.o.lib.orc_rng_free(rng)
        return out

    def encrypt_gh(self, gh: np.ndarray, seed: int, scale: int = 40):
        """gh: (count, 2) float64 → (2*count, 2*nw) uint32 ciphertexts, encryptions."""
        gh = np.ascontiguousarray(gh, dtype=np.float64)
        count = gh.shape[0]
        out = np.zeros((2 * count, 2 * self.nw), np.uint32)
        enc = C.c_uint64(0)
        rng = self.o.lib.orc_rng_new(seed)
        try:
            self.o._check(self.o.lib.orc_encrypt_gh(self.h, rng, gh.reshape(-1), count, scale, out, C.byref(enc)))
        finally:
            self.o.lib.orc_rng_free(rng)
        return out, enc.value

    def accumulate(self, cts, bins, node_offsets, rows, n_bins):
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        bins = np.ascontiguousarray(bins, dtype=np.uint16)
        J, n_samples = bins.shape
        n_nodes = len(node_offsets) - 1
        out = np.zeros((n_nodes * J * n_bins * 2, 2 * self.nw), np.uint32)
        adds = C.c_uint64(0)
        self.o._check(self.o.lib.orc_accumulate(
            self.h, cts.reshape(-1), n_samples, bins.reshape(-1), J,
            np.ascontiguousarray(node_offsets, dtype=np.uint32), n_nodes,
            np.ascontiguousarray(rows, dtype=np.uint32), n_bins, out, C.byref(adds)))
        return out, adds.value

    def decrypt(self, c: int, crt: bool = False) -> int:
        out = np.zeros(self.nw, np.uint32)
        fn = self.o.lib.orc_decrypt_crt if crt else self.o.lib.orc_decrypt
        self.o._check(fn(self.h, to_words(c, 2 * self.nw), out))
        return from_words(out)

    def decrypt_slots(self, cts, scale: int = 40):
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        out = np.zeros(cts.shape[0], np.float64)
        decs = C.c_uint64(0)
        self.o._check(self.o.lib.orc_decrypt_slots(self.h, cts.reshape(-1), cts.shape[0], scale, out, C.byref(decs)))
        return out, decs.value

    def decode_int_sum(self, terms, scale: int = 40) -> float:
        t = np.ascontiguousarray(terms, dtype=np.int64)
        return self.o.lib.orc_decode_int_sum(self.h, t, len(t), scale)

    def intsum_hist(self, q, bins, offs, rows, n_bins: int, scale: int = 40):
        """Decrypted histograms of one frontier from the plaintexts (orc_intsum_hist):
        (values N×J×K×2 doubles, reference additions, reference decryptions)."""
        q = np.ascontiguousarray(q, dtype=np.int64)
        bins = np.ascontiguousarray(bins, dtype=np.uint16)
        J = bins.shape[0]
        N = len(offs) - 1
        out = np.empty(N * J * n_bins * 2, np.float64)
        adds, decs = C.c_uint64(0), C.c_uint64(0)
        self.o._check(self.o.lib.orc_intsum_hist(
            self.h, q, len(q) // 2, bins.reshape(-1), J, np.ascontiguousarray(offs, dtype=np.uint32), N,
            np.ascontiguousarray(rows, dtype=np.uint32), n_bins, scale, out, C.byref(adds), C.byref(decs)))
        return out, adds.value, decs.value


# ---------------------------------------------------------------- reference


def reference_available() -> bool:
    return os.path.exists(REF_CAPI_SO)


class RefError(RuntimeError):
    pass


class Reference:
    """The unmodified reference library via oracle/ref_capi.cpp."""

    def __init__(self):
        if not reference_available():
            raise RefError("oracle/_ref not built (run `make -C oracle ref` in the dev container)")
        # global symbol scope, as for a program linked against the reference:
        # an interposed plugin (LD_PRELOAD) calls back into the reference's
        # public helpers (e.g. pack_plain, he.hpp)
        lib = C.CDLL(REF_CAPI_SO, mode=C.RTLD_GLOBAL)
        self.lib = lib
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_keygen.argtypes = [C.c_uint, C.c_uint64, _u32p, _u32p, _u32p, C.c_size_t]
        lib.ref_key_id.restype = C.c_uint64
        lib.ref_key_id.argtypes = [_u32p, C.c_size_t]
        lib.ref_write_private_key.argtypes = [C.c_uint, C.c_uint64, C.c_char_p, C.c_char_p]
        lib.ref_rng_draw.argtypes = [C.c_uint64, _u32p, C.c_size_t, C.c_size_t, _u32p]
        lib.ref_encrypt_with_r.argtypes = [_u32p, C.c_size_t, _u32p, _u32p, _u32p]
        lib.ref_plugin_new.restype = C.c_void_p
        lib.ref_plugin_new.argtypes = [_u32p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint]
        lib.ref_plugin_free.argtypes = [C.c_void_p]
        lib.ref_plugin_counters.argtypes = [C.c_void_p, C.POINTER(C.c_uint64 * 4)]
        lib.ref_plugin_name.restype = C.c_char_p
        lib.ref_plugin_name.argtypes = [C.c_void_p]
        lib.ref_encrypt_gh.argtypes = [C.c_void_p, _f64p, C.c_size_t, _u32p]
        lib.ref_accumulate.argtypes = [C.c_void_p, _u32p, C.c_uint32, _u16p, C.c_uint32, _i32p, _u32p,
                                       _u32p, C.c_uint32, _u32p, C.c_uint32, _u32p]
        lib.ref_decrypt_slots.argtypes = [C.c_void_p, _u32p, C.c_uint32, C.c_uint32, C.c_uint32, _f64p]
        lib.ref_accumulate_threaded.argtypes = [_u32p, C.c_size_t, _u32p, C.c_uint32, _u16p, C.c_uint32,
                                                _u32p, C.c_uint32, _u32p, C.c_uint32, C.c_int,
                                                C.POINTER(C.c_uint64)]
        lib.ref_encrypt_threaded.argtypes = [_u32p, C.c_size_t, C.c_uint32, C.c_int, C.POINTER(C.c_uint64),
                                             C.POINTER(C.c_double)]
        lib.ref_decrypt_threaded.argtypes = [_u32p, _u32p, C.c_size_t, _u32p, C.c_uint32, C.c_int,
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        lib.ref_gradients.argtypes = [_f64p, np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS"), C.c_size_t,
                                      C.c_uint, _u32p, C.c_size_t, _i64p, _f64p, C.POINTER(C.c_size_t)]
        lib.ref_train.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t,
                                  C.POINTER(C.c_uint64 * 4), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_double * 6)]

    def _check(self, rc):
        if rc != 0:
            raise RefError(self.lib.ref_last_error().decode())

    def keygen(self, bits: int, seed: int):
        nw = bits // 32
        n, p, q = (np.zeros(nw, np.uint32) for _ in range(3))
        self._check(self.lib.ref_keygen(bits, seed, n, p, q, nw))
        return from_words(n), from_words(p), from_words(q)

    def key_id(self, n: int, nw: int) -> int:
        return self.lib.ref_key_id(to_words(n, nw), nw)

    def rng_draw(self, seed: int, n: int, nw: int, count: int) -> np.ndarray:
        out = np.zeros((count, nw), np.uint32)
        self._check(self.lib.ref_rng_draw(seed, to_words(n, nw), nw, count, out))
        return out

    def encrypt_with_r(self, n: int, nw: int, m: int, r: int) -> int:
        out = np.zeros(2 * nw, np.uint32)
        self._check(self.lib.ref_encrypt_with_r(to_words(n, nw), nw, to_words(m, nw), to_words(r, nw), out))
        return from_words(out)

    def train(self, ini_text: str):
        forest = C.create_string_buffer(1 << 22)
        partials = C.create_string_buffer(1 << 22)
        counters = (C.c_uint64 * 4)()
        fnv, total = C.c_uint64(), C.c_uint64()
        phases = (C.c_double * 6)()
        self._check(self.lib.ref_train(ini_text.encode(), forest, len(forest), partials, len(partials),
                                       C.byref(counters), C.byref(fnv), C.byref(total), C.byref(phases)))
        return {
            "forest": forest.value.decode(),
            "partials": partials.value.decode(),
            "counters": list(counters),
            "transcript_fnv": fnv.value,
            "transcript_bytes": total.value,
            "phases": list(phases),
        }


class RefPlugin:
    """make_paillier_plugin from the reference library."""

    def __init__(self, ref: Reference, n: int, nw: int, p: int | None = None, q: int | None = None,
                 rng_seed: int = 1, scale_bits: int = 40):
        self.ref, self.nw, self.n = ref, nw, n
        if p is not None:
            pw, qw = to_words(p, nw), to_words(q, nw)
            self.h = ref.lib.ref_plugin_new(to_words(n, nw), pw.ctypes.data, qw.ctypes.data, nw,
                                            rng_seed, scale_bits)
        else:
            self.h = ref.lib.ref_plugin_new(to_words(n, nw), None, None, nw, rng_seed, scale_bits)
        if not self.h:
            raise RefError(ref.lib.ref_last_error().decode())

    def __del__(self):
        try:
            self.ref.lib.ref_plugin_free(self.h)
        except Exception:
            pass

    def counters(self):
        c = (C.c_uint64 * 4)()
        self.ref.lib.ref_plugin_counters(self.h, C.byref(c))
        return list(c)

    def name(self) -> str:
        return self.ref.lib.ref_plugin_name(self.h).decode()

    def encrypt_gh(self, gh: np.ndarray) -> np.ndarray:
        gh = np.ascontiguousarray(gh, dtype=np.float64)
        out = np.zeros((2 * gh.shape[0], 2 * self.nw), np.uint32)
        self.ref._check(self.ref.lib.ref_encrypt_gh(self.h, gh.reshape(-1), gh.shape[0], out))
        return out

    def accumulate(self, cts, bins, node_offsets, rows, n_bins, feature_ids=None, node_ids=None):
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        bins = np.ascontiguousarray(bins, dtype=np.uint16)
        J, n_samples = bins.shape
        n_nodes = len(node_offsets) - 1
        fids = np.arange(J, dtype=np.int32) if feature_ids is None else np.asarray(feature_ids, np.int32)
        nids = np.arange(n_nodes, dtype=np.uint32) if node_ids is None else np.asarray(node_ids, np.uint32)
        out = np.zeros((n_nodes * J * n_bins * 2, 2 * self.nw), np.uint32)
        self.ref._check(self.ref.lib.ref_accumulate(
            self.h, cts.reshape(-1), n_samples, bins.reshape(-1), J, fids,
            np.ascontiguousarray(node_offsets, dtype=np.uint32), nids, n_nodes,
            np.ascontiguousarray(rows, dtype=np.uint32), n_bins, out))
        return out

    def decrypt_slots(self, slots, n_nodes: int, n_features: int, n_bins: int) -> np.ndarray:
        slots = np.ascontiguousarray(slots, dtype=np.uint32)
        out = np.zeros(n_nodes * n_features * n_bins * 2, np.float64)
        self.ref._check(self.ref.lib.ref_decrypt_slots(self.h, slots.reshape(-1), n_nodes, n_features,
                                                       n_bins, out))
        return out
