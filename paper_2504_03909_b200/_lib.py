"""ctypes binding of libsfxb_cuda.so (the C ABI in include/sfxb_cuda.h).

This is plumbing for the Python tests and bench.py; the product boundary is
the C ABI itself (and the C++ EncryptionPlugin adapter in host/).  There is no
CPU fallback: if the shared library or a B200 is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFXB_LIB") or os.path.join(PKG, "lib", "libsfxb_cuda.so")

SFXB_OK = 0
SFXB_ERR_ARG = -1
SFXB_ERR_CUDA = -2
SFXB_ERR_AUTH = -3
SFXB_ERR_RANGE = -4
SFXB_ERR_COPRIME = -5
SFXB_ERR_UNSUPPORTED = -6


class SfxbError(RuntimeError):
    """Carries the C ABI error code and the reference-compatible message."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class AuthorizationError(SfxbError):
    """Mirrors sfxb::AuthorizationError (errors.hpp:26-28)."""


_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SfxbError(SFXB_ERR_CUDA, f"{LIB_PATH} not built (run __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    vp, sz = C.c_void_p, C.c_size_t
    sig = {
        "sfxb_ctx_create": (C.c_int, [C.POINTER(vp), C.c_int, _u32p, C.c_uint32, vp, vp, C.c_uint32]),
        "sfxb_ctx_create_multi": (C.c_int, [C.POINTER(vp), _i32p, C.c_uint32, _u32p, C.c_uint32, vp, vp,
                                            C.c_uint32]),
        "sfxb_ctx_n_shards": (C.c_uint32, [vp]),
        "sfxb_ctx_enc_wave": (C.c_size_t, [vp]),
        "sfxb_device_count": (C.c_int, []),
        "sfxb_ctx_shard_device": (C.c_int, [vp, C.c_uint32]),
        "sfxb_ctx_destroy": (None, [vp]),
        "sfxb_last_error": (C.c_char_p, [vp]),
        "sfxb_create_error": (C.c_char_p, []),
        "sfxb_ctx_n_words": (C.c_uint32, [vp]),
        "sfxb_ctx_ct_words": (C.c_uint32, [vp]),
        "sfxb_ctx_has_private": (C.c_int, [vp]),
        "sfxb_ctx_key_id": (C.c_uint64, [vp]),
        "sfxb_ctx_launches": (C.c_uint64, [vp]),
        "sfxb_ctx_dec_derived": (C.c_uint64, [vp]),
        "sfxb_ctx_stream": (vp, [vp]),
        "sfxb_ctx_sync": (C.c_int, [vp]),
        "sfxb_encrypt": (C.c_int, [vp, _i64p, _u32p, sz, _u32p, vp]),
        "sfxb_encrypt_dev": (C.c_int, [vp, vp, vp, sz, vp, vp]),
        "sfxb_encrypt_plain": (C.c_int, [vp, _u32p, _u32p, sz, _u32p, vp]),
        "sfxb_encode_check": (C.c_int, [vp, C.c_double, C.c_uint32, C.POINTER(C.c_int64)]),
        "sfxb_encode_batch": (C.c_int, [vp, _f64p, C.c_size_t, C.c_uint32, _i64p, C.POINTER(C.c_size_t)]),
        "sfxb_gradients_dev": (C.c_int, [vp, vp, vp, C.c_size_t, C.c_uint32, vp, vp, C.POINTER(C.c_size_t)]),
        "sfxb_blind_create": (C.c_int, [vp, C.c_size_t, C.POINTER(vp)]),
        "sfxb_blind_free": (None, [vp]),
        "sfxb_blind_size": (C.c_size_t, [vp]),
        "sfxb_blind_append": (C.c_int, [vp, vp, _u32p, C.c_size_t, vp]),
        "sfxb_blind_pop": (C.c_int, [vp, C.c_size_t]),
        "sfxb_encrypt_blind": (C.c_int, [vp, vp, vp, vp, C.c_size_t, _u32p]),
        "sfxb_ctx_set_low_priority": (C.c_int, [vp]),
        "sfxb_bins_upload": (C.c_int, [vp, _u16p, C.c_uint32, C.c_uint32, C.POINTER(vp)]),
        "sfxb_bins_free": (None, [vp]),
        "sfxb_accumulate_tree_bins": (C.c_int, [vp, vp, vp, _u32p, C.c_uint32, _u32p, C.c_uint32, _i32p, _u32p,
                                                C.POINTER(C.c_uint64)]),
        "sfxb_add": (C.c_int, [vp, _u32p, _u32p, sz, _u32p]),
        "sfxb_accumulate": (C.c_int, [vp, _u32p, C.c_uint32, _u16p, C.c_uint32, _u32p, C.c_uint32, _u32p,
                                      C.c_uint32, _u32p, C.POINTER(C.c_uint64)]),
        "sfxb_gh_upload": (C.c_int, [vp, _u32p, C.c_uint32, C.POINTER(vp)]),
        "sfxb_gh_from_dev": (C.c_int, [vp, vp, C.c_uint32, C.POINTER(vp)]),
        "sfxb_gh_free": (None, [vp]),
        "sfxb_accumulate_dev": (C.c_int, [vp, vp, vp, C.c_uint32, vp, C.c_uint32, vp, C.c_uint32, C.c_uint32,
                                          vp, C.c_int, C.POINTER(C.c_uint64)]),
        "sfxb_accumulate_gh": (C.c_int, [vp, vp, _u16p, C.c_uint32, _u32p, C.c_uint32, _u32p, C.c_uint32,
                                         _u32p, C.POINTER(C.c_uint64)]),
        "sfxb_accumulate_tree_dev": (C.c_int, [vp, vp, vp, C.c_uint32, vp, _u32p, C.c_uint32, vp, C.c_uint32,
                                               C.c_uint32, _i32p, vp, C.c_int, C.POINTER(C.c_uint64)]),
        "sfxb_accumulate_tree_gh": (C.c_int, [vp, vp, _u16p, C.c_uint32, _u32p, C.c_uint32, _u32p, C.c_uint32,
                                              _i32p, _u32p, C.POINTER(C.c_uint64)]),
        "sfxb_tree_reset": (C.c_int, [vp]),
        "sfxb_ctx_tree_derived": (C.c_uint64, [vp]),
        "sfxb_reduce_partials_dev": (C.c_int, [vp, vp, C.c_uint32, sz, vp]),
        "sfxb_slice_width": (C.c_uint32, [C.c_uint32, C.c_uint32, C.c_uint32]),
        "sfxb_accumulate_part_dev": (C.c_int, [vp, vp, vp, C.c_uint32, vp, _u32p, C.c_uint32, vp, C.c_uint32,
                                               C.c_uint32, vp, vp, C.c_uint32, vp, vp]),
        "sfxb_combine_slices_dev": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                              C.c_uint32, vp, vp, vp]),
        "sfxb_count_additions_dev": (C.c_int, [vp, vp, sz, C.POINTER(C.c_uint64)]),
        "sfxb_decrypt": (C.c_int, [vp, _u32p, sz, C.c_uint32, _f64p, vp, C.POINTER(C.c_uint64)]),
        "sfxb_decrypt_dev": (C.c_int, [vp, vp, sz, C.c_uint32, vp, vp, C.POINTER(C.c_uint64)]),
        "sfxb_decrypt_tree": (C.c_int, [vp, C.c_uint64, _u32p, C.c_uint32, C.c_uint32, vp, C.c_uint32, _f64p,
                                        C.POINTER(C.c_uint64)]),
        "sfxb_imad_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "sfxb_ctx_profile": (C.c_int, [vp, C.c_int]),
        "sfxb_ctx_kernel_time": (C.c_int, [vp, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
        "sfxb_ctx_kernel_stats": (C.c_int, [vp, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                            C.POINTER(C.c_uint64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    """Names declared in include/sfxb_cuda.h (checked against the .so by the CPU tests)."""
    import re

    hdr = os.path.join(os.path.dirname(PKG), "include", "sfxb_cuda.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(sfxb_[a-z0-9_]+)\s*\(", text)))


def to_words(x: int, words: int) -> np.ndarray:
    return np.frombuffer(int(x).to_bytes(4 * words, "little"), dtype=np.uint32).copy()


def from_words(w) -> int:
    return int.from_bytes(np.ascontiguousarray(w, dtype=np.uint32).tobytes(), "little")


class Context:
    """One Paillier key on one device (sfxb_ctx), or on a device group when
    `devices` lists several GPUs (sfxb_ctx_create_multi)."""

    def __init__(self, n: int, p: int | None = None, q: int | None = None, device: int = 0,
                 devices: list[int] | None = None):
        lib = load()
        self.lib = lib
        self.n = n
        self.nw = (n.bit_length() + 31) // 32
        h = C.c_void_p()
        nw_arr = to_words(n, self.nw)
        pa = qa = None
        pw = 0
        if p is not None:
            pw = max((p.bit_length() + 31) // 32, (q.bit_length() + 31) // 32)
            pa, qa = to_words(p, pw), to_words(q, pw)
        pp = pa.ctypes.data if pa is not None else None
        qp = qa.ctypes.data if qa is not None else None
        if devices is not None:
            dv = np.ascontiguousarray(devices, dtype=np.int32)
            rc = lib.sfxb_ctx_create_multi(C.byref(h), dv, len(dv), nw_arr, self.nw, pp, qp, pw)
        else:
            rc = lib.sfxb_ctx_create(C.byref(h), device, nw_arr, self.nw, pp, qp, pw)
        if rc != SFXB_OK:
            raise SfxbError(rc, lib.sfxb_create_error().decode())
        self.h = h
        self.ct_words = lib.sfxb_ctx_ct_words(h)
        self.key_id = lib.sfxb_ctx_key_id(h)
        self.has_private = bool(lib.sfxb_ctx_has_private(h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.sfxb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != SFXB_OK:
            msg = self.lib.sfxb_last_error(self.h).decode()
            if rc == SFXB_ERR_AUTH:
                raise AuthorizationError(rc, msg)
            raise SfxbError(rc, msg)

    def profile(self, enable: bool = True):
        self._check(self.lib.sfxb_ctx_profile(self.h, 1 if enable else 0))

    def kernel_time(self, family: int):
        """(launches, total ms) of a hot-kernel family since profile(True)."""
        n, ms = C.c_uint64(), C.c_double()
        self._check(self.lib.sfxb_ctx_kernel_time(self.h, family, C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def kernel_stats(self, family: int):
        """(launches, total ms, Montgomery multiplications) of a kernel family since profile(True)."""
        n, ms, mm = C.c_uint64(), C.c_double(), C.c_uint64()
        self._check(self.lib.sfxb_ctx_kernel_stats(self.h, family, C.byref(n), C.byref(ms), C.byref(mm)))
        return n.value, ms.value, mm.value

    @property
    def n_shards(self) -> int:
        return self.lib.sfxb_ctx_n_shards(self.h)

    @property
    def launches(self) -> int:
        return self.lib.sfxb_ctx_launches(self.h)

    @property
    def dec_derived(self) -> int:
        """Slots decrypt_tree derived by verified sibling reuse."""
        return self.lib.sfxb_ctx_dec_derived(self.h)

    def encrypt_plain(self, m_words, r_words):
        """Encrypt plaintexts m ∈ [0, n) given as words (packed vectors)."""
        m_words = np.ascontiguousarray(m_words, dtype=np.uint32)
        r_words = np.ascontiguousarray(r_words, dtype=np.uint32)
        count = m_words.shape[0]
        out = np.zeros((count, self.ct_words), np.uint32)
        self._check(self.lib.sfxb_encrypt_plain(self.h, m_words.reshape(-1), r_words.reshape(-1), count,
                                                out.reshape(-1), None))
        return out

    def encode_check(self, x: float, scale: int = 40) -> int:
        q = C.c_int64()
        self._check(self.lib.sfxb_encode_check(self.h, float(x), scale, C.byref(q)))
        return q.value

    def encode_batch(self, x, scale: int = 40):
        """encode_fixed of every value (sfxb_encode_batch): (q, first failing index or None)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        q = np.zeros(len(x), np.int64)
        bad = C.c_size_t(0)
        rc = self.lib.sfxb_encode_batch(self.h, x, len(x), scale, q, C.byref(bad))
        if rc != SFXB_OK and bad.value >= len(x):
            self._check(rc)
        return q, (bad.value if rc != SFXB_OK else None)

    def encrypt(self, q_fixed, r):
        """q_fixed: int64[count]; r: uint32[count, n_words] -> uint32[count, ct_words]."""
        q_fixed = np.ascontiguousarray(q_fixed, dtype=np.int64)
        r = np.ascontiguousarray(r, dtype=np.uint32)
        count = q_fixed.shape[0]
        out = np.zeros((count, self.ct_words), np.uint32)
        flags = np.zeros(count, np.uint8)
        self._check(self.lib.sfxb_encrypt(self.h, q_fixed, r.reshape(-1), count, out, flags.ctypes.data))
        return out

    def add(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.zeros_like(a)
        self._check(self.lib.sfxb_add(self.h, a.reshape(-1), b.reshape(-1), a.shape[0], out.reshape(-1)))
        return out

    def accumulate(self, gh_cts, bins, node_offsets, rows, n_bins):
        gh_cts = np.ascontiguousarray(gh_cts, dtype=np.uint32)
        bins = np.ascontiguousarray(bins, dtype=np.uint16)
        J, n_samples = bins.shape
        n_nodes = len(node_offsets) - 1
        out = np.zeros((n_nodes * J * n_bins * 2, self.ct_words), np.uint32)
        adds = C.c_uint64(0)
        self._check(self.lib.sfxb_accumulate(
            self.h, gh_cts.reshape(-1), n_samples, bins.reshape(-1), J,
            np.ascontiguousarray(node_offsets, dtype=np.uint32), n_nodes,
            np.ascontiguousarray(rows, dtype=np.uint32), n_bins, out.reshape(-1), C.byref(adds)))
        return out, adds.value

    def decrypt(self, cts, scale: int = 40, want_plain: bool = False):
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        count = cts.shape[0]
        vals = np.zeros(count, np.float64)
        plain = np.zeros((count, self.nw), np.uint32) if want_plain else None
        decs = C.c_uint64(0)
        self._check(self.lib.sfxb_decrypt(self.h, cts.reshape(-1), count, scale, vals,
                                          plain.ctypes.data if want_plain else None, C.byref(decs)))
        return (vals, decs.value, plain) if want_plain else (vals, decs.value)

    def decrypt_tree(self, tag: int, cts, n_nodes: int, parent=None, scale: int = 40):
        """sfxb_decrypt_tree: one tree level of histogram stream `tag`
        (n_nodes × slots_per_node ciphertexts), with verified sibling reuse
        against the previous level of the same tag."""
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        count = cts.shape[0]
        spn = count // n_nodes if n_nodes else 0
        if n_nodes * spn != count:
            raise ValueError("ciphertext count is not a multiple of n_nodes")
        vals = np.zeros(count, np.float64)
        par = None if parent is None else np.ascontiguousarray(parent, dtype=np.int32)
        decs = C.c_uint64(0)
        self._check(self.lib.sfxb_decrypt_tree(self.h, tag, cts.reshape(-1), n_nodes, spn,
                                               None if par is None else par.ctypes.data, scale, vals,
                                               C.byref(decs)))
        return vals, decs.value


class GhHandle:
    """Device-resident gradient ciphertexts (sfxb_gh, Montgomery form)."""

    def __init__(self, ctx: "Context", h):
        self.ctx, self.h = ctx, h

    def free(self):
        if self.h:
            self.ctx.lib.sfxb_gh_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _ptr(t) -> int:
    """Device pointer of a torch tensor (plumbing only)."""
    return int(t.data_ptr())


class DeviceOps:
    """Device-pointer entry points (`*_dev`) driven with torch tensors.

    torch provides device memory and the stream order; every call syncs torch's
    stream before enqueueing on the context stream and returns after the
    context stream drained (tests/bench time their own regions)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        import torch

        self.torch = torch

    def _pre(self):
        self.torch.cuda.synchronize()

    def _post(self):
        self.ctx._check(self.ctx.lib.sfxb_ctx_sync(self.ctx.h))

    def gh_from_dev(self, d_gh, n_samples: int) -> GhHandle:
        self._pre()
        h = C.c_void_p()
        self.ctx._check(self.ctx.lib.sfxb_gh_from_dev(self.ctx.h, _ptr(d_gh), n_samples, C.byref(h)))
        return GhHandle(self.ctx, h)

    def accumulate_host(self, gh: GhHandle, bins, node_offsets, rows, n_bins: int, out=None):
        """Host-buffer accumulate over a resident gh (sfxb_accumulate_gh)."""
        bins = np.ascontiguousarray(bins, dtype=np.uint16)
        J = bins.shape[0]
        n_nodes = len(node_offsets) - 1
        if out is None:
            out = np.zeros((n_nodes * J * n_bins * 2, self.ctx.ct_words), np.uint32)
        adds = C.c_uint64(0)
        self.ctx._check(self.ctx.lib.sfxb_accumulate_gh(
            self.ctx.h, gh.h, bins.reshape(-1), J, np.ascontiguousarray(node_offsets, dtype=np.uint32), n_nodes,
            np.ascontiguousarray(rows, dtype=np.uint32), n_bins, out.reshape(-1), C.byref(adds)))
        return out, adds.value

    def gh_upload(self, gh_cts) -> GhHandle:
        gh_cts = np.ascontiguousarray(gh_cts, dtype=np.uint32)
        h = C.c_void_p()
        self.ctx._check(self.ctx.lib.sfxb_gh_upload(self.ctx.h, gh_cts.reshape(-1), gh_cts.shape[0] // 2, C.byref(h)))
        return GhHandle(self.ctx, h)

    def accumulate(self, gh: GhHandle, d_bins, n_features: int, d_offsets, n_nodes: int, d_rows, n_rows: int,
                   n_bins: int, d_out, mont_out: bool = False, sync: bool = True) -> int:
        if sync:
            self._pre()
        adds = C.c_uint64(0)
        self.ctx._check(self.ctx.lib.sfxb_accumulate_dev(
            self.ctx.h, gh.h, _ptr(d_bins), n_features, _ptr(d_offsets), n_nodes, _ptr(d_rows), n_rows, n_bins,
            _ptr(d_out), 1 if mont_out else 0, C.byref(adds)))
        if sync:
            self._post()
        return adds.value

    def accumulate_tree(self, gh: GhHandle, d_bins, n_features: int, d_offsets, h_offsets, n_nodes: int, d_rows,
                        n_rows: int, n_bins: int, parent, d_out, mont_out: bool = False, sync: bool = True) -> int:
        """Tree-mode accumulate (sibling subtraction), device buffers + host metadata."""
        if sync:
            self._pre()
        adds = C.c_uint64(0)
        self.ctx._check(self.ctx.lib.sfxb_accumulate_tree_dev(
            self.ctx.h, gh.h, _ptr(d_bins), n_features, _ptr(d_offsets),
            np.ascontiguousarray(h_offsets, dtype=np.uint32), n_nodes, _ptr(d_rows), n_rows, n_bins,
            np.ascontiguousarray(parent, dtype=np.int32), _ptr(d_out), 1 if mont_out else 0, C.byref(adds)))
        if sync:
            self._post()
        return adds.value

    def accumulate_tree_host(self, gh: GhHandle, bins, node_offsets, rows, n_bins: int, parent, out=None):
        bins = np.ascontiguousarray(bins, dtype=np.uint16)
        J = bins.shape[0]
        n_nodes = len(node_offsets) - 1
        if out is None:
            out = np.zeros((n_nodes * J * n_bins * 2, self.ctx.ct_words), np.uint32)
        adds = C.c_uint64(0)
        self.ctx._check(self.ctx.lib.sfxb_accumulate_tree_gh(
            self.ctx.h, gh.h, bins.reshape(-1), J, np.ascontiguousarray(node_offsets, dtype=np.uint32), n_nodes,
            np.ascontiguousarray(rows, dtype=np.uint32), n_bins, np.ascontiguousarray(parent, dtype=np.int32),
            out.reshape(-1), C.byref(adds)))
        return out, adds.value

    def bins_upload(self, bins):
        """Device-resident bin columns (sfxb_bins_upload); free with bins_free."""
        bins = np.ascontiguousarray(bins, dtype=np.uint16)
        h = C.c_void_p()
        self.ctx._check(self.ctx.lib.sfxb_bins_upload(self.ctx.h, bins.reshape(-1), bins.shape[0], bins.shape[1],
                                                      C.byref(h)))
        return h

    def bins_free(self, h):
        self.ctx.lib.sfxb_bins_free(h)

    def accumulate_tree_bins(self, gh: GhHandle, bins_h, n_features: int, node_offsets, rows, n_bins: int, parent,
                             out=None):
        """Tree-mode accumulate over resident gh and bins, host frontier and output."""
        n_nodes = len(node_offsets) - 1
        if out is None:
            out = np.zeros((n_nodes * n_features * n_bins * 2, self.ctx.ct_words), np.uint32)
        adds = C.c_uint64(0)
        self.ctx._check(self.ctx.lib.sfxb_accumulate_tree_bins(
            self.ctx.h, gh.h, bins_h, np.ascontiguousarray(node_offsets, dtype=np.uint32), n_nodes,
            np.ascontiguousarray(rows, dtype=np.uint32), n_bins, np.ascontiguousarray(parent, dtype=np.int32),
            out.reshape(-1), C.byref(adds)))
        return out, adds.value

    def slice_width(self, n_features: int, n_bins: int, world: int) -> int:
        return self.ctx.lib.sfxb_slice_width(n_features, n_bins, world)

    def accumulate_part(self, gh: GhHandle, d_bins, n_features: int, d_offsets, h_offsets, n_nodes: int, d_rows,
                        n_rows: int, n_bins: int, parent, sizes, world: int, d_send, d_real, sync: bool = True):
        """Rank-sliced partials (sfxb_accumulate_part_dev): d_send = world x n_nodes x jl
        Montgomery-form slices, d_real = 2*n_nodes*J*K real-ciphertext counts."""
        if sync:
            self._pre()
        par = None if parent is None else np.ascontiguousarray(parent, dtype=np.int32)
        siz = None if sizes is None else np.ascontiguousarray(sizes, dtype=np.uint32)
        self.ctx._check(self.ctx.lib.sfxb_accumulate_part_dev(
            self.ctx.h, gh.h, _ptr(d_bins), n_features, _ptr(d_offsets),
            np.ascontiguousarray(h_offsets, dtype=np.uint32), n_nodes, _ptr(d_rows), n_rows, n_bins,
            None if par is None else par.ctypes.data, None if siz is None else siz.ctypes.data, world,
            _ptr(d_send), _ptr(d_real)))
        if sync:
            self._post()

    def combine_slices(self, gh: GhHandle, d_recv, world: int, rank: int, n_nodes: int, n_features: int,
                       n_bins: int, parent, sizes, d_out, sync: bool = True):
        """Product of the received slices + sibling subtraction on this rank's
        slice (sfxb_combine_slices_dev) -> plain n_nodes x jl slice in d_out."""
        if sync:
            self._pre()
        par = None if parent is None else np.ascontiguousarray(parent, dtype=np.int32)
        siz = None if sizes is None else np.ascontiguousarray(sizes, dtype=np.uint32)
        self.ctx._check(self.ctx.lib.sfxb_combine_slices_dev(
            self.ctx.h, gh.h, _ptr(d_recv), world, rank, n_nodes, n_features, n_bins,
            None if par is None else par.ctypes.data, None if siz is None else siz.ctypes.data, _ptr(d_out)))
        if sync:
            self._post()

    def count_additions(self, d_real, n: int) -> int:
        self._pre()
        adds = C.c_uint64(0)
        self.ctx._check(self.ctx.lib.sfxb_count_additions_dev(self.ctx.h, _ptr(d_real), n, C.byref(adds)))
        return adds.value

    def tree_reset(self):
        self.ctx._check(self.ctx.lib.sfxb_tree_reset(self.ctx.h))

    def reduce_partials(self, d_parts, parts: int, n_slots: int, d_out, sync: bool = True):
        if sync:
            self._pre()
        self.ctx._check(self.ctx.lib.sfxb_reduce_partials_dev(self.ctx.h, _ptr(d_parts), parts, n_slots, _ptr(d_out)))
        if sync:
            self._post()

    def encrypt(self, d_q, d_r, count: int, d_out, sync: bool = True):
        if sync:
            self._pre()
        self.ctx._check(self.ctx.lib.sfxb_encrypt_dev(self.ctx.h, _ptr(d_q), _ptr(d_r), count, _ptr(d_out), None))
        if sync:
            self._post()

    def decrypt(self, d_cts, count: int, d_values, scale: int = 40, sync: bool = True) -> int:
        if sync:
            self._pre()
        decs = C.c_uint64(0)
        self.ctx._check(self.ctx.lib.sfxb_decrypt_dev(self.ctx.h, _ptr(d_cts), count, scale, _ptr(d_values), None,
                                                      C.byref(decs)))
        if sync:
            self._post()
        return decs.value


def imad_peak(device: int = 0):
    lib = load()
    p, clk = C.c_double(), C.c_double()
    rc = lib.sfxb_imad_peak(device, C.byref(p), C.byref(clk))
    if rc != SFXB_OK:
        raise SfxbError(rc, "imad peak microbenchmark failed")
    return p.value, clk.value
