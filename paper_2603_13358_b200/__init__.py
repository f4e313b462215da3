"""paper_2603_13358_b200 — B200-native PPD serving data path.

Python here is only a ctypes view of the C-ABI (include/ppd_b200.h) used by the
tests and bench.py. The product is native: libppd_b200.so (sm_100a kernels +
C-ABI) and libppd_engine.so (the host C++ engine with the reference's
ppd:: API surface). There is no CPU fallback: if the shared library is missing
every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libppd_b200.so")
HEADER_PATH = os.path.join(REPO_DIR, "include", "ppd_b200.h")

PPD_OK = 0
PPD_ERR_INVALID = -1
PPD_ERR_CUDA = -2
PPD_ERR_OOM = -3
PPD_ERR_STATE = -4
PREFILL_FULL = 0
PREFILL_APPEND = 1


class PPDError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"ppd error {code}: {msg}")
        self.code = code


class InvalidArgument(PPDError, ValueError):
    """Mirrors the reference's std::invalid_argument (costmodel.cpp:319, :325-327, :335)."""


class ModelCfg(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int32), ("d_model", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("d_ff", ctypes.c_int32),
        ("vocab", ctypes.c_int32), ("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_float),
        ("qkv_bias", ctypes.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def tiny_cfg() -> ModelCfg:
    """Builder-defined tiny config (no analogue in the reference)."""
    return ModelCfg(2, 512, 4, 1, 128, 1024, 2048, 1e-5, 5e5, 0)


def llama8b_cfg(n_layers: int = 32) -> ModelCfg:
    return ModelCfg(n_layers, 4096, 32, 8, 128, 14336, 128256, 1e-5, 5e5, 0)


def qwen32b_cfg(n_layers: int = 64) -> ModelCfg:
    return ModelCfg(n_layers, 5120, 40, 8, 128, 27648, 152064, 1e-6, 1e6, 1)


class GemmParts(ctypes.Structure):
    """ppd_gemm_parts: how the fp32 GEMM output is spread over K-partial slices."""
    _fields_ = [("n", ctypes.c_int32), ("kbt", ctypes.c_int32), ("slots", ctypes.c_int32),
                ("rows", ctypes.c_int32), ("bn", ctypes.c_int32), ("n_tiles_t", ctypes.c_int32),
                ("total", ctypes.c_int64), ("stride", ctypes.c_uint64), ("dp", ctypes.c_int32)]

    def owner(self, x):
        return ((x + 1) * self.slots + self.total - 1) // self.total - 1

    def valid(self, col, tok):
        """Valid slice count for output column `col` of token row `tok` (numpy arrays ok)."""
        if self.kbt == 0:
            return col * 0 + tok * 0 + self.n
        t = (col // self.rows) * self.n_tiles_t + tok // self.bn - self.dp
        tail = t * (t >= 0)  # whole-K tiles [0, dp) have one valid slice
        v = self.owner(tail * self.kbt + self.kbt - 1) - self.owner(tail * self.kbt) + 1
        return v * (t >= 0) + 1 * (t < 0)


class DevStats(ctypes.Structure):
    _fields_ = [
        ("steps", ctypes.c_int64), ("own_launches", ctypes.c_int64), ("lib_launches", ctypes.c_int64),
        ("attn_launches", ctypes.c_int64), ("attn_ms", ctypes.c_double), ("gemm_ms", ctypes.c_double),
        ("attn_bytes", ctypes.c_double), ("step_ms", ctypes.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Batch(ctypes.Structure):
    _fields_ = [
        ("n_seqs", ctypes.c_int32), ("q_len", ctypes.c_void_p), ("ctx", ctypes.c_void_p),
        ("tokens", ctypes.c_void_p), ("block_tables", ctypes.c_void_p),
        ("max_blocks", ctypes.c_int32), ("want_token", ctypes.c_void_p),
    ]


_lib = None


def load_lib(path: str = LIB_PATH, strict: bool = True):
    """Load a build of libppd_b200.so and declare the C-ABI signatures.
    strict=False skips entry points an older build does not export (A/B tools)."""
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `make -C {PKG_DIR}` (no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i32, u64, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int64
    P = ctypes.POINTER
    L.ppd_last_error.restype = ctypes.c_char_p
    sig = {
        "ppd_version": [],
        "ppd_device_count": [P(i32)],
        "ppd_dev_open": [i32, P(ModelCfg), i32, i32, P(vp)],
        "ppd_dev_close": [vp],
        "ppd_load_random_weights": [vp, u64],
        "ppd_kv_pool_init": [vp, i32, i32],
        "ppd_kv_block_bytes": [P(ModelCfg), i32, P(u64)],
        "ppd_kv_pool_ptr": [vp, P(vp), P(u64)],
        "ppd_kv_pool_write": [vp, u64, vp, u64],
        "ppd_kv_pool_read": [vp, u64, vp, u64],
        "ppd_step": [vp, P(Batch), vp, P(ctypes.c_float)],
        "ppd_step_submit": [vp, P(Batch)],
        "ppd_step_wait": [vp, vp, P(ctypes.c_float)],
        "ppd_last_logits": [vp, vp, i64],
        "ppd_prefill": [vp, i32, vp, i32, i32, vp, i32, vp, P(ctypes.c_float)],
        "ppd_kv_copy": [vp, vp, vp, vp, i32, i32, i32, P(ctypes.c_float)],
        "ppd_kv_copy_submit": [vp, vp, vp, vp, i32, i32, i32, P(u64)],
        "ppd_kv_copy_wait": [vp, u64, P(ctypes.c_float)],
        "ppd_p2p_bandwidth": [i32, i32, u64, i32, i32, P(ctypes.c_double)],
        "ppd_weights_info": [vp, P(u64), P(i32)],
        "ppd_op_attention": [P(ModelCfg), vp, vp, i32, i32, i32, i32, vp, vp, vp, i32, vp, vp],
        "ppd_op_gemm": [vp, vp, vp, i32, i32, i32, i32, vp],
        "ppd_op_gemm_tc": [vp, vp, vp, i32, i32, i32, i32, i32, vp],
        "ppd_op_fill_random": [vp, u64, u64, i32, i32, vp],
        "ppd_set_tuning": [ctypes.c_char_p, i32],
        "ppd_op_gemm_silu": [vp, vp, vp, i32, i32, i32, vp],
        "ppd_op_gemm_parts": [vp, vp, vp, i32, i32, i32, i32, P(GemmParts), vp],
        "ppd_dev_set_profiling": [vp, i32],
        "ppd_dev_get_stats": [vp, P(DevStats)],
        "ppd_dev_reset_stats": [vp],
    }
    for name, args in sig.items():
        if not strict and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    return L


def lib():
    global _lib
    if _lib is None:
        _lib = load_lib()
    return _lib


def check(rc: int):
    if rc != PPD_OK:
        msg = lib().ppd_last_error().decode()
        if rc == PPD_ERR_INVALID:
            raise InvalidArgument(rc, msg)
        raise PPDError(rc, msg)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class StepResult:
    tokens: np.ndarray
    ms: float


class Device:
    """One GPU worker (weights + paged KV pool) behind the C-ABI."""

    def __init__(self, gpu: int, cfg: ModelCfg, max_step_tokens: int = 4096, max_step_seqs: int = 256):
        self.cfg = cfg
        self.h = ctypes.c_void_p()
        check(lib().ppd_dev_open(gpu, ctypes.byref(cfg), max_step_tokens, max_step_seqs, ctypes.byref(self.h)))
        self.block_tokens = 16
        self.num_blocks = 0

    def close(self):
        if self.h:
            check(lib().ppd_dev_close(self.h))
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_random_weights(self, seed: int):
        check(lib().ppd_load_random_weights(self.h, seed))

    def kv_pool_init(self, num_blocks: int, block_tokens: int = 16):
        check(lib().ppd_kv_pool_init(self.h, block_tokens, num_blocks))
        self.block_tokens, self.num_blocks = block_tokens, num_blocks

    def kv_pool_ptr(self):
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        check(lib().ppd_kv_pool_ptr(self.h, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def weights_info(self):
        n, k = ctypes.c_uint64(), ctypes.c_int32()
        check(lib().ppd_weights_info(self.h, ctypes.byref(n), ctypes.byref(k)))
        return n.value, k.value

    def kv_pool_write(self, host: np.ndarray, offset: int = 0):
        host = np.ascontiguousarray(host)
        check(lib().ppd_kv_pool_write(self.h, offset, _ptr(host), host.nbytes))

    def kv_pool_read(self, n_bytes: int = None, offset: int = 0) -> np.ndarray:
        if n_bytes is None:
            n_bytes = self.kv_pool_ptr()[1] - offset
        out = np.empty(n_bytes // 2, dtype=np.uint16)
        check(lib().ppd_kv_pool_read(self.h, offset, _ptr(out), out.nbytes))
        return out

    def _batch(self, q_len, ctx, tokens, block_tables, want_token=None):
        q_len, ctx, tokens = _i32(q_len), _i32(ctx), _i32(tokens)
        bt = _i32(block_tables)
        if bt.ndim == 1:
            bt = bt.reshape(1, -1)
        keep = [q_len, ctx, tokens, bt]
        wt = None
        if want_token is not None:
            wt = _i32(want_token)
            keep.append(wt)
        b = Batch(len(q_len), _ptr(q_len).value, _ptr(ctx).value, _ptr(tokens).value, _ptr(bt).value,
                  bt.shape[1], _ptr(wt).value if wt is not None else None)
        return b, keep

    def step(self, q_len, ctx, tokens, block_tables, want_token=None) -> StepResult:
        b, keep = self._batch(q_len, ctx, tokens, block_tables, want_token)
        n_out = len(q_len) if want_token is None else int(np.count_nonzero(want_token))
        out = np.zeros(max(n_out, 1), dtype=np.int32)
        ms = ctypes.c_float()
        check(lib().ppd_step(self.h, ctypes.byref(b), _ptr(out), ctypes.byref(ms)))
        del keep
        return StepResult(out[:n_out], ms.value)

    def step_submit(self, q_len, ctx, tokens, block_tables, want_token=None):
        b, keep = self._batch(q_len, ctx, tokens, block_tables, want_token)
        self._keep = keep
        check(lib().ppd_step_submit(self.h, ctypes.byref(b)))

    def step_wait(self, n_out: int) -> StepResult:
        out = np.zeros(max(n_out, 1), dtype=np.int32)
        ms = ctypes.c_float()
        check(lib().ppd_step_wait(self.h, _ptr(out), ctypes.byref(ms)))
        self._keep = None
        return StepResult(out[:n_out], ms.value)

    def set_profiling(self, on: bool):
        check(lib().ppd_dev_set_profiling(self.h, 1 if on else 0))

    def stats(self) -> dict:
        st = DevStats()
        check(lib().ppd_dev_get_stats(self.h, ctypes.byref(st)))
        return st.as_dict()

    def reset_stats(self):
        check(lib().ppd_dev_reset_stats(self.h))

    def last_logits(self, n_rows: int) -> np.ndarray:
        out = np.zeros((n_rows, self.cfg.vocab), dtype=np.float32)
        check(lib().ppd_last_logits(self.h, _ptr(out), out.size))
        return out

    def prefill(self, kind: int, tokens, n_ctx: int, block_table) -> StepResult:
        tokens, bt = _i32(tokens), _i32(block_table)
        out = np.zeros(1, dtype=np.int32)
        ms = ctypes.c_float()
        check(lib().ppd_prefill(self.h, kind, _ptr(tokens), len(tokens), n_ctx, _ptr(bt), len(bt),
                                _ptr(out), ctypes.byref(ms)))
        return StepResult(out, ms.value)


def kv_copy(src: Device, dst: Device, src_blocks, dst_blocks, start: int, n_tokens: int) -> float:
    sb, db = _i32(src_blocks), _i32(dst_blocks)
    assert len(sb) == len(db)
    ms = ctypes.c_float()
    check(lib().ppd_kv_copy(src.h, dst.h, _ptr(sb), _ptr(db), len(sb), start, n_tokens, ctypes.byref(ms)))
    return ms.value


def kv_copy_submit(src: Device, dst: Device, src_blocks, dst_blocks, start: int, n_tokens: int) -> int:
    sb, db = _i32(src_blocks), _i32(dst_blocks)
    assert len(sb) == len(db)
    t = ctypes.c_uint64()
    check(lib().ppd_kv_copy_submit(src.h, dst.h, _ptr(sb), _ptr(db), len(sb), start, n_tokens, ctypes.byref(t)))
    return t.value


def kv_copy_wait(dst: Device, ticket: int) -> float:
    ms = ctypes.c_float()
    check(lib().ppd_kv_copy_wait(dst.h, ticket, ctypes.byref(ms)))
    return ms.value


def p2p_bandwidth(src_gpu: int, dst_gpu: int, n_bytes: int = 1 << 30, iters: int = 5, mode: int = 0) -> float:
    gbs = ctypes.c_double()
    check(lib().ppd_p2p_bandwidth(src_gpu, dst_gpu, n_bytes, iters, mode, ctypes.byref(gbs)))
    return gbs.value


def kv_block_bytes(cfg: ModelCfg, block_tokens: int = 16) -> int:
    n = ctypes.c_uint64()
    check(lib().ppd_kv_block_bytes(ctypes.byref(cfg), block_tokens, ctypes.byref(n)))
    return n.value


def header_symbols(path: str = HEADER_PATH):
    """Names of every function the C-ABI header declares."""
    import re
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ppd_\w+)\s*\(", text, re.M)))
