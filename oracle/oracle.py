"""oracle.py — TEST INFRASTRUCTURE ONLY (checker, never the product path).

ctypes view of oracle/_ref/libmodel_oracle.so (the CPU model restatement,
model_oracle.c) and a runner for oracle/_ref/ref_tool (the UNMODIFIED reference
library behind a JSON driver). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.

Parity of the model restatement is UNPINNED against the reference: the
reference has no model. The ref_tool side IS the reference.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ORACLE_DIR, "_ref")
MODEL_LIB = os.path.join(REF_DIR, "libmodel_oracle.so")
REF_TOOL = os.path.join(REF_DIR, "ref_tool")
ACCEPTANCE = os.path.join(REF_DIR, "acceptance")


class MoCfg(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int), ("d_model", ctypes.c_int), ("n_q_heads", ctypes.c_int),
        ("n_kv_heads", ctypes.c_int), ("head_dim", ctypes.c_int), ("d_ff", ctypes.c_int),
        ("vocab", ctypes.c_int), ("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_float),
        ("qkv_bias", ctypes.c_int),
    ]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(MODEL_LIB):
            build()
        L = ctypes.CDLL(MODEL_LIB)
        vp, i32, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64
        L.mo_weight_bf16.restype = ctypes.c_uint16
        L.mo_weight_bf16.argtypes = [u64, i32, i32, u64]
        L.mo_token_id.restype = ctypes.c_uint32
        L.mo_token_id.argtypes = [u64, u64, i32, ctypes.c_int64, i32]
        L.mo_model_create.restype = vp
        L.mo_model_create.argtypes = [ctypes.POINTER(MoCfg), u64]
        L.mo_model_free.argtypes = [vp]
        L.mo_set_active_layers.argtypes = [vp, i32]
        L.mo_step.restype = i32
        L.mo_step.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, i32, vp, vp, vp]
        L.mo_attention_paged.argtypes = [ctypes.POINTER(MoCfg), vp, vp, i32, i32, i32, vp, vp, vp, i32, vp]
        L.mo_rope_table.argtypes = [ctypes.c_float, i32, i32, vp, vp]
        L.mo_fill_tensor.argtypes = [u64, i32, i32, u64, vp]
        _lib = L
    return _lib


def cfg_from(dev_cfg) -> MoCfg:
    d = dev_cfg.as_dict() if hasattr(dev_cfg, "as_dict") else dict(dev_cfg)
    return MoCfg(*[d[k] for k, _ in MoCfg._fields_])


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def weight(seed: int, tensor: int, layer: int, idx: int) -> int:
    return lib().mo_weight_bf16(seed, tensor, layer, idx)


def tensor_bf16(seed: int, tensor: int, layer: int, n: int) -> np.ndarray:
    """The first n weights of one logical tensor (bf16 bits), the same values
    the device fill kernels and mo_model_create produce."""
    out = np.empty(n, dtype=np.uint16)
    lib().mo_fill_tensor(seed, tensor, layer, n, _p(out))
    return out


class KvPool:
    """CPU paged pool, same block-major layout as the device pool."""

    def __init__(self, cfg: MoCfg, num_blocks: int, block_tokens: int = 16):
        self.cfg, self.bt, self.nb = cfg, block_tokens, num_blocks
        self.data = np.zeros((num_blocks, cfg.n_layers, 2, cfg.n_kv_heads, block_tokens, cfg.head_dim),
                             dtype=np.uint16)


class Model:
    def __init__(self, cfg: MoCfg, seed: int):
        self.cfg = cfg
        self.h = lib().mo_model_create(ctypes.byref(cfg), seed)

    def set_active_layers(self, n: int):
        lib().mo_set_active_layers(self.h, n)

    def __del__(self):
        try:
            lib().mo_model_free(self.h)
        except Exception:
            pass

    def step(self, pool: KvPool, q_len, ctx, tokens, block_tables, want_logits=True):
        q_len = np.asarray(q_len, dtype=np.int32)
        n = len(q_len)
        qs = np.zeros(n + 1, dtype=np.int32)
        qs[1:] = np.cumsum(q_len)
        ctx = np.ascontiguousarray(ctx, dtype=np.int32)
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        bt = np.ascontiguousarray(block_tables, dtype=np.int32).reshape(n, -1)
        logits = np.zeros((n, self.cfg.vocab), dtype=np.float32) if want_logits else None
        out = np.zeros(n, dtype=np.int32)
        margin = np.zeros(n, dtype=np.float32)
        rc = lib().mo_step(self.h, _p(pool.data), pool.bt, n, _p(qs), _p(ctx), _p(tokens), _p(bt), bt.shape[1],
                           _p(logits) if want_logits else None, _p(out), _p(margin))
        assert rc == 0
        return out, logits, margin


def attention(cfg: MoCfg, q_bf16: np.ndarray, pool: np.ndarray, block_tokens: int, layer: int,
              q_start, ctx, block_tables) -> np.ndarray:
    q = np.ascontiguousarray(q_bf16, dtype=np.uint16)
    out = np.zeros(q.shape, dtype=np.float32)
    qs = np.ascontiguousarray(q_start, dtype=np.int32)
    cx = np.ascontiguousarray(ctx, dtype=np.int32)
    bt = np.ascontiguousarray(block_tables, dtype=np.int32)
    pool = np.ascontiguousarray(pool, dtype=np.uint16)
    lib().mo_attention_paged(ctypes.byref(cfg), _p(q), _p(pool), block_tokens, layer, len(cx), _p(qs), _p(cx),
                             _p(bt), bt.shape[-1], _p(out))
    return out


def ref_tool(job: dict) -> dict:
    """Run one job through the UNMODIFIED reference library (oracle/_ref/ref_tool)."""
    if not os.path.exists(REF_TOOL):
        build()
    p = subprocess.run([REF_TOOL], input=json.dumps(job), capture_output=True, text=True)
    out = json.loads(p.stdout)
    if "error" in out:
        raise RuntimeError(out["error"])
    return out
