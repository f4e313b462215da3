"""ctypes view of libppd_engine.so (include/ppd_engine.h): the host C++ PPD
engine. run() takes the same job dict as the reference driver
(oracle/ref_tool.cpp op=simulate) plus "clock": "virtual" | "device"."""
from __future__ import annotations

import ctypes
import json
import os

from . import PKG_DIR, lib as _device_lib

ENGINE_PATH = os.path.join(PKG_DIR, "libppd_engine.so")
_eng = None


class EngineError(RuntimeError):
    pass


def _lib():
    global _eng
    if _eng is None:
        if not os.path.exists(ENGINE_PATH):
            raise RuntimeError(f"{ENGINE_PATH} missing: run `make -C {PKG_DIR}` (no CPU fallback)")
        _device_lib()  # libppd_b200.so first (the engine links it)
        L = ctypes.CDLL(ENGINE_PATH)
        L.ppd_engine_run_json.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.ppd_engine_run_json.restype = ctypes.c_int
        L.ppd_engine_free.argtypes = [ctypes.c_void_p]
        L.ppd_engine_last_error.restype = ctypes.c_char_p
        _eng = L
    return _eng


def run(job: dict) -> dict:
    L = _lib()
    out = ctypes.c_void_p()
    rc = L.ppd_engine_run_json(json.dumps(job).encode(), ctypes.byref(out))
    if rc != 0:
        msg = L.ppd_engine_last_error().decode()
        if rc == -1:
            raise ValueError(msg)
        raise EngineError(msg)
    try:
        return json.loads(ctypes.string_at(out.value).decode())
    finally:
        L.ppd_engine_free(out)


def records(result: dict) -> list:
    return [json.loads(x) for x in result["records_jsonl"].splitlines()[1:]]


class Gateway:
    """ctypes view of the routing gateway (ppd_gateway_* in include/ppd_engine.h;
    reference proj/include/ppd/gateway.hpp). handle() is one wire message in
    process; serve() starts the loopback TCP server (4-byte big-endian length +
    JSON frames)."""

    def __init__(self, policy: dict | None = None):
        L = _lib()
        L.ppd_gateway_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.ppd_gateway_handle.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_double,
                                         ctypes.POINTER(ctypes.c_void_p)]
        L.ppd_gateway_serve.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ppd_gateway_stop.argtypes = [ctypes.c_void_p]
        L.ppd_gateway_destroy.argtypes = [ctypes.c_void_p]
        self._L = L
        self._h = ctypes.c_void_p()
        self._check(L.ppd_gateway_create(json.dumps(policy or {}).encode(), ctypes.byref(self._h)))

    def _check(self, rc):
        if rc != 0:
            msg = self._L.ppd_engine_last_error().decode()
            raise ValueError(msg) if rc == -1 else EngineError(msg)

    def handle(self, payload: str, now: float) -> str:
        out = ctypes.c_void_p()
        self._check(self._L.ppd_gateway_handle(self._h, payload.encode(), now, ctypes.byref(out)))
        try:
            return ctypes.string_at(out.value).decode()
        finally:
            self._L.ppd_engine_free(out)

    def serve(self, port: int = 0) -> int:
        bound = ctypes.c_int(0)
        self._check(self._L.ppd_gateway_serve(self._h, port, ctypes.byref(bound)))
        return bound.value

    def stop(self):
        self._check(self._L.ppd_gateway_stop(self._h))

    def close(self):
        if self._h:
            self._L.ppd_gateway_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
