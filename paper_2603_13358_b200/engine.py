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
