"""ctypes binding of libpdcs_io.so (csrc/pdcs_io.cpp): the multi-threaded
reader of problem-file JSON documents.  `load_document(path)` returns the
document as a dict whose large arrays are numpy arrays, or None when the file
is outside the reader's plain grammar (escaped strings, NaN tokens, ...); the
caller then parses with the json module so the reference's exact errors are
kept (conic_pdhg fileio.py:183-189).  Host I/O only; the solve path never
depends on it."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpdcs_io.so")
SRC = os.path.join(HERE, "csrc", "pdcs_io.cpp")

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= os.path.getmtime(SRC):
        return LIB_PATH
    cmd = ["g++", "-O3", "-std=c++17", "-shared", "-fPIC", "-pthread", "-o", LIB_PATH + ".tmp", SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({' '.join(cmd)}):\n{res.stderr}")
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            lib = C.CDLL(LIB_PATH)
            lib.pdcs_io_parse_file.restype = C.c_int
            lib.pdcs_io_parse_file.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]
            lib.pdcs_io_nkeys.restype = C.c_int32
            lib.pdcs_io_nkeys.argtypes = [C.c_void_p]
            lib.pdcs_io_key.restype = C.c_char_p
            lib.pdcs_io_key.argtypes = [C.c_void_p, C.c_int32]
            lib.pdcs_io_scalar.restype = C.c_int32
            lib.pdcs_io_scalar.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_double)]
            lib.pdcs_io_len.restype = C.c_int64
            lib.pdcs_io_len.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int32)]
            lib.pdcs_io_copy.restype = C.c_int32
            lib.pdcs_io_copy.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
            lib.pdcs_io_free.restype = None
            lib.pdcs_io_free.argtypes = [C.c_void_p]
            lib.pdcs_io_error.restype = C.c_char_p
            _lib = lib
    return _lib


def _array(lib, h, key: str):
    kind = C.c_int32(0)
    n = lib.pdcs_io_len(h, key.encode(), C.byref(kind))
    if n < 0:
        return None
    out = np.empty(n, dtype=np.int64 if kind.value == 1 else np.float64)
    if n:
        lib.pdcs_io_copy(h, key.encode(), out.ctypes.data)
    return out


def load_document(path: str, threads: int = 0):
    lib = _load()
    h = C.c_void_p()
    if lib.pdcs_io_parse_file(os.fsencode(path), int(threads), C.byref(h)) != 0:
        return None
    try:
        doc = {}
        for i in range(lib.pdcs_io_nkeys(h)):
            key = lib.pdcs_io_key(h, i).decode()
            if key == "G":
                g = {}
                for sub in ("rows", "cols", "vals"):
                    a = _array(lib, h, "G." + sub)
                    if a is not None:
                        g[sub] = a
                doc["G"] = g
                continue
            v = C.c_double()
            if lib.pdcs_io_scalar(h, key.encode(), C.byref(v)):
                x = float(v.value)
                doc[key] = int(x) if x.is_integer() else x
                continue
            a = _array(lib, h, key)
            doc[key] = a if a is not None else None  # unknown key: only its name matters
        return doc
    finally:
        lib.pdcs_io_free(h)
