"""ctypes wrapper for the plain-C set-semantics oracle (oracle/setsem.c).

ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "setsem.c")
_LIB = os.path.join(_HERE, "libsetsem.so")
_lib = None

ERRORS = {0: "OK", 1: "INVALID_ARG", 2: "OUT_OF_RANGE", 3: "EXAMPLE_CONFLICT",
          4: "BAD_EXPR", 7: "OOM"}


class OracleError(RuntimeError):
    def __init__(self, code, root=None):
        super().__init__(f"oracle error {ERRORS.get(code, code)}" + (f" at root {root}" if root is not None else ""))
        self.code = code
        self.root = root


def build(force: bool = False) -> str:
    """Compile oracle/setsem.c with gcc -O2 (no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               _SRC, "-o", _LIB + ".tmp", "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.c_void_p
        lib.oracle_kb_new.argtypes = [C.c_uint32, C.c_uint32, P, C.c_uint32, P, P, P,
                                      C.c_uint32, P, P, P, C.c_uint32, P, C.c_uint32, P,
                                      C.c_uint32, P, P, P, P, C.POINTER(C.c_void_p)]
        lib.oracle_kb_new.restype = C.c_int
        lib.oracle_kb_free.argtypes = [P]
        lib.oracle_eval.argtypes = [P, P, C.c_uint32, P, C.c_uint64, P, C.c_uint32, C.c_uint32,
                                    C.c_uint32, P, P, P, P, C.c_int, C.POINTER(C.c_uint32)]
        lib.oracle_eval.restype = C.c_int
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


class OracleKB:
    """The oracle's own load of a KB dict (synth format): deduped pair sets."""

    def __init__(self, kb: dict):
        lib = _load()
        self._keep = []

        def arr(name, dt):
            a = np.ascontiguousarray(kb[name], dtype=dt)
            self._keep.append(a)
            return a

        cb = arr("concept_bits", np.uint32)
        ro, es, eo = arr("role_edge_off", np.uint64), arr("edge_subj", np.uint32), arr("edge_obj", np.uint32)
        do, ds, dv = arr("data_off", np.uint64), arr("data_subj", np.uint32), arr("data_val", np.float32)
        pos, neg = arr("pos_ids", np.uint32), arr("neg_ids", np.uint32)
        from synth.format import string_fields
        so, ss, sv, sb = string_fields(kb)
        self._keep += [so, ss, sv, sb]
        self.N = int(kb["N"])
        self.W = (self.N + 31) // 32
        h = C.c_void_p()
        rc = lib.oracle_kb_new(self.N, cb.shape[0] if cb.ndim == 2 else 0, _p(cb),
                               len(ro) - 1, _p(ro), _p(es), _p(eo),
                               len(do) - 1, _p(do), _p(ds), _p(dv),
                               len(pos), _p(pos), len(neg), _p(neg),
                               len(so) - 1, _p(so), _p(ss), _p(sv), _p(sb), C.byref(h))
        if rc:
            raise OracleError(rc)
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _load().oracle_kb_free(self._h)
            self._h = None

    def evaluate(self, nodes, child_idx, roots, flags: int = 0, want_bits: bool = True,
                 threads: int = 1, patterns=None):
        """-> (bits [n_roots][W] u32 or None, counts [n_roots][4] u64 = tp, fp, fn, tn).
        `patterns`: string-restriction patterns (list of bytes; defaults to the table `nodes` carries)."""
        lib = _load()
        from synth.format import node_patterns, pack_strings
        if patterns is None:
            patterns = node_patterns(nodes)
        po, pb = pack_strings(patterns)
        nodes = np.ascontiguousarray(nodes)
        kids = np.ascontiguousarray(child_idx, dtype=np.uint32)
        roots = np.ascontiguousarray(roots, dtype=np.uint32)
        n = len(roots)
        bits = np.zeros((n, self.W), dtype=np.uint32) if want_bits else None
        counts = np.zeros((n, 4), dtype=np.uint64)
        bad = C.c_uint32(0)
        rc = lib.oracle_eval(self._h, _p(nodes), len(nodes), _p(kids), len(kids), _p(roots), n,
                             flags, len(po) - 1, _p(po), _p(pb), _p(bits) if want_bits else None, _p(counts),
                             threads, C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value)
        return bits, counts


def evaluate(kb: dict, nodes, child_idx, roots, flags: int = 0, want_bits: bool = True, threads: int = 1,
             patterns=None):
    return OracleKB(kb).evaluate(nodes, child_idx, roots, flags, want_bits, threads, patterns)
