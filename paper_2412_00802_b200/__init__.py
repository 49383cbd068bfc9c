"""B200-native HT-HEDL hot path (arxiv 2412.00802): Python binding of libhedl.so.

Argument marshalling only -- every step of the evaluation runs in the CUDA
library (paper_2412_00802_b200/csrc, C ABI in include/hedl.h).  PyTorch is
used for device memory (output buffers) and streams.  There is no CPU
fallback: if libhedl.so is missing or fails to load, every entry point raises.

Names follow the ABI: hedl_kb_load, hedl_compile, hedl_eval_one, hedl_eval_batch.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhedl.so")

HEDL_COMPILE_NO_CSE = 1
HEDL_COMPILE_NO_REWRITE = 2
HEDL_COMPILE_COMPAT_PAPER_MAX = 4
HEDL_COMPILE_HOST_INPUT = 8
HEDL_EVAL_COUNTS_DEVICE = 1
HEDL_EVAL_PER_NODE = 2
HEDL_EVAL_FORCE_SLICE = 4
HEDL_EVAL_NO_FUSE = 8
HEDL_EVAL_NO_RESTRICT_U = 16
HEDL_EVAL_NO_USWEEP = 32

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "OUT_OF_RANGE", 3: "EXAMPLE_CONFLICT", 4: "BAD_EXPR",
          5: "PARSE", 6: "CUDA", 7: "OOM", 8: "UNSUPPORTED"}

# every symbol include/hedl.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ["hedl_kb_load", "hedl_kb_free", "hedl_kb_get_info", "hedl_compile", "hedl_compile_ex",
               "hedl_compile_device", "hedl_compile_text", "hedl_score_topk",
               "hedl_program_free", "hedl_set_allocator", "hedl_alloc_counters",
               "hedl_program_workspace_bytes", "hedl_program_set_workspace", "hedl_kb_set_concept_rows",
               "hedl_program_get_info", "hedl_program_root_bytes", "hedl_eval_one", "hedl_eval_batch",
               "hedl_program_set_workspace_limit", "hedl_last_error", "hedl_version", "hedl_prof_enable",
               "hedl_prof_reset", "hedl_prof_read", "hedl_launch_count", "hedl_io_counters"]


# the hedl_node record of include/hedl.h (28 bytes)
HEDL_NODE_DTYPE = np.dtype({"names": ["op", "flags", "pad", "arg", "n", "lo", "hi", "child_begin", "child_count"],
                            "formats": ["u1", "u1", "<u2", "<u4", "<u4", "<f4", "<f4", "<u4", "<u4"],
                            "offsets": [0, 1, 2, 4, 8, 12, 16, 20, 24], "itemsize": 28})


class HedlError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hedl {STATUS.get(code, code)}: {msg}")
        self.code = code


class _KbDesc(C.Structure):
    _fields_ = [("n_individuals", C.c_uint32), ("n_concepts", C.c_uint32), ("concept_bits", C.c_void_p),
                ("n_roles", C.c_uint32), ("role_edge_off", C.c_void_p), ("edge_subj", C.c_void_p),
                ("edge_obj", C.c_void_p), ("n_data", C.c_uint32), ("data_off", C.c_void_p),
                ("data_subj", C.c_void_p), ("data_val", C.c_void_p), ("n_pos", C.c_uint32),
                ("pos_ids", C.c_void_p), ("n_neg", C.c_uint32), ("neg_ids", C.c_void_p),
                ("n_strings", C.c_uint32), ("str_off", C.c_void_p), ("str_subj", C.c_void_p),
                ("str_val_off", C.c_void_p), ("str_bytes", C.c_void_p)]


class _KbInfo(C.Structure):
    _fields_ = [("n_individuals", C.c_uint32), ("words", C.c_uint32), ("words_padded", C.c_uint32),
                ("n_concepts", C.c_uint32), ("n_roles", C.c_uint32), ("n_data", C.c_uint32),
                ("n_pos", C.c_uint64), ("n_neg", C.c_uint64), ("device_bytes", C.c_uint64),
                ("edges", C.c_uint64 * 64), ("heavy", C.c_uint64 * 64), ("n_strings", C.c_uint32),
                ("str_pairs", C.c_uint64 * 32), ("str_values", C.c_uint64 * 32)]


class _ProgInfo(C.Structure):
    _fields_ = [("n_roots", C.c_uint32), ("n_nodes", C.c_uint32), ("n_levels", C.c_uint32),
                ("n_bool", C.c_uint32), ("n_restrict", C.c_uint32), ("n_drange", C.c_uint32),
                ("alg_bytes_total", C.c_double), ("alg_bytes_shared", C.c_double), ("n_string", C.c_uint32)]


class _Names(C.Structure):
    _fields_ = [("n_concepts", C.c_uint32), ("concepts", C.c_void_p), ("n_roles", C.c_uint32),
                ("roles", C.c_void_p), ("n_data", C.c_uint32), ("data", C.c_void_p),
                ("n_strings", C.c_uint32), ("strings", C.c_void_p)]


class _ProfEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("total_ms", C.c_double),
                ("alg_bytes", C.c_double), ("units", C.c_double)]


_lib = None

# hedl_set_allocator callbacks: device memory of the library comes from torch's caching
# allocator (north_star: PyTorch supplies device memory).  Kept referenced for the process.
_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p)


def _torch_alloc(nbytes, device, stream, ctx):
    try:
        import torch
        return torch.cuda.caching_allocator_alloc(int(nbytes), int(device), int(stream or 0))
    except Exception:                  # out of memory (or torch unusable): the library reports OOM
        return None


def _torch_free(ptr, device, stream, ctx):
    try:
        import torch
        torch.cuda.caching_allocator_delete(int(ptr))
    except Exception:                  # interpreter shutdown: torch may already be torn down
        pass


_CALLBACKS = (_ALLOC_FN(_torch_alloc), _FREE_FN(_torch_free))


def use_torch_allocator(on: bool = True):
    """Route the library's device allocations through torch's caching allocator (the default
    once the library is loaded) or back to cudaMalloc / cudaFree.  Only while no KB is alive."""
    if on:
        _check(lib().hedl_set_allocator(C.cast(_CALLBACKS[0], C.c_void_p), C.cast(_CALLBACKS[1], C.c_void_p), None))
    else:
        _check(lib().hedl_set_allocator(None, None, None))


def alloc_counters() -> tuple:
    """(device allocations, device frees) the library has made so far."""
    a, b = C.c_uint64(), C.c_uint64()
    _check(lib().hedl_alloc_counters(C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


def lib():
    """Load libhedl.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    P, U32, U64, I32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
    sig = {
        "hedl_kb_load": ([C.POINTER(_KbDesc), C.c_int, P, C.POINTER(P)], I32),
        "hedl_kb_free": ([P], I32),
        "hedl_kb_get_info": ([P, C.POINTER(_KbInfo)], I32),
        "hedl_compile": ([P, P, U32, P, U64, P, U32, U32, C.POINTER(P)], I32),
        "hedl_compile_ex": ([P, P, U32, P, U64, P, U32, U32, U32, P, P, C.POINTER(P)], I32),
        "hedl_compile_device": ([P, P, U32, P, U64, P, U32, U32, P, C.POINTER(P)], I32),
        "hedl_score_topk": ([P, U32, U32, U32, P, P, P, C.c_int, P], I32),
        "hedl_program_free": ([P], I32),
        "hedl_program_get_info": ([P, C.POINTER(_ProgInfo)], I32),
        "hedl_program_root_bytes": ([P, U32, U32, P], I32),
        "hedl_eval_one": ([P, P, U32, P, P, P], I32),
        "hedl_eval_batch": ([P, P, U32, U32, P, P, P, U32], I32),
        "hedl_program_set_workspace_limit": ([P, U64], I32),
        "hedl_last_error": ([], C.c_char_p),
        "hedl_version": ([], C.c_char_p),
        "hedl_prof_enable": ([C.c_int], I32),
        "hedl_prof_reset": ([], I32),
        "hedl_prof_read": ([C.POINTER(_ProfEntry), C.c_int], C.c_int),
        "hedl_launch_count": ([], U64),
        "hedl_io_counters": ([C.POINTER(U64), C.POINTER(U64)], I32),
        "hedl_set_allocator": ([P, P, P], I32),
        "hedl_alloc_counters": ([C.POINTER(U64), C.POINTER(U64)], I32),
        "hedl_program_workspace_bytes": ([P, P, U32, U32, C.c_int, U32, C.POINTER(U64)], I32),
        "hedl_program_set_workspace": ([P, P, U64], I32),
        "hedl_kb_set_concept_rows": ([P, U32, U32, P, U32, U32, P], I32),
        "hedl_compile_text": ([P, C.POINTER(_Names), P, U32, U32, C.POINTER(P), C.POINTER(U32), C.POINTER(U32)], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    if os.environ.get("HEDL_ALLOCATOR", "torch") == "torch":
        _check(L.hedl_set_allocator(C.cast(_CALLBACKS[0], C.c_void_p), C.cast(_CALLBACKS[1], C.c_void_p), None))
    return L


def _check(code: int):
    if code:
        raise HedlError(code, lib().hedl_last_error().decode(errors="replace"))


def _ptr(a: Optional[np.ndarray]):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _stream(stream):
    import torch
    if stream is None and not torch.cuda.is_available():
        return None               # the library itself reports HEDL_ERR_UNSUPPORTED
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class KB:
    """A loaded knowledge base (hedl_kb*) on one CUDA device."""

    def __init__(self, handle, device: int, n: int):
        self._h = handle
        self._pid = os.getpid()          # a forked child (e.g. a generator pool) never frees it
        self.device = device
        self.N = n
        self.W = (n + 31) // 32

    def info(self) -> dict:
        inf = _KbInfo()
        _check(lib().hedl_kb_get_info(self._h, C.byref(inf)))
        R = inf.n_roles
        return {"N": inf.n_individuals, "W": inf.words, "W4": inf.words_padded, "C": inf.n_concepts,
                "R": R, "D": inf.n_data, "n_pos": inf.n_pos, "n_neg": inf.n_neg,
                "device_bytes": inf.device_bytes, "edges": list(inf.edges[:2 * R]),
                "heavy": list(inf.heavy[:2 * R])}

    def set_concept_rows(self, first: int, rows, parts: int = 1, part_words: Optional[int] = None, stream=None):
        """hedl_kb_set_concept_rows: rows = CUDA int32/uint32 tensor [parts][n][part_words] (or
        [n][W] with parts = 1) holding the complete rows of concepts first .. first+n-1."""
        import torch
        assert rows.is_cuda and rows.is_contiguous() and rows.element_size() == 4
        pw = part_words if part_words is not None else rows.shape[-1]
        n = rows.numel() // (parts * pw) if pw else 0
        with torch.cuda.device(self.device):
            _check(lib().hedl_kb_set_concept_rows(self._h, first, n, C.c_void_p(rows.data_ptr()), parts, pw,
                                                  _stream(stream)))

    def free(self):
        """Release this handle (programs compiled against it keep the KB alive until freed)."""
        if self._h and not getattr(self, "_released", False) and getattr(self, "_pid", None) == os.getpid():
            lib().hedl_kb_free(self._h)
            self._released = True

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Program:
    """A compiled hypothesis batch (hedl_program*)."""

    def __init__(self, handle, kb: KB, n_roots: int):
        self._h = handle
        self._pid = os.getpid()
        self.kb = kb
        self.n_roots = n_roots

    def info(self) -> dict:
        inf = _ProgInfo()
        _check(lib().hedl_program_get_info(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in _ProgInfo._fields_}

    def root_bytes(self, first: int = 0, n: Optional[int] = None) -> np.ndarray:
        n = self.n_roots - first if n is None else n
        out = np.zeros(n, dtype=np.float64)
        _check(lib().hedl_program_root_bytes(self._h, first, n, _ptr(out)))
        return out

    def set_workspace_limit(self, nbytes: int):
        _check(lib().hedl_program_set_workspace_limit(self._h, int(nbytes)))

    def workspace_bytes(self, first: int = 0, n: Optional[int] = None, with_bits: bool = False,
                        flags: int = 0) -> int:
        """hedl_program_workspace_bytes: device bytes one eval_batch(first, n) needs."""
        n = self.n_roots - first if n is None else n
        out = C.c_uint64()
        _check(lib().hedl_program_workspace_bytes(self.kb._h, self._h, first, n, 1 if with_bits else 0, flags,
                                                  C.byref(out)))
        return int(out.value)

    def set_workspace(self, buf):
        """hedl_program_set_workspace over a CUDA tensor (kept referenced here), or None."""
        self._ws = buf
        if buf is None:
            _check(lib().hedl_program_set_workspace(self._h, None, 0))
        else:
            assert buf.is_cuda and buf.is_contiguous()
            _check(lib().hedl_program_set_workspace(self._h, C.c_void_p(buf.data_ptr()),
                                                    buf.numel() * buf.element_size()))

    def free(self):
        if self._h and getattr(self, "_pid", None) == os.getpid():
            lib().hedl_program_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def hedl_kb_load(kb: dict, device: int = 0, stream=None) -> KB:
    """hedl_kb_load over a KB dict with the hedl_kb_desc arrays (see synth/format.py)."""
    import torch
    L = lib()
    arrs = {
        "concept_bits": np.ascontiguousarray(kb["concept_bits"], dtype=np.uint32),
        "role_edge_off": np.ascontiguousarray(kb["role_edge_off"], dtype=np.uint64),
        "edge_subj": np.ascontiguousarray(kb["edge_subj"], dtype=np.uint32),
        "edge_obj": np.ascontiguousarray(kb["edge_obj"], dtype=np.uint32),
        "data_off": np.ascontiguousarray(kb["data_off"], dtype=np.uint64),
        "data_subj": np.ascontiguousarray(kb["data_subj"], dtype=np.uint32),
        "data_val": np.ascontiguousarray(kb["data_val"], dtype=np.float32),
        "pos_ids": np.ascontiguousarray(kb["pos_ids"], dtype=np.uint32),
        "neg_ids": np.ascontiguousarray(kb["neg_ids"], dtype=np.uint32),
        "str_off": np.ascontiguousarray(kb.get("str_off", np.zeros(1, np.uint64)), dtype=np.uint64),
        "str_subj": np.ascontiguousarray(kb.get("str_subj", np.zeros(0, np.uint32)), dtype=np.uint32),
        "str_val_off": np.ascontiguousarray(kb.get("str_val_off", np.zeros(1, np.uint64)), dtype=np.uint64),
        "str_bytes": np.ascontiguousarray(kb.get("str_bytes", np.zeros(0, np.uint8)), dtype=np.uint8),
    }
    cb = arrs["concept_bits"]
    d = _KbDesc()
    d.n_individuals = int(kb["N"])
    d.n_concepts = cb.shape[0] if cb.ndim == 2 else 0
    d.concept_bits = _ptr(cb)
    d.n_roles = len(arrs["role_edge_off"]) - 1
    d.role_edge_off = _ptr(arrs["role_edge_off"])
    d.edge_subj, d.edge_obj = _ptr(arrs["edge_subj"]), _ptr(arrs["edge_obj"])
    d.n_data = len(arrs["data_off"]) - 1
    d.data_off = _ptr(arrs["data_off"])
    d.data_subj, d.data_val = _ptr(arrs["data_subj"]), _ptr(arrs["data_val"])
    d.n_pos, d.pos_ids = len(arrs["pos_ids"]), _ptr(arrs["pos_ids"])
    d.n_neg, d.neg_ids = len(arrs["neg_ids"]), _ptr(arrs["neg_ids"])
    d.n_strings = len(arrs["str_off"]) - 1
    d.str_off, d.str_subj = _ptr(arrs["str_off"]), _ptr(arrs["str_subj"])
    d.str_val_off, d.str_bytes = _ptr(arrs["str_val_off"]), _ptr(arrs["str_bytes"])
    h = C.c_void_p()
    if not torch.cuda.is_available():
        _check(L.hedl_kb_load(C.byref(d), device, None, C.byref(h)))
    with torch.cuda.device(device):
        _check(L.hedl_kb_load(C.byref(d), device, _stream(stream), C.byref(h)))
    return KB(h, device, int(kb["N"]))


def hedl_compile(kb: KB, nodes: np.ndarray, child_idx: np.ndarray, roots: np.ndarray,
                 flags: int = 0, patterns=None) -> Program:
    """patterns: the SEQUAL / SCONTAIN pattern table (list of bytes); defaults to the table a
    synth.format node array carries (`nodes.patterns`).  With patterns -> hedl_compile_ex."""
    if patterns is None:
        patterns = list(getattr(nodes, "patterns", None) or [])
    if patterns:
        return hedl_compile_ex(kb, nodes, child_idx, roots, flags, patterns)
    nodes = np.ascontiguousarray(nodes)
    assert nodes.dtype.itemsize == 28, "nodes must use synth.format.NODE_DTYPE (hedl_node)"
    kids = np.ascontiguousarray(child_idx, dtype=np.uint32)
    roots = np.ascontiguousarray(roots, dtype=np.uint32)
    h = C.c_void_p()
    _check(lib().hedl_compile(kb._h, _ptr(nodes), len(nodes), _ptr(kids), len(kids), _ptr(roots),
                              len(roots), flags, C.byref(h)))
    return Program(h, kb, len(roots))


def hedl_compile_ex(kb: KB, nodes: np.ndarray, child_idx: np.ndarray, roots: np.ndarray,
                    flags: int = 0, patterns=()) -> Program:
    nodes = np.ascontiguousarray(nodes)
    assert nodes.dtype.itemsize == 28, "nodes must use synth.format.NODE_DTYPE (hedl_node)"
    kids = np.ascontiguousarray(child_idx, dtype=np.uint32)
    roots = np.ascontiguousarray(roots, dtype=np.uint32)
    pats = [p.encode() if isinstance(p, str) else bytes(p) for p in patterns]
    off = np.zeros(len(pats) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(p) for p in pats], dtype=np.uint64) if pats else []
    blob = np.frombuffer(b"".join(pats), dtype=np.uint8).copy() if pats else np.zeros(0, np.uint8)
    h = C.c_void_p()
    _check(lib().hedl_compile_ex(kb._h, _ptr(nodes), len(nodes), _ptr(kids), len(kids), _ptr(roots),
                                 len(roots), flags, len(pats), _ptr(off), _ptr(blob), C.byref(h)))
    return Program(h, kb, len(roots))


class ParseError(HedlError):
    """HEDL_ERR_PARSE from hedl_compile_text: .index = hypothesis, .pos = byte offset."""

    def __init__(self, code, msg, index, pos):
        super().__init__(code, msg)
        self.index = index
        self.pos = pos


def _cstr_array(names):
    if names is None:
        return 0, None, None
    enc = [s.encode() if isinstance(s, str) else bytes(s) for s in names]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    return len(enc), C.cast(arr, C.c_void_p), arr


def hedl_compile_text(kb: KB, exprs, names: Optional[dict] = None, flags: int = 0) -> Program:
    """hedl_compile_text: SPEC's s-expression hypotheses (list of str) -> one program.
    names: {"concepts": [...], "roles": [...], "data": [...], "strings": [...]} (each optional;
    a missing list means the spelling c<id> / r<id> / d<id> / s<id>)."""
    names = names or {}
    keep = []
    nm = _Names()
    for f in ("concepts", "roles", "data", "strings"):
        n, p, arr = _cstr_array(names.get(f))
        keep.append(arr)
        setattr(nm, "n_" + f, n)
        setattr(nm, f, p)
    enc = [e.encode() if isinstance(e, str) else bytes(e) for e in exprs]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    h = C.c_void_p()
    ei, ep = C.c_uint32(0), C.c_uint32(0)
    code = lib().hedl_compile_text(kb._h, C.byref(nm), C.cast(arr, C.c_void_p), len(enc), flags, C.byref(h),
                                   C.byref(ei), C.byref(ep))
    if code == 5:
        raise ParseError(code, lib().hedl_last_error().decode(errors="replace"), int(ei.value), int(ep.value))
    _check(code)
    return Program(h, kb, len(enc))


def _dev_u8(a, device):
    """numpy array (any dtype) or CUDA tensor -> (uint8 CUDA tensor sharing the bytes, n elements)."""
    import torch
    if isinstance(a, torch.Tensor):
        assert a.is_cuda and a.is_contiguous()
        return a, None
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr.view(np.uint8).reshape(-1)).to(f"cuda:{device}", non_blocking=False)
    return t, len(arr)


def hedl_compile_device(kb: KB, nodes, child_idx, roots, flags: int = 0, stream=None,
                        n_nodes: Optional[int] = None, n_kids: Optional[int] = None,
                        n_roots: Optional[int] = None) -> Program:
    """hedl_compile_device: the node / child / root arrays in DEVICE memory (CUDA tensors of
    their bytes, with the counts given), or all three in HOST memory (numpy arrays or CPU
    tensors, ideally page-locked): then the library copies them itself
    (HEDL_COMPILE_HOST_INPUT) -- host arrays to program in one C-ABI call."""
    import torch
    host = [not (isinstance(a, torch.Tensor) and a.is_cuda) for a in (nodes, child_idx, roots)]
    if all(host):
        def hp(a, dt):
            if isinstance(a, torch.Tensor):
                assert a.is_contiguous()
                return a, a.data_ptr(), None
            arr = np.ascontiguousarray(a, dtype=dt) if dt is not None else np.ascontiguousarray(a)
            return arr, arr.ctypes.data, len(arr)
        an, pn, nn = hp(nodes, None)
        ak, pk, nk = hp(child_idx, np.uint32)
        ar, pr, nr = hp(roots, np.uint32)
        nn = n_nodes if n_nodes is not None else nn
        nk = n_kids if n_kids is not None else nk
        nr = n_roots if n_roots is not None else nr
        h = C.c_void_p()
        with torch.cuda.device(kb.device):
            _check(lib().hedl_compile_device(kb._h, C.c_void_p(pn), nn, C.c_void_p(pk), nk, C.c_void_p(pr), nr,
                                             flags | HEDL_COMPILE_HOST_INPUT, _stream(stream), C.byref(h)))
        return Program(h, kb, nr)
    with torch.cuda.device(kb.device):
        tn, nn = _dev_u8(nodes, kb.device)
        tk, nk = _dev_u8(np.ascontiguousarray(child_idx, dtype=np.uint32)
                         if not isinstance(child_idx, torch.Tensor) else child_idx, kb.device)
        tr, nr = _dev_u8(np.ascontiguousarray(roots, dtype=np.uint32)
                         if not isinstance(roots, torch.Tensor) else roots, kb.device)
        nn = n_nodes if n_nodes is not None else nn
        nk = n_kids if n_kids is not None else nk
        nr = n_roots if n_roots is not None else nr
        h = C.c_void_p()
        _check(lib().hedl_compile_device(kb._h, C.c_void_p(tn.data_ptr()), nn, C.c_void_p(tk.data_ptr()), nk,
                                         C.c_void_p(tr.data_ptr()), nr, flags, _stream(stream), C.byref(h)))
    return Program(h, kb, nr)


HEDL_SCORE_ACCURACY = 0
HEDL_SCORE_F1 = 1


def hedl_score_topk(counts, metric: int = HEDL_SCORE_ACCURACY, k: int = 0, want_scores: bool = True,
                    stream=None):
    """counts: CUDA int64 tensor [n][4] (tp, fp, fn, tn) -> (scores float64 [n] or None,
    top_idx int32 [k], top_scores float64 [k]) on the same device."""
    import torch
    assert counts.is_cuda and counts.dtype == torch.int64 and counts.is_contiguous()
    n = counts.shape[0]
    dev = counts.device
    with torch.cuda.device(dev):
        sc = torch.empty(n, dtype=torch.float64, device=dev) if want_scores else None
        ti = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        ts = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
        _check(lib().hedl_score_topk(C.c_void_p(counts.data_ptr()), n, metric, k,
                                     C.c_void_p(sc.data_ptr()) if sc is not None else None,
                                     C.c_void_p(ti.data_ptr()), C.c_void_p(ts.data_ptr()),
                                     dev.index if dev.index is not None else torch.cuda.current_device(),
                                     _stream(stream)))
    return sc, ti[:k], ts[:k]


def hedl_eval_one(kb: KB, prog: Program, root: int, want_bits: bool = False, stream=None):
    """-> (bits int32 tensor [W] on the KB's device or None, (tp, fp, fn, tn)).
    The latency path: the library switches to the KB's device itself, so no torch device
    context is entered here (it costs microseconds per call)."""
    import torch
    out = np.zeros(4, dtype=np.uint64)
    bits = None
    if want_bits:
        bits = torch.empty(max(kb.W, 1), dtype=torch.int32, device=f"cuda:{kb.device}")
    st = stream if stream is not None else torch.cuda.current_stream(kb.device)
    _check(lib().hedl_eval_one(kb._h, prog._h, root, C.c_void_p(bits.data_ptr()) if want_bits else None,
                               out.ctypes.data, C.c_void_p(st.cuda_stream)))
    return (bits[:kb.W] if want_bits else None), tuple(int(v) for v in out)


def hedl_eval_batch(kb: KB, prog: Program, first: int = 0, n: Optional[int] = None, want_bits: bool = False,
                    counts_device: bool = False, stream=None, flags: int = 0, out_bits=None, out_counts=None):
    """-> (bits int32 tensor [n][W] or None, counts [n][4] (numpy u64 on host, or int64 tensor on device))."""
    import torch
    n = prog.n_roots - first if n is None else n
    dev = f"cuda:{kb.device}"
    with torch.cuda.device(kb.device):
        bits = out_bits
        if want_bits and bits is None:
            bits = torch.empty((n, max(kb.W, 1)), dtype=torch.int32, device=dev)
        if counts_device:
            counts = out_counts if out_counts is not None else torch.empty((n, 4), dtype=torch.int64, device=dev)
            cptr = C.c_void_p(counts.data_ptr())
            flags |= HEDL_EVAL_COUNTS_DEVICE
        else:
            # page-locked output (torch's pinned caching allocator): the counts D2H runs at
            # full PCIe rate straight into the returned array
            pinned = torch.empty((n, 4), dtype=torch.int64, pin_memory=True) if n >= 4096 else None
            counts = pinned.numpy().view(np.uint64) if pinned is not None else np.zeros((n, 4), dtype=np.uint64)
            cptr = _ptr(counts)
        _check(lib().hedl_eval_batch(kb._h, prog._h, first, n,
                                     C.c_void_p(bits.data_ptr()) if bits is not None else None,
                                     cptr, _stream(stream), flags))
    if bits is not None and kb.W == 0:
        bits = bits[:, :0]
    return bits, counts


def prof_enable(on: bool = True):
    _check(lib().hedl_prof_enable(1 if on else 0))


def prof_reset():
    _check(lib().hedl_prof_reset())


def prof_read() -> list:
    L = lib()
    n = L.hedl_prof_read(None, 0)
    arr = (_ProfEntry * max(n, 1))()
    n = L.hedl_prof_read(arr, n)
    return [{"name": arr[i].name.decode(), "launches": arr[i].launches, "total_ms": arr[i].total_ms,
             "alg_bytes": arr[i].alg_bytes, "units": arr[i].units} for i in range(n)]


def launch_count() -> int:
    return int(lib().hedl_launch_count())


def io_counters() -> tuple:
    a, b = C.c_uint64(), C.c_uint64()
    _check(lib().hedl_io_counters(C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


def version() -> str:
    return lib().hedl_version().decode()
