"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the CPU checkers.

* ``Ref``  — the unmodified reference library (oracle/_ref/libpcref_*.so, built by
  oracle/Makefile from /root/reference sources + oracle/ref_shim.cpp).
* ``COracle`` — our plain-C restatement (oracle/liboracle.so, pc_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    fl = set(line.split())
                    return {"avx512f", "avx512bw", "avx512vl", "avx512dq", "avx512cd"} <= fl
    except OSError:
        pass
    return False


def ref_lib_path() -> str:
    isa = "v4" if _cpu_has_avx512() else "v3"
    return os.path.join(REF_DIR, f"libpcref_{isa}.so")


def build(ref: bool = True) -> None:
    """Build the C oracle, and the reference shim when /root/reference exists."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def ref_available() -> bool:
    return os.path.exists(ref_lib_path())


TINY = dict(n_layers=4, n_heads=8, head_dim=32, hidden=256, vocab_size=512,
            pos_encoding="rope", max_position=8192, bytes_per_element=4, seed=42)
C1 = dict(n_layers=2, n_heads=4, head_dim=64, hidden=256, vocab_size=512,
          pos_encoding="rope", max_position=8192, bytes_per_element=4, seed=42)


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Ref:
    """Bindings over oracle/ref_shim.cpp (each forwards to the reference function)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            path = ref_lib_path()
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
            L = C.CDLL(path)
            vp, cp, i32, i64, u64 = C.c_void_p, C.c_char_p, C.c_int, C.c_int64, C.c_uint64
            L.pcref_last_error.restype = cp
            L.pcref_free.argtypes = [vp]
            L.pcref_model_create.restype = vp
            L.pcref_model_create.argtypes = [cp]
            L.pcref_model_destroy.argtypes = [vp]
            L.pcref_config_hash.argtypes = [cp, C.POINTER(u64)]
            L.pcref_config_canonical.restype = vp
            L.pcref_config_canonical.argtypes = [cp]
            L.pcref_weight_checksum.argtypes = [vp, cp, C.POINTER(u64)]
            L.pcref_forward.argtypes = [vp, vp, vp, i64, vp, vp, vp, C.POINTER(vp)]
            L.pcref_generate.argtypes = [vp, vp, i32, i64, i32, vp]
            L.pcref_forward_tokens.restype = i64
            L.pcref_forward_tokens.argtypes = [vp]
            L.pcref_kv_destroy.argtypes = [vp]
            L.pcref_kv_rows.restype = i64
            L.pcref_kv_rows.argtypes = [vp]
            L.pcref_kv_positions.argtypes = [vp, vp]
            L.pcref_kv_layer.argtypes = [vp, i32, i32, vp]
            L.pcref_kv_synthetic.restype = vp
            L.pcref_kv_synthetic.argtypes = [i32, i32, i64, u64]
            L.pcref_kv_from_arrays.restype = vp
            L.pcref_kv_from_arrays.argtypes = [i32, i32, i64, vp, vp, vp]
            L.pcref_kv_concat.restype = vp
            L.pcref_kv_concat.argtypes = [C.POINTER(vp), i32]
            for fn in ("pcref_parse_schema",):
                getattr(L, fn).restype = vp
                getattr(L, fn).argtypes = [cp, i32]
            L.pcref_parse_prompt.restype = vp
            L.pcref_parse_prompt.argtypes = [cp]
            L.pcref_serialize_schema.restype = vp
            L.pcref_serialize_schema.argtypes = [cp]
            L.pcref_serialize_prompt.restype = vp
            L.pcref_serialize_prompt.argtypes = [cp]
            L.pcref_validate.restype = vp
            L.pcref_validate.argtypes = [cp, i32, cp, i32]
            L.pcref_plan.restype = vp
            L.pcref_plan.argtypes = [cp, i32]
            L.pcref_resolve.restype = vp
            L.pcref_resolve.argtypes = [cp, i32, cp, i32]
            L.pcref_random_case.restype = vp
            L.pcref_random_case.argtypes = [C.c_uint32]
            L.pcref_random_ast.restype = vp
            L.pcref_random_ast.argtypes = [C.c_uint32]
            L.pcref_synthetic_text.restype = vp
            L.pcref_synthetic_text.argtypes = [i64, u64]
            L.pcref_encode_module.restype = vp
            L.pcref_encode_module.argtypes = [vp, cp, i32, cp]
            L.pcref_encode_scaffold.restype = vp
            L.pcref_encode_scaffold.argtypes = [vp, cp, i32, cp]
            L.pcref_serve.restype = vp
            L.pcref_serve.argtypes = [vp, cp, i32, cp, i32, i32, i32, cp, i32]
            L.pcref_time_cached_step.argtypes = [vp, vp, i64, i64, C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double)]
            L.pcref_store_save.argtypes = [vp, cp, i32, cp, cp]
            L.pcref_per_token_bytes.restype = i64
            L.pcref_per_token_bytes.argtypes = [cp]
            cls._lib = L
        return cls._lib

    # ---- helpers ----
    @classmethod
    def _str(cls, p) -> str:
        L = cls.lib()
        if not p:
            raise RefError(-1, L.pcref_last_error().decode())
        s = C.string_at(p).decode("utf-8", "surrogateescape")
        L.pcref_free(p)
        return s

    @classmethod
    def _json(cls, p):
        return json.loads(cls._str(p))

    @staticmethod
    def _b(s):
        if isinstance(s, (dict, list)):
            s = json.dumps(s)
        return s.encode("utf-8", "surrogateescape")

    @staticmethod
    def _is_ast(s):
        return 1 if isinstance(s, (dict, list)) else 0

    # ---- pml / layout ----
    @classmethod
    def parse_schema(cls, text: str, expand: bool = True):
        return cls._json(cls.lib().pcref_parse_schema(cls._b(text), int(expand)))

    @classmethod
    def parse_prompt(cls, text: str):
        return cls._json(cls.lib().pcref_parse_prompt(cls._b(text)))

    @classmethod
    def serialize_schema(cls, ast) -> str:
        return cls._str(cls.lib().pcref_serialize_schema(cls._b(ast)))

    @classmethod
    def serialize_prompt(cls, ast) -> str:
        return cls._str(cls.lib().pcref_serialize_prompt(cls._b(ast)))

    @classmethod
    def validate(cls, prompt, schema):
        return cls._json(cls.lib().pcref_validate(cls._b(prompt), cls._is_ast(prompt),
                                                  cls._b(schema), cls._is_ast(schema)))

    @classmethod
    def plan(cls, schema):
        return cls._json(cls.lib().pcref_plan(cls._b(schema), cls._is_ast(schema)))

    @classmethod
    def resolve(cls, schema, prompt):
        return cls._json(cls.lib().pcref_resolve(cls._b(schema), cls._is_ast(schema),
                                                 cls._b(prompt), cls._is_ast(prompt)))

    @classmethod
    def random_case(cls, seed: int):
        return cls._json(cls.lib().pcref_random_case(seed))

    @classmethod
    def random_ast(cls, seed: int):
        return cls._json(cls.lib().pcref_random_ast(seed))

    @classmethod
    def synthetic_text(cls, n: int, seed: int) -> str:
        return cls._str(cls.lib().pcref_synthetic_text(n, seed))

    @classmethod
    def per_token_bytes(cls, cfg: dict) -> int:
        return cls.lib().pcref_per_token_bytes(json.dumps(cfg).encode())

    @classmethod
    def config_hash(cls, cfg: dict) -> int:
        out = C.c_uint64()
        cls.lib().pcref_config_hash(json.dumps(cfg).encode(), C.byref(out))
        return out.value


class RefKV:
    def __init__(self, h, n_layers, hidden):
        self.h, self.n_layers, self.hidden = h, n_layers, hidden

    def __del__(self):
        if self.h and Ref._lib is not None:
            Ref._lib.pcref_kv_destroy(self.h)
            self.h = None

    @property
    def rows(self) -> int:
        return Ref.lib().pcref_kv_rows(self.h)

    def positions(self) -> np.ndarray:
        out = np.zeros(self.rows, np.int64)
        Ref.lib().pcref_kv_positions(self.h, out.ctypes.data)
        return out

    def layer(self, l: int, which: int) -> np.ndarray:
        out = np.zeros((self.rows, self.hidden), np.float32)
        Ref.lib().pcref_kv_layer(self.h, l, which, out.ctypes.data)
        return out

    def k(self) -> np.ndarray:
        return np.stack([self.layer(l, 0) for l in range(self.n_layers)])

    def v(self) -> np.ndarray:
        return np.stack([self.layer(l, 1) for l in range(self.n_layers)])


class RefModel:
    def __init__(self, cfg: dict):
        self.cfg = dict(cfg)
        L = Ref.lib()
        self.h = L.pcref_model_create(json.dumps(cfg).encode())
        if not self.h:
            raise RefError(-1, L.pcref_last_error().decode())
        self.n_layers, self.hidden, self.vocab = cfg["n_layers"], cfg["hidden"], cfg["vocab_size"]

    def __del__(self):
        if getattr(self, "h", None) and Ref._lib is not None:
            Ref._lib.pcref_model_destroy(self.h)
            self.h = None

    def weight_checksum(self, name: str) -> int:
        out = C.c_uint64()
        rc = Ref.lib().pcref_weight_checksum(self.h, name.encode(), C.byref(out))
        if rc:
            raise RefError(rc, Ref.lib().pcref_last_error().decode())
        return out.value

    def forward(self, tokens, positions, past: RefKV | None = None, mask=None):
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int64)
        n = len(t)
        logits = np.zeros((n, self.vocab), np.float32)
        kv = C.c_void_p()
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        rc = Ref.lib().pcref_forward(self.h, t.ctypes.data, p.ctypes.data, n,
                                     past.h if past else None,
                                     mk.ctypes.data if mk is not None else None,
                                     logits.ctypes.data, C.byref(kv))
        if rc:
            raise RefError(rc, Ref.lib().pcref_last_error().decode())
        return logits, RefKV(kv.value, self.n_layers, self.hidden)

    def generate(self, kv: RefKV, last_token: int, last_pos: int, n_steps: int):
        out = np.zeros(max(n_steps, 1), np.int32)
        Ref.lib().pcref_generate(self.h, kv.h, last_token, last_pos, n_steps, out.ctypes.data)
        return out[:n_steps].tolist()

    def encode_module(self, schema, name: str) -> RefKV:
        h = Ref.lib().pcref_encode_module(self.h, Ref._b(schema), Ref._is_ast(schema), name.encode())
        if not h:
            raise RefError(-1, Ref.lib().pcref_last_error().decode())
        return RefKV(h, self.n_layers, self.hidden)

    def encode_scaffold(self, schema, members) -> RefKV:
        h = Ref.lib().pcref_encode_scaffold(self.h, Ref._b(schema), Ref._is_ast(schema),
                                            json.dumps(members).encode())
        if not h:
            raise RefError(-1, Ref.lib().pcref_last_error().decode())
        return RefKV(h, self.n_layers, self.hidden)

    def serve(self, schema, prompt, max_new: int = 4, mode: str = "cached", scaffold=None,
              slow: bool = False):
        m = {"cached": 0, "baseline": 1, "oracle": 2}[mode]
        sc = json.dumps(scaffold).encode() if scaffold else b""
        p = Ref.lib().pcref_serve(self.h, Ref._b(schema), Ref._is_ast(schema), Ref._b(prompt),
                                  Ref._is_ast(prompt), max_new, m, sc, int(slow))
        return Ref._json(p)

    def store_save(self, schema, path: str, scaffold=None):
        sc = json.dumps(scaffold).encode() if scaffold else b""
        rc = Ref.lib().pcref_store_save(self.h, Ref._b(schema), Ref._is_ast(schema), sc, path.encode())
        if rc:
            raise RefError(rc, Ref.lib().pcref_last_error().decode())


def ref_kv(k, v, positions) -> "RefKV":
    """A reference KVState holding k/v [L][rows][hidden] (fp32) at `positions`."""
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    p = np.ascontiguousarray(positions, np.int64)
    h = Ref.lib().pcref_kv_from_arrays(k.shape[0], k.shape[2], len(p), k.ctypes.data, v.ctypes.data, p.ctypes.data)
    return RefKV(h, k.shape[0], k.shape[2])


def ref_concat(kvs):
    arr = (C.c_void_p * len(kvs))(*[k.h for k in kvs])
    h = Ref.lib().pcref_kv_concat(arr, len(kvs))
    if not h:
        raise RefError(-1, Ref.lib().pcref_last_error().decode())
    return RefKV(h, kvs[0].n_layers, kvs[0].hidden)


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------

class _Cfg(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("n_heads", C.c_int), ("head_dim", C.c_int),
                ("hidden", C.c_int), ("vocab_size", C.c_int), ("pos_encoding", C.c_int),
                ("max_position", C.c_int64), ("seed", C.c_uint64)]


_POS = {"rope": 0, "alibi": 1, "abs_table": 2}


class COracle:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            path = os.path.join(HERE, "liboracle.so")
            if not os.path.exists(path):
                build(ref=False)
            L = C.CDLL(path)
            vp = C.c_void_p
            L.pco_model_create.restype = vp
            L.pco_model_create.argtypes = [C.POINTER(_Cfg)]
            L.pco_model_destroy.argtypes = [vp]
            L.pco_weight_checksum.argtypes = [vp, C.c_char_p, C.POINTER(C.c_uint64)]
            L.pco_forward.argtypes = [vp, vp, vp, C.c_int64, vp, vp, vp, C.c_int64, vp, vp, vp, vp]
            L.pco_fill_uniform.argtypes = [vp, C.c_uint64, C.c_char_p, C.c_uint64, C.c_float]
            L.pco_argmax_lowest.argtypes = [vp, C.c_int]
            cls._lib = L
        return cls._lib

    def __init__(self, cfg: dict):
        self.cfg = dict(cfg)
        c = _Cfg(cfg["n_layers"], cfg["n_heads"], cfg["head_dim"], cfg["hidden"], cfg["vocab_size"],
                 _POS[cfg.get("pos_encoding", "rope")], cfg["max_position"], cfg["seed"])
        self.h = self.lib().pco_model_create(C.byref(c))
        if not self.h:
            raise ValueError("bad config")

    def __del__(self):
        if getattr(self, "h", None) and COracle._lib is not None:
            COracle._lib.pco_model_destroy(self.h)
            self.h = None

    def weight_checksum(self, name: str) -> int:
        out = C.c_uint64()
        rc = self.lib().pco_weight_checksum(self.h, name.encode(), C.byref(out))
        if rc:
            raise KeyError(name)
        return out.value

    def forward(self, tokens, positions, past_k=None, past_v=None, past_pos=None, mask=None):
        """Returns (logits [n,V], new_k [L,n,d], new_v [L,n,d])."""
        c = self.cfg
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int64)
        n = len(t)
        P = 0 if past_k is None else past_k.shape[1]
        pk = None if past_k is None else np.ascontiguousarray(past_k, np.float32)
        pv = None if past_v is None else np.ascontiguousarray(past_v, np.float32)
        pp = None if past_pos is None else np.ascontiguousarray(past_pos, np.int64)
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        logits = np.zeros((n, c["vocab_size"]), np.float32)
        nk = np.zeros((c["n_layers"], n, c["hidden"]), np.float32)
        nv = np.zeros_like(nk)
        rc = self.lib().pco_forward(self.h, t.ctypes.data, p.ctypes.data, n,
                                    pk.ctypes.data if pk is not None else None,
                                    pv.ctypes.data if pv is not None else None,
                                    pp.ctypes.data if pp is not None else None, P,
                                    mk.ctypes.data if mk is not None else None,
                                    logits.ctypes.data, nk.ctypes.data, nv.ctypes.data)
        if rc:
            raise ValueError(f"oracle forward error {rc}")
        return logits, nk, nv

    @classmethod
    def fill_uniform(cls, count: int, name: str, seed: int, scale: float) -> np.ndarray:
        out = np.zeros(count, np.float32)
        cls.lib().pco_fill_uniform(out.ctypes.data, count, name.encode(), seed, C.c_float(scale))
        return out


def max_rel_diff(a, b) -> float:
    """tests/common.hpp:235-244: max |a-b| / max(1, |a|)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        return 1e30
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(a))))
