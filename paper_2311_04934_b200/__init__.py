"""B200-native Prompt Cache hot path (arXiv 2311.04934), Python binding.

Thin ctypes layer over ``lib/libpcb200.so`` — the C ABI declared in
``include/promptcache_b200.h``.  Names and semantics mirror the reference's
C++ API (``pc::pml``, ``pc::layout``, ``pc::model``, ``pc::cache``,
``pc::engine``); every numeric op runs in sm_100a kernels.  There is no CPU
fallback: importing works anywhere (host-only PML / layout calls included),
but model creation fails loudly without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "PromptCacheError", "Schema", "Prompt", "Model", "KV", "ModuleStore", "ServeResponse",
    "serve", "serve_batch", "oracle_serve", "TPGroup", "PeerRegion", "peer_group", "nccl_unique_id", "tp_shard_plan", "share_nccl_id", "concat_kv", "config_hash", "config_canonical", "per_token_bytes",
    "F32", "BF16", "FAST", "SLOW", "lib", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCB_LIB_PATH") or os.path.join(HERE, "lib", "libpcb200.so")  # override: A/B builds
F32, BF16 = 0, 1
FAST, SLOW = 0, 1

ERROR_NAMES = [
    "SyntaxError", "MissingSchemaAttr", "UnknownRole", "TokenizerFailure", "FreeTextOverflow", "ArgTooLong",
    "InvalidConfig", "PositionOutOfRange", "ShapeMismatch", "UnknownModule", "CapacityExceeded", "IoError",
    "VersionMismatch", "ConfigHashMismatch", "ValidationFailed", "PositionOverlap", "UnknownCall",
    "RecursionDetected", "DuplicateName", "InvalidProgram", "Internal", "CudaError",
]


class PromptCacheError(RuntimeError):
    """Mirror of pc::Error: ``code`` is the pc::ErrorCode name (errors.hpp:8-30)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.code = ERROR_NAMES[status - 1] if 0 < status <= len(ERROR_NAMES) else "Unknown"


_lib = None


def lib():
    """Load the native library (built by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, cp, i32, i64, u64 = C.c_void_p, C.c_char_p, C.c_int, C.c_int64, C.c_uint64
    pvp = C.POINTER(C.c_void_p)
    sig = {
        "pcb_last_error": (cp, []), "pcb_last_error_code": (i32, []), "pcb_free": (None, [vp]),
        "pcb_version": (cp, []),
        "pcb_schema_parse": (i32, [cp, i32, pvp]), "pcb_schema_from_ast": (i32, [cp, pvp]),
        "pcb_schema_destroy": (None, [vp]), "pcb_schema_to_ast": (vp, [vp]),
        "pcb_schema_serialize": (vp, [vp]), "pcb_schema_plan_json": (vp, [vp]),
        "pcb_prompt_parse": (i32, [cp, pvp]), "pcb_prompt_from_ast": (i32, [cp, pvp]),
        "pcb_prompt_destroy": (None, [vp]), "pcb_prompt_to_ast": (vp, [vp]),
        "pcb_prompt_serialize": (vp, [vp]), "pcb_validate": (vp, [vp, vp]), "pcb_resolve": (vp, [vp, vp]),
        "pcb_config_canonical": (vp, [cp]), "pcb_config_hash": (i32, [cp, C.POINTER(u64)]),
        "pcb_per_token_bytes": (i64, [cp]),
        "pcb_model_create": (i32, [cp, i32, i32, pvp]), "pcb_model_destroy": (None, [vp]),
        "pcb_model_set_option": (i32, [vp, cp, i64]),
        "pcb_model_weight_checksum": (i32, [vp, cp, C.POINTER(u64)]),
        "pcb_model_forward": (i32, [vp, vp, vp, i64, vp, vp, vp, pvp]),
        "pcb_model_generate": (i32, [vp, vp, i32, i64, i32, vp]),
        "pcb_model_forward_tokens": (i64, [vp]), "pcb_model_launches": (i64, [vp]),
        "pcb_model_profile_json": (vp, [vp]), "pcb_model_timer": (i32, [vp, i32, C.POINTER(C.c_double)]),
        "pcb_model_sync": (i32, [vp]),
        "pcb_kv_rows": (i64, [vp]), "pcb_kv_positions": (i32, [vp, vp]),
        "pcb_kv_read": (i32, [vp, i32, i32, vp]), "pcb_kv_upload": (i32, [vp, vp, vp, vp, i64, pvp]),
        "pcb_kv_concat": (i32, [vp, pvp, i32, pvp]), "pcb_kv_destroy": (None, [vp]),
        "pcb_store_create": (i32, [vp, pvp]), "pcb_store_destroy": (None, [vp]),
        "pcb_store_set_capacity": (i32, [vp, i32, i64]),
        "pcb_store_encode_module": (i32, [vp, vp, cp, i32]),
        "pcb_store_encode_schema": (i32, [vp, vp, i32, C.POINTER(i32)]),
        "pcb_store_encode_scaffold": (i32, [vp, vp, cp, i32]),
        "pcb_store_lookup": (i32, [vp, cp, cp, pvp]), "pcb_store_size": (i64, [vp]),
        "pcb_store_put_kv": (i32, [vp, vp, cp, vp, i32]),
        "pcb_store_stats_json": (vp, [vp]), "pcb_store_save": (i32, [vp, cp]),
        "pcb_store_load": (i32, [vp, cp]),
        "pcb_serve": (i32, [vp, vp, vp, i32, i32, i32, pvp]),
        "pcb_oracle_serve": (i32, [vp, vp, vp, i32, pvp]),
        "pcb_serve_batch": (i32, [vp, vp, pvp, i32, i32, pvp]),
        "pcb_nccl_unique_id": (i32, [vp]),
        "pcb_group_create": (i32, [i32, pvp]),
        "pcb_group_destroy": (None, [vp]),
        "pcb_model_create_tp": (i32, [C.c_char_p, i32, i32, i32, i32, vp, vp, pvp]),
        "pcb_peer_create": (i32, [i32, i32, i32, i64, vp, pvp]), "pcb_peer_open": (i32, [vp, vp]),
        "pcb_peer_destroy": (None, [vp]), "pcb_model_create_tp_peer": (i32, [cp, i32, vp, pvp]),
        "pcb_response_json": (vp, [vp]), "pcb_response_tokens": (i32, [vp, vp, i32]),
        "pcb_response_first_logits": (i32, [vp, vp, i32]), "pcb_response_destroy": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(status: int):
    if status:
        raise PromptCacheError(status, lib().pcb_last_error().decode("utf-8", "replace"))


def _take_str(p) -> str:
    if not p:
        _check(lib().pcb_last_error_code() or 21)
    s = C.string_at(p).decode("utf-8", "surrogateescape")
    lib().pcb_free(p)
    return s


def _enc(s: str) -> bytes:
    return s.encode("utf-8", "surrogateescape")


class _Handle:
    _destroy = ""

    def __init__(self, h):
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            getattr(_lib, self._destroy)(h)
            self._h = None

    @property
    def handle(self):
        return self._h


# ---------------------------------------------------------------------------
# PML / layout (pml.hpp:142-155, layout.hpp:88-94)
# ---------------------------------------------------------------------------

class Schema(_Handle):
    """Parsed schema (chat tags expanded with the llama2 template) + its layout plan."""
    _destroy = "pcb_schema_destroy"

    @classmethod
    def parse(cls, pml: str, expand_chat: bool = True) -> "Schema":
        h = C.c_void_p()
        _check(lib().pcb_schema_parse(_enc(pml), int(expand_chat), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_ast(cls, ast) -> "Schema":
        h = C.c_void_p()
        _check(lib().pcb_schema_from_ast(_enc(ast if isinstance(ast, str) else json.dumps(ast)), C.byref(h)))
        return cls(h.value)

    def ast(self) -> dict:
        return json.loads(_take_str(lib().pcb_schema_to_ast(self._h)))

    def serialize(self) -> str:
        return _take_str(lib().pcb_schema_serialize(self._h))

    def plan(self) -> dict:
        return json.loads(_take_str(lib().pcb_schema_plan_json(self._h)))

    @property
    def name(self) -> str:
        return self.ast()["name"]


class Prompt(_Handle):
    _destroy = "pcb_prompt_destroy"

    @classmethod
    def parse(cls, pml: str) -> "Prompt":
        h = C.c_void_p()
        _check(lib().pcb_prompt_parse(_enc(pml), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_ast(cls, ast) -> "Prompt":
        h = C.c_void_p()
        _check(lib().pcb_prompt_from_ast(_enc(ast if isinstance(ast, str) else json.dumps(ast)), C.byref(h)))
        return cls(h.value)

    def ast(self) -> dict:
        return json.loads(_take_str(lib().pcb_prompt_to_ast(self._h)))

    def serialize(self) -> str:
        return _take_str(lib().pcb_prompt_serialize(self._h))

    def validate(self, schema: Schema) -> dict:
        return json.loads(_take_str(lib().pcb_validate(self._h, schema.handle)))

    def resolve(self, schema: Schema) -> dict:
        return json.loads(_take_str(lib().pcb_resolve(self._h, schema.handle)))


def config_canonical(cfg: dict) -> str:
    return _take_str(lib().pcb_config_canonical(_enc(json.dumps(cfg))))


def config_hash(cfg: dict) -> int:
    out = C.c_uint64()
    _check(lib().pcb_config_hash(_enc(json.dumps(cfg)), C.byref(out)))
    return out.value


def per_token_bytes(cfg: dict) -> int:
    return int(lib().pcb_per_token_bytes(_enc(json.dumps(cfg))))


# ---------------------------------------------------------------------------
# Model / KV (model.hpp:34-91)
# ---------------------------------------------------------------------------

class KV(_Handle):
    """Device-resident KV rows ([L][2][rows][hidden], K post-RoPE) + int64 positions."""
    _destroy = "pcb_kv_destroy"

    def __init__(self, h, n_layers: int, hidden: int):
        super().__init__(h)
        self.n_layers, self.hidden = n_layers, hidden

    @property
    def rows(self) -> int:
        return int(lib().pcb_kv_rows(self._h))

    def positions(self) -> np.ndarray:
        out = np.zeros(self.rows, np.int64)
        lib().pcb_kv_positions(self._h, out.ctypes.data)
        return out

    def layer(self, l: int, which: int) -> np.ndarray:
        out = np.zeros((self.rows, self.hidden), np.float32)
        _check(lib().pcb_kv_read(self._h, l, which, out.ctypes.data))
        return out

    def k(self) -> np.ndarray:
        return np.stack([self.layer(l, 0) for l in range(self.n_layers)])

    def v(self) -> np.ndarray:
        return np.stack([self.layer(l, 1) for l in range(self.n_layers)])


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes), created on one rank and shared out of band."""
    buf = C.create_string_buffer(128)
    _check(lib().pcb_nccl_unique_id(buf))
    return buf.raw


def tp_shard_plan(config: dict, tp_size: int) -> list:
    """Per rank, the slices of the reference tensors a head-sharded model holds (mirrors
    Model::Model, model.cpp): rows of wq/wk/wv and w1 and unembed (column-parallel GEMMs),
    columns of wo and w2 (row-parallel GEMMs, all-reduced), heads and KV columns."""
    d = config.get("hidden", config["n_heads"] * config["head_dim"])
    H, V = config["n_heads"], config["vocab_size"]
    if H % tp_size or V % tp_size:
        raise PromptCacheError(3, "InvalidConfig: n_heads and vocab_size must divide by the tensor-parallel size")
    dl, fl, vl = d // tp_size, 4 * d // tp_size, V // tp_size
    return [{"heads": (r * H // tp_size, (r + 1) * H // tp_size), "qkv_rows": (r * dl, (r + 1) * dl),
             "wo_cols": (r * dl, (r + 1) * dl), "kv_cols": (r * dl, (r + 1) * dl),
             "w1_rows": (r * fl, (r + 1) * fl), "w2_cols": (r * fl, (r + 1) * fl),
             "unembed_rows": (r * vl, (r + 1) * vl)} for r in range(tp_size)]


def share_nccl_id(dist, make=None) -> bytes:
    """Rank 0 creates the NCCL unique id, every rank of the torch.distributed group receives it."""
    obj = [(make or nccl_unique_id)() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class TPGroup(_Handle):
    """Tensor-parallel ranks as threads of one process on one device (single-GPU tests of the
    head-sharded path; NCCL is the multi-GPU transport)."""
    _destroy = "pcb_group_destroy"

    def __init__(self, size: int):
        h = C.c_void_p()
        _check(lib().pcb_group_create(size, C.byref(h)))
        super().__init__(h.value)
        self.size = size


class PeerRegion(_Handle):
    """This rank's CUDA-IPC region of a peer-memory tensor-parallel group (one process per
    rank, no NCCL): create, exchange ``handle`` with every rank out of band, then ``open``
    with all handles in rank order (see ``peer_group``)."""
    _destroy = "pcb_peer_destroy"

    def __init__(self, tp_rank: int, tp_size: int, device: int = 0, cap_floats: int = 1 << 22):
        h = C.c_void_p()
        buf = C.create_string_buffer(64)
        _check(lib().pcb_peer_create(tp_rank, tp_size, device, cap_floats, buf, C.byref(h)))
        super().__init__(h.value)
        self.handle_bytes = buf.raw
        self.tp_rank, self.tp_size, self.device = tp_rank, tp_size, device

    def open(self, handles: list[bytes]):
        blob = b"".join(handles)
        _check(lib().pcb_peer_open(self._h, C.create_string_buffer(blob, len(blob))))


def peer_group(dist, device: int = 0, cap_floats: int = 1 << 22) -> PeerRegion:
    """Every rank of a torch.distributed group: its region, opened over all ranks' handles."""
    r = PeerRegion(dist.get_rank(), dist.get_world_size(), device, cap_floats)
    handles = [None] * dist.get_world_size()
    dist.all_gather_object(handles, r.handle_bytes)
    r.open(handles)
    return r


class Model(_Handle):
    _destroy = "pcb_model_destroy"

    def __init__(self, config: dict, dtype: int = BF16, device: int = 0, tp_rank: int = 0, tp_size: int = 1,
                 nccl_id: bytes | None = None, group: "TPGroup | None" = None, peer: "PeerRegion | None" = None):
        """tp_size > 1: head-sharded rank over NCCL (nccl_id), a TPGroup
        (threads), or a PeerRegion (processes sharing CUDA-IPC buffers)."""
        h = C.c_void_p()
        if peer is not None:
            tp_rank, tp_size, device = peer.tp_rank, peer.tp_size, peer.device
            _check(lib().pcb_model_create_tp_peer(_enc(json.dumps(config)), dtype, peer.handle, C.byref(h)))
            self._peer = peer  # the region outlives the model's collectives
        elif tp_size == 1:
            _check(lib().pcb_model_create(_enc(json.dumps(config)), dtype, device, C.byref(h)))
        else:
            nid = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
            _check(lib().pcb_model_create_tp(_enc(json.dumps(config)), dtype, device, tp_rank, tp_size, nid,
                                             group.handle if group else None, C.byref(h)))
        super().__init__(h.value)
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.config = dict(config)
        self.dtype = dtype
        self.n_layers = config.get("n_layers", 4)
        self.hidden = config.get("hidden", config.get("n_heads", 8) * config.get("head_dim", 32))
        self.vocab = config.get("vocab_size", 512)

    def set_option(self, key: str, value: int):
        _check(lib().pcb_model_set_option(self._h, _enc(key), int(value)))

    def weight_checksum(self, name: str) -> int:
        out = C.c_uint64()
        _check(lib().pcb_model_weight_checksum(self._h, _enc(name), C.byref(out)))
        return out.value

    def forward(self, tokens, positions, past: KV | None = None, mask=None, want_kv: bool = True):
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int64)
        n = len(t)
        if len(p) != n:  # reference model.cpp:312-313
            raise PromptCacheError(9, "ShapeMismatch: tokens/position_ids length mismatch")
        logits = np.zeros((n, self.vocab), np.float32)
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        kv = C.c_void_p()
        _check(lib().pcb_model_forward(self._h, t.ctypes.data, p.ctypes.data, n, past.handle if past else None,
                                       mk.ctypes.data if mk is not None else None, logits.ctypes.data,
                                       C.byref(kv) if want_kv else None))
        return logits, (KV(kv.value, self.n_layers, self.hidden) if want_kv else None)

    def generate(self, kv: KV, last_token: int, last_position: int, n_steps: int) -> list[int]:
        out = np.zeros(max(n_steps, 1), np.int32)
        _check(lib().pcb_model_generate(self._h, kv.handle, last_token, last_position, n_steps, out.ctypes.data))
        return out[:n_steps].tolist()

    def upload_kv(self, k: np.ndarray, v: np.ndarray, positions) -> KV:
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        p = np.ascontiguousarray(positions, np.int64)
        h = C.c_void_p()
        _check(lib().pcb_kv_upload(self._h, k.ctypes.data, v.ctypes.data, p.ctypes.data, len(p), C.byref(h)))
        return KV(h.value, self.n_layers, self.hidden)

    @property
    def forward_tokens(self) -> int:
        return int(lib().pcb_model_forward_tokens(self._h))

    def profile(self) -> dict:
        """Per kernel class CUDA-event times since the last call (needs set_option("profile", 1))."""
        return json.loads(_take_str(lib().pcb_model_profile_json(self._h)))

    def timer_start(self):
        """Record a CUDA event on the model's stream (device-side timing of a region)."""
        _check(lib().pcb_model_timer(self._h, 0, None))

    def timer_stop(self) -> float:
        """Record the end event, wait for it; returns device milliseconds since timer_start()."""
        ms = C.c_double()
        _check(lib().pcb_model_timer(self._h, 1, C.byref(ms)))
        return ms.value

    @property
    def launches(self) -> int:
        return int(lib().pcb_model_launches(self._h))

    def sync(self):
        _check(lib().pcb_model_sync(self._h))


def concat_kv(model: Model, kvs: list[KV]) -> KV:
    arr = (C.c_void_p * len(kvs))(*[k.handle for k in kvs])
    h = C.c_void_p()
    _check(lib().pcb_kv_concat(model.handle, arr, len(kvs), C.byref(h)))
    return KV(h.value, model.n_layers, model.hidden)


# ---------------------------------------------------------------------------
# Store / engine (cache.hpp:46-108, engine.hpp:13-62)
# ---------------------------------------------------------------------------

class ModuleStore(_Handle):
    _destroy = "pcb_store_destroy"

    def __init__(self, model: Model):
        h = C.c_void_p()
        _check(lib().pcb_store_create(model.handle, C.byref(h)))
        super().__init__(h.value)
        self.model = model  # keep the model alive

    def set_capacity(self, tier: int, nbytes: int):
        _check(lib().pcb_store_set_capacity(self._h, tier, nbytes))

    def encode_module(self, schema: Schema, name: str, tier: int = FAST):
        _check(lib().pcb_store_encode_module(self._h, schema.handle, _enc(name), tier))

    def encode_schema(self, schema: Schema, tier: int = FAST) -> int:
        n = C.c_int()
        _check(lib().pcb_store_encode_schema(self._h, schema.handle, tier, C.byref(n)))
        return n.value

    def encode_scaffold(self, schema: Schema, members: list[str], tier: int = FAST):
        _check(lib().pcb_store_encode_scaffold(self._h, schema.handle, _enc(json.dumps(members)), tier))

    def put_kv(self, schema: Schema, name: str, kv: KV, tier: int = FAST):
        """Install precomputed rows as module `name` (rows/positions must be its schema span)."""
        _check(lib().pcb_store_put_kv(self._h, schema.handle, _enc(name), kv.handle, tier))

    def lookup(self, schema_name: str, name: str) -> KV | None:
        h = C.c_void_p()
        _check(lib().pcb_store_lookup(self._h, _enc(schema_name), _enc(name), C.byref(h)))
        return KV(h.value, self.model.n_layers, self.model.hidden) if h.value else None

    def __len__(self):
        return int(lib().pcb_store_size(self._h))

    def stats(self) -> dict:
        return json.loads(_take_str(lib().pcb_store_stats_json(self._h)))

    def save(self, path: str):
        _check(lib().pcb_store_save(self._h, _enc(path)))

    def load(self, path: str):
        _check(lib().pcb_store_load(self._h, _enc(path)))


@dataclass
class ServeResponse:
    output_tokens: list[int]
    output_text: str
    first_token_logits: np.ndarray
    timings: dict = field(default_factory=dict)
    cache_report: dict = field(default_factory=dict)

    @classmethod
    def _from(cls, h, vocab: int) -> "ServeResponse":
        L = lib()
        try:
            j = json.loads(_take_str(L.pcb_response_json(h)))
            logits = np.zeros(vocab, np.float32)
            n = L.pcb_response_first_logits(h, logits.ctypes.data, vocab)
            return cls(j["output_tokens"], j["output_text"], logits[:n], j["timings"], j["cache_report"])
        finally:
            L.pcb_response_destroy(h)


def _prompt(p) -> Prompt:
    return p if isinstance(p, Prompt) else (Prompt.parse(p) if isinstance(p, str) else Prompt.from_ast(p))


def serve(store: ModuleStore, schema: Schema, prompt, max_new_tokens: int = 16, use_cache: bool = True,
          use_scaffolds: bool = False) -> ServeResponse:
    """engine::serve (reference engine.cpp:187-258) on the device."""
    p = _prompt(prompt)
    h = C.c_void_p()
    _check(lib().pcb_serve(store.handle, schema.handle, p.handle, max_new_tokens, int(use_cache),
                           int(use_scaffolds), C.byref(h)))
    return ServeResponse._from(h.value, store.model.vocab)


def serve_batch(store: ModuleStore, schema: Schema, prompts, micro_batch: int = 4, after=None) -> list:
    """engine::serve_batch: first tokens of many requests, micro_batch requests per assembly
    launch and suffix prefill.  ``after`` (optional) is called as soon
    as the native call returns, before the Python response objects are built (timing)."""
    ps = [_prompt(p) for p in prompts]
    n = len(ps)
    arr = (C.c_void_p * max(n, 1))(*[p.handle for p in ps])
    outs = (C.c_void_p * max(n, 1))()
    _check(lib().pcb_serve_batch(store.handle, schema.handle, arr, n, micro_batch, outs))
    if after is not None:
        after()
    return [ServeResponse._from(outs[i], store.model.vocab) for i in range(n)]


def oracle_serve(model: Model, schema: Schema, prompt, max_new_tokens: int = 16) -> ServeResponse:
    """engine::oracle_serve (reference engine.cpp:260-334): exact block-masked pass on the device."""
    p = _prompt(prompt)
    h = C.c_void_p()
    _check(lib().pcb_oracle_serve(model.handle, schema.handle, p.handle, max_new_tokens, C.byref(h)))
    return ServeResponse._from(h.value, model.vocab)
