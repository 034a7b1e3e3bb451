"""paper_2505_04846_b200 -- thin Python binding of the C ABI in include/hiper.h.

B200-native (sm_100a) ColTrast late-interaction scoring from HiPerRAG (arXiv 2505.04846):
``S(q,d) = sum_i max_j <q_i, d_j>`` over NORM'd token embeddings (§2.2
Fig. 3B), driving exact top-k retrieval and the in-batch ColTrast
InfoNCE loss.

This module only marshals arguments (torch tensors -> device pointers, host length arrays, streams)
into ``libhiper.so``; every step of the path runs in the library's CUDA kernels.  There is no CPU
fallback: if the library or an sm_100 device is missing, calls raise ``HiperError``.

Function names follow the C ABI one to one: ``hiper_index_build``, ``hiper_maxsim_topk``,
``hiper_coltrast_scores_loss``, ``hiper_maxsim_scores``, ``hiper_prepare_queries``,
``hiper_infonce_loss``, ``hiper_comm_*``, plus small conveniences (``Index``, ``Comm``).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HIPER_LIB=debug loads the build with device-side checks (libhiper_debug.so; tests/test_gpu_debug_build.py)
LIB_PATH = os.path.join(_HERE, "libhiper_debug.so" if os.environ.get("HIPER_LIB") == "debug"
                        else "libhiper.so")

HIPER_F32, HIPER_BF16 = 0, 1
HIPER_ASSUME_NORMALIZED = 1
HIPER_CHECK_FINITE = 2
HIPER_BORROW_TOKENS = 4
HIPER_VALIDATE_SYNC = 8
HIPER_PACKED = 16
HIPER_POOLED = 32

STATUS = {
    0: "HIPER_OK", 1: "HIPER_ERR_INVALID_ARG", 2: "HIPER_ERR_DIM_MISMATCH",
    3: "HIPER_ERR_EMPTY_TOKENS", 4: "HIPER_ERR_EMPTY_BATCH", 5: "HIPER_ERR_BAD_TEMPERATURE",
    6: "HIPER_ERR_BAD_POSITIVE", 7: "HIPER_ERR_NONFINITE", 8: "HIPER_ERR_ZERO_VECTOR",
    9: "HIPER_ERR_OUT_OF_MEMORY", 10: "HIPER_ERR_CUDA", 11: "HIPER_ERR_NCCL",
    12: "HIPER_ERR_UNSUPPORTED", 13: "HIPER_ERR_WORKSPACE",
}

# Every symbol include/hiper.h declares (tests/test_abi.py checks the header and the .so agree).
EXPORTS = [
    "hiper_status_string", "hiper_last_error", "hiper_version", "hiper_comm_unique_id",
    "hiper_comm_create", "hiper_comm_destroy", "hiper_comm_info", "hiper_index_build",
    "hiper_index_destroy", "hiper_index_info", "hiper_prepare_queries",
    "hiper_maxsim_topk_workspace_size", "hiper_maxsim_topk", "hiper_maxsim_scores_workspace_size",
    "hiper_maxsim_scores", "hiper_coltrast_workspace_size", "hiper_coltrast_scores_loss",
    "hiper_infonce_loss", "hiper_workspace_status", "hiper_last_launch_count",
    "hiper_profile_enable", "hiper_profile_read", "hiper_coltrast_loss_workspace_size",
    "hiper_coltrast_loss", "hiper_coltrast_grad_workspace_size", "hiper_coltrast_scores_loss_grad",
    "hiper_two_stage_workspace_size", "hiper_two_stage_topk", "hiper_pack_plan",
    "hiper_index_pack_info", "hiper_maxsim_topk_keys", "hiper_topk_merge_keys",
    "hiper_profile_read_tagged", "hiper_shard_range", "hiper_coltrast_loss_simulated",
    "hiper_coltrast_loss_simulated_workspace_size",
]


class HiperError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {detail}")


_lib = None


def lib():
    """Load libhiper.so (fails loudly when the extension has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HiperError(12, f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u32, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                            ctypes.c_size_t)
    sig = {
        "hiper_status_string": ([i32], ctypes.c_char_p),
        "hiper_last_error": ([], ctypes.c_char_p),
        "hiper_version": ([], i32),
        "hiper_last_launch_count": ([], i32),
        "hiper_comm_unique_id": ([P], i32),
        "hiper_comm_create": ([P, i32, i32, i32, P], i32),
        "hiper_comm_destroy": ([P], i32),
        "hiper_comm_info": ([P, P, P], i32),
        "hiper_index_build": ([P, i32, P, i64, i32, i32, i64, u32, P, P], i32),
        "hiper_index_destroy": ([P], i32),
        "hiper_index_info": ([P, P, P, P, P, P, P, P], i32),
        "hiper_prepare_queries": ([P, i32, P, i32, i32, i32, u32, P, P, P], i32),
        "hiper_maxsim_topk_workspace_size": ([P, i32, i32, P], sz),
        "hiper_maxsim_topk": ([P, P, i32, P, i32, i32, i32, i32, u32, P, P, sz, P, P, P], i32),
        "hiper_maxsim_scores_workspace_size": ([P, i32], sz),
        "hiper_maxsim_scores": ([P, P, i32, P, i32, i32, i32, u32, P, sz, P, P], i32),
        "hiper_coltrast_workspace_size": ([i32, i32, i32, i32], sz),
        "hiper_coltrast_scores_loss": ([P, P, i32, i32, P, P, i32, i32, i32, i32, u32, P,
                                        ctypes.c_float, P, sz, P, P, P], i32),
        "hiper_infonce_loss": ([P, i32, i32, P, ctypes.c_float, P, sz, P, P], i32),
        "hiper_workspace_status": ([P, P], i32),
        "hiper_profile_enable": ([i32], None),
        "hiper_coltrast_loss_workspace_size": ([i32, i32, i32, i32, i32, P], sz),
        "hiper_coltrast_grad_workspace_size": ([i32, i32, i32, i32], sz),
        "hiper_two_stage_workspace_size": ([P, P, i32, i32, P], sz),
        "hiper_two_stage_topk": ([P, P, P, P, i32, P, i32, i32, i32, i32, u32, P, P, sz, P, P, P], i32),
        "hiper_coltrast_scores_loss_grad": ([P, P, i32, i32, P, P, i32, i32, i32, i32, u32, P,
                                             ctypes.c_float, P, sz, P, P, P, P, P], i32),
        "hiper_coltrast_loss": ([P, P, i32, P, P, i32, i32, P, P, i32, i32, i32, u32, i32,
                                 ctypes.c_float, ctypes.c_float, P, P, sz, P, P, P, P], i32),
        "hiper_profile_read": ([P, P], i32),
        "hiper_pack_plan": ([P, i64, P, P, P, P], i32),
        "hiper_index_pack_info": ([P, P, P, P, P, P], i32),
        "hiper_maxsim_topk_keys": ([P, P, i32, P, i32, i32, i32, i32, u32, P, sz, P, P], i32),
        "hiper_topk_merge_keys": ([P, i32, i32, i32, P, P, P], i32),
        "hiper_profile_read_tagged": ([i32, P, P], i32),
        "hiper_shard_range": ([i64, i32, i32, P, P], i32),
        "hiper_coltrast_loss_simulated_workspace_size": ([i32, i32, i32, i32, i32, i32], sz),
        "hiper_coltrast_loss_simulated": ([P, P, i32, P, P, i32, i32, P, P, i32, i32, i32, u32, i32,
                                           ctypes.c_float, ctypes.c_float, i32, i32, P, sz, P, P, P,
                                           P], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise HiperError(status, lib().hiper_last_error().decode(errors="replace"))


# ---------------------------------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return HIPER_F32
    if t.dtype == torch.bfloat16:
        return HIPER_BF16
    raise TypeError(f"token tensors must be float32 or bfloat16, got {t.dtype}")


def _host_i32(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _stream_ptr(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _keep(buf, stream):
    """The library enqueues on `stream`; a temporary torch allocation (workspace, contiguous copy)
    used by that work must not be recycled by the caching allocator before `stream` reaches it."""
    if buf is not None:
        buf.record_stream(stream if stream is not None else _torch().cuda.current_stream())


def _workspace(nbytes: int, device):
    """1024-B aligned device workspace from the torch caching allocator."""
    torch = _torch()
    buf = torch.empty(int(nbytes) + 1024, dtype=torch.uint8, device=device)
    off = (-buf.data_ptr()) % 1024
    return buf, buf.data_ptr() + off, int(nbytes)


def _dev_ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise HiperError(1, "tensor must live on a CUDA device")
    if not t.is_contiguous():
        raise HiperError(1, "tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


# ---------------------------------------------------------------------------------------- comm
def hiper_shard_range(n: int, world: int, rank: int):
    """(c0, c1): the chunks rank `rank` of `world` holds (the library's shard plan; id_base = c0)."""
    c0, c1 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().hiper_shard_range(int(n), int(world), int(rank), ctypes.byref(c0), ctypes.byref(c1)))
    return c0.value, c1.value


class Comm:
    """NCCL communicator for the corpus-sharded search; bootstrapped over torch.distributed."""

    def __init__(self, group=None, device: int | None = None):
        torch = _torch()
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _check(lib().hiper_comm_unique_id(uid))
        backend_dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=backend_dev)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        dev = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        _check(lib().hiper_comm_create(uid, world, rank, dev, ctypes.byref(h)))
        self.handle, self.world, self.rank = h, world, rank

    def close(self):
        if self.handle:
            _check(lib().hiper_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------------------- index
class Index:
    """Handle of a built corpus layout (hiper_index_build).  Keeps borrowed token storage alive."""

    def __init__(self, handle, keepalive=None):
        self.handle = handle
        self._keep = keepalive
        n, ml, dim, ldp, idb = (ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(),
                                ctypes.c_int32(), ctypes.c_int64())
        lay, lens = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().hiper_index_info(handle, ctypes.byref(n), ctypes.byref(ml), ctypes.byref(dim),
                                      ctypes.byref(ldp), ctypes.byref(idb), ctypes.byref(lay),
                                      ctypes.byref(lens)))
        self.n, self.max_len, self.dim, self.ld_pad = n.value, ml.value, dim.value, ldp.value
        self.id_base, self.layout_ptr, self.lens_ptr = idb.value, lay.value, lens.value
        pk, nt, nr, tp, ep = (ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_void_p(),
                              ctypes.c_void_p())
        _check(lib().hiper_index_pack_info(handle, ctypes.byref(pk), ctypes.byref(nt),
                                           ctypes.byref(nr), ctypes.byref(tp), ctypes.byref(ep)))
        self.packed, self.n_tiles, self.n_rows = bool(pk.value), nt.value, nr.value
        self._tiles_ptr, self._ents_ptr = tp.value, ep.value

    def layout(self):
        """The device layout aliasing the index (test support; valid while the index lives -- clone
        it to keep it): bf16 [n][ld_pad][dim], or [n_rows][dim] for a packed index."""
        torch = _torch()
        if self.packed:
            if self.n_rows == 0:
                return torch.empty((0, self.dim), dtype=torch.bfloat16, device="cuda")
            src = _raw_u8_view(self.layout_ptr, self.n_rows * self.dim * 2)
            return src.view(torch.bfloat16).view(self.n_rows, self.dim)
        if self.n == 0:
            return torch.empty((0, self.ld_pad, self.dim), dtype=torch.bfloat16, device="cuda")
        src = _raw_u8_view(self.layout_ptr, self.n * self.ld_pad * self.dim * 2)
        return src.view(torch.bfloat16).view(self.n, self.ld_pad, self.dim)

    def pack_tables(self):
        """(tiles int32 [n_tiles][4], ents int32 [n][2]) of a packed index, copied to the host."""
        torch = _torch()
        if not self.packed or self.n == 0:
            return np.zeros((0, 4), np.int32), np.zeros((0, 2), np.int32)
        t = _raw_u8_view(self._tiles_ptr, self.n_tiles * 16).view(torch.int32).view(-1, 4)
        e = _raw_u8_view(self._ents_ptr, self.n * 8).view(torch.int32).view(-1, 2)
        return t.cpu().numpy(), e.cpu().numpy()

    def close(self):
        if self.handle:
            _check(lib().hiper_index_destroy(self.handle))
            self.handle = None
            self._keep = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _raw_u8_view(ptr: int, nbytes: int):
    """A torch uint8 CUDA tensor aliasing raw device memory (via __cuda_array_interface__)."""
    torch = _torch()

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3}

    return torch.as_tensor(_Arr(), device="cuda")


def hiper_index_build(tokens, lens, *, id_base: int = 0, flags: int = 0, max_len: int | None = None,
                      stream=None) -> Index:
    """Step a1.  tokens: CUDA tensor [n][max_len][dim] (f32/bf16); lens: host ints [n].
    With HIPER_PACKED | HIPER_BORROW_TOKENS, tokens is the packed bf16 buffer [n_rows][dim]
    (hiper_pack_dst_rows) and n = len(lens); max_len defaults to 256."""
    ln = _host_i32(lens)
    if tokens.dim() == 2:
        if not (flags & HIPER_PACKED and flags & HIPER_BORROW_TOKENS):
            raise HiperError(1, "a 2-D token buffer needs HIPER_PACKED | HIPER_BORROW_TOKENS")
        n, dim = ln.shape[0], tokens.shape[1]
        max_len = max_len or 256
        torch = _torch()
        if tokens.dtype != torch.bfloat16:
            raise HiperError(1, "a borrowed packed buffer must be bfloat16")
        # the library NORMs the buffer in place and writes padding rows up to the plan's n_rows:
        # it cannot see the buffer's size, so check it here
        _, n_rows = hiper_pack_dst_rows(ln) if n else (None, 0)
        if tokens.shape[0] < n_rows:
            raise HiperError(1, f"packed buffer has {tokens.shape[0]} rows < the plan's {n_rows}")
    else:
        n, max_len, dim = tokens.shape
    if ln.shape != (n,):
        raise HiperError(1, f"lens shape {ln.shape} != ({n},)")
    h = ctypes.c_void_p()
    _check(lib().hiper_index_build(_dev_ptr(tokens) if n else None, _dtype_code(tokens), _ptr(ln),
                                   n, max_len, dim, id_base, flags, _stream_ptr(stream),
                                   ctypes.byref(h)))
    keep = tokens if flags & HIPER_BORROW_TOKENS else None
    return Index(h, keep)


def hiper_pack_plan(lens):
    """NEXT N4 packing plan (host only): (tiles int32 [n_tiles][4] = row0, n_rows, e0, e1;
    ents int32 [n][2] = chunk, (col << 16) | len; n_rows total)."""
    ln = _host_i32(lens)
    n = ln.shape[0]
    tiles = np.zeros((max(n, 1), 4), np.int32)
    ents = np.zeros((max(n, 1), 2), np.int32)
    nt, nr = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().hiper_pack_plan(_ptr(ln), n, _ptr(tiles), _ptr(ents), ctypes.byref(nt),
                                 ctypes.byref(nr)))
    return tiles[:nt.value].copy(), ents[:n].copy(), nr.value


def hiper_pack_dst_rows(lens):
    """(dst_row int64 [n], n_rows) of hiper_pack_plan(lens): chunk c's token j lives at packed row
    dst_row[c] + j.  For callers that generate or copy a corpus straight into the packed layout and
    then build with HIPER_PACKED | HIPER_BORROW_TOKENS."""
    tiles, ents, n_rows = hiper_pack_plan(lens)
    n = ents.shape[0]
    dst = np.zeros(n, np.int64)
    if n:
        tile_of_ent = np.repeat(np.arange(len(tiles)), tiles[:, 3] - tiles[:, 2])
        dst[ents[:, 0]] = tiles[tile_of_ent, 0].astype(np.int64) + (ents[:, 1] >> 16)
    return dst, n_rows


def hiper_prepare_queries(q_tokens, q_lens, *, flags: int = 0, stream=None):
    """Step a2 alone: returns (layout bf16 [n_q_pad][32][dim], status uint32[1]) on the device."""
    torch = _torch()
    n_q, q_max_len, dim = q_tokens.shape
    ql = _host_i32(q_lens)
    qs = 32 if q_max_len <= 32 else (64 if q_max_len <= 64 else 128)   # query slot rows
    per = 256 // qs
    n_pad = max(per, (n_q + per - 1) // per * per)
    out = torch.empty((n_pad, qs, dim), dtype=torch.bfloat16, device=q_tokens.device)
    status = torch.zeros(1, dtype=torch.int32, device=q_tokens.device)
    _check(lib().hiper_prepare_queries(_dev_ptr(q_tokens), _dtype_code(q_tokens), _ptr(ql), n_q,
                                       q_max_len, dim, flags, _dev_ptr(out), _dev_ptr(status),
                                       _stream_ptr(stream)))
    return out, status


class TopkWorkspace:
    """Reusable workspace for repeated hiper_maxsim_topk calls of one shape."""

    def __init__(self, index: Index, n_q: int, k: int, comm: Comm | None = None, device=None):
        nb = lib().hiper_maxsim_topk_workspace_size(index.handle, n_q, k,
                                                    comm.handle if comm else None)
        self.buf, self.ptr, self.nbytes = _workspace(nb, device or "cuda")


def hiper_maxsim_topk(index: Index, q_tokens, q_lens, k: int, *, flags: int = 0,
                      comm: Comm | None = None, workspace: TopkWorkspace | None = None,
                      out=None, stream=None):
    """Steps a2-a9: (scores float32 [n_q][k], ids int64 [n_q][k]) on the device."""
    torch = _torch()
    n_q, q_max_len, dim = q_tokens.shape
    ql = _host_i32(q_lens)
    if workspace is None:
        workspace = TopkWorkspace(index, n_q, k, comm, q_tokens.device)
        _keep(workspace.buf, stream)
    if out is None:
        out = (torch.empty((n_q, k), dtype=torch.float32, device=q_tokens.device),
               torch.empty((n_q, k), dtype=torch.int64, device=q_tokens.device))
    _check(lib().hiper_maxsim_topk(index.handle, _dev_ptr(q_tokens), _dtype_code(q_tokens),
                                   _ptr(ql), n_q, q_max_len, dim, k, flags,
                                   comm.handle if comm else None, ctypes.c_void_p(workspace.ptr),
                                   workspace.nbytes, _dev_ptr(out[0]), _dev_ptr(out[1]),
                                   _stream_ptr(stream)))
    return out


def hiper_maxsim_topk_keys(index: Index, q_tokens, q_lens, k: int, *, flags: int = 0,
                           workspace: TopkWorkspace | None = None, out=None, stream=None):
    """a8, first half: this shard's top-k as sortable keys (the all-gather payload), returned as a
    torch int64 tensor [n_q][k] holding the uint64 key bits (include/hiper.h key format)."""
    torch = _torch()
    n_q, q_max_len, dim = q_tokens.shape
    ql = _host_i32(q_lens)
    if workspace is None:
        workspace = TopkWorkspace(index, n_q, k, None, q_tokens.device)
        _keep(workspace.buf, stream)
    if out is None:
        out = torch.empty((n_q, k), dtype=torch.int64, device=q_tokens.device)
    _check(lib().hiper_maxsim_topk_keys(index.handle, _dev_ptr(q_tokens), _dtype_code(q_tokens),
                                        _ptr(ql), n_q, q_max_len, dim, k, flags,
                                        ctypes.c_void_p(workspace.ptr), workspace.nbytes,
                                        _dev_ptr(out), _stream_ptr(stream)))
    return out


def hiper_topk_merge_keys(lists, k: int, *, out=None, stream=None):
    """a8, second half: lists = int64 tensor [n_lists][n_q][k] of uint64 key bits (e.g. the
    all-gathered per-shard keys) -> (scores float32 [n_q][k], ids int64 [n_q][k])."""
    torch = _torch()
    n_lists, n_q, kk = lists.shape
    if kk != k:
        raise HiperError(1, f"lists last dim {kk} != k {k}")
    if out is None:
        out = (torch.empty((n_q, k), dtype=torch.float32, device=lists.device),
               torch.empty((n_q, k), dtype=torch.int64, device=lists.device))
    _check(lib().hiper_topk_merge_keys(_dev_ptr(lists) if lists.numel() else None, n_lists, n_q, k,
                                       _dev_ptr(out[0]), _dev_ptr(out[1]), _stream_ptr(stream)))
    return out


def hiper_maxsim_scores(index: Index, q_tokens, q_lens, *, flags: int = 0, out=None, stream=None):
    """Dense S [n_q][n] (test support; same kernel mainloop as the top-k path)."""
    torch = _torch()
    n_q, q_max_len, dim = q_tokens.shape
    ql = _host_i32(q_lens)
    nb = lib().hiper_maxsim_scores_workspace_size(index.handle, n_q)
    ws, wp, wn = _workspace(nb, q_tokens.device)
    _keep(ws, stream)
    if out is None:
        out = torch.empty((n_q, index.n), dtype=torch.float32, device=q_tokens.device)
    _check(lib().hiper_maxsim_scores(index.handle, _dev_ptr(q_tokens), _dtype_code(q_tokens),
                                     _ptr(ql), n_q, q_max_len, dim, flags, ctypes.c_void_p(wp), wn,
                                     _dev_ptr(out), _stream_ptr(stream)))
    out._hiper_ws = ws  # keep the workspace alive until the stream consumes it
    return out


class ColtrastWorkspace:
    def __init__(self, n_q, n_d, d_max_len, dim, device=None):
        nb = lib().hiper_coltrast_workspace_size(n_q, n_d, d_max_len, dim)
        self.buf, self.ptr, self.nbytes = _workspace(nb, device or "cuda")


def hiper_coltrast_scores_loss(q_tokens, q_lens, d_tokens, d_lens, *, pos_idx=None,
                               temperature: float = 1.0, flags: int = 0, want_scores: bool = True,
                               workspace: ColtrastWorkspace | None = None, out=None, stream=None):
    """Steps a10-a11: (S float32 [n_q][n_d] or None, loss float32 [1]) on the device."""
    torch = _torch()
    n_q, q_max_len, dim = q_tokens.shape
    n_d, d_max_len, dim2 = d_tokens.shape
    if dim2 != dim:
        raise HiperError(2, f"query dim {dim} != doc dim {dim2}")
    if d_tokens.dtype != q_tokens.dtype:
        raise HiperError(1, "query and doc tokens must share a dtype")
    ql, dl = _host_i32(q_lens), _host_i32(d_lens)
    pos = None if pos_idx is None else _host_i32(pos_idx)
    if workspace is None:
        workspace = ColtrastWorkspace(n_q, n_d, d_max_len, dim, q_tokens.device)
        _keep(workspace.buf, stream)
    if out is None:
        S = (torch.empty((n_q, n_d), dtype=torch.float32, device=q_tokens.device)
             if want_scores else None)
        loss = torch.empty(1, dtype=torch.float32, device=q_tokens.device)
    else:
        S, loss = out
    _check(lib().hiper_coltrast_scores_loss(
        _dev_ptr(q_tokens), _ptr(ql), n_q, q_max_len, _dev_ptr(d_tokens), _ptr(dl), n_d, d_max_len,
        dim, _dtype_code(q_tokens), flags, _ptr(pos) if pos is not None else None,
        float(temperature), ctypes.c_void_p(workspace.ptr), workspace.nbytes, _dev_ptr(S),
        _dev_ptr(loss), _stream_ptr(stream)))
    return S, loss


def hiper_infonce_loss(scores, *, pos_idx=None, temperature: float = 1.0, stream=None):
    """Step a11 alone over a device score matrix -> loss float32 [1]."""
    torch = _torch()
    n_q, n_d = scores.shape
    pos = None if pos_idx is None else _host_i32(pos_idx)
    ws, wp, wn = _workspace(max(1024, (n_q * 4 + 1023) // 1024 * 1024), scores.device)
    _keep(ws, stream)
    loss = torch.empty(1, dtype=torch.float32, device=scores.device)
    _check(lib().hiper_infonce_loss(_dev_ptr(scores), n_q, n_d,
                                    _ptr(pos) if pos is not None else None, float(temperature),
                                    ctypes.c_void_p(wp), wn, _dev_ptr(loss), _stream_ptr(stream)))
    loss._hiper_ws = ws
    return loss


def hiper_workspace_status(workspace, stream=None) -> str:
    st = lib().hiper_workspace_status(ctypes.c_void_p(workspace.ptr), _stream_ptr(stream))
    return STATUS.get(st, str(st))


def last_launch_count() -> int:
    return int(lib().hiper_last_launch_count())


def hiper_profile_enable(on: bool = True):
    lib().hiper_profile_enable(int(bool(on)))


HIPER_PROF_MAXSIM, HIPER_PROF_POOLED, HIPER_PROF_RERANK = 0, 1, 2


def hiper_profile_read(tag: int | None = None):
    """(summed kernel milliseconds, launches) of the hot kernels (or of one class `tag`) since the
    last read (synchronises)."""
    ms, n = ctypes.c_double(), ctypes.c_int32()
    if tag is None:
        _check(lib().hiper_profile_read(ctypes.byref(ms), ctypes.byref(n)))
    else:
        _check(lib().hiper_profile_read_tagged(int(tag), ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def hiper_coltrast_loss(q_tokens, q_lens, d_tokens, d_lens, q_pooled, d_pooled, *, n_max: int,
                        tau_li: float = 1.0, tau_c: float = 0.05, comm: Comm | None = None,
                        flags: int = 0, want_scores: bool = False, stream=None):
    """NEXT N2: (losses float32[3] = [L_LI, L_C, L] on the device, S_C [b][m] or None, m).

    Collective over `comm` (every rank calls it with its local batch)."""
    torch = _torch()
    b, q_max_len, dim = q_tokens.shape
    _, d_max_len, _ = d_tokens.shape
    dp = q_pooled.shape[-1]
    ql, dl = _host_i32(q_lens), _host_i32(d_lens)
    world = comm.world if comm else 1
    m = min(n_max, world * b)
    nb = lib().hiper_coltrast_loss_workspace_size(b, d_max_len, dim, dp, n_max,
                                                  comm.handle if comm else None)
    ws, wp, wn = _workspace(nb, q_tokens.device)
    _keep(ws, stream)
    losses = torch.empty(3, dtype=torch.float32, device=q_tokens.device)
    S = torch.empty((b, m), dtype=torch.float32, device=q_tokens.device) if want_scores else None
    mo = ctypes.c_int32()
    _check(lib().hiper_coltrast_loss(
        _dev_ptr(q_tokens), _ptr(ql), q_max_len, _dev_ptr(d_tokens), _ptr(dl), d_max_len, dim,
        _dev_ptr(q_pooled), _dev_ptr(d_pooled), dp, b, _dtype_code(q_tokens), flags, n_max,
        float(tau_li), float(tau_c), comm.handle if comm else None, ctypes.c_void_p(wp), wn,
        _dev_ptr(losses), _dev_ptr(S), ctypes.byref(mo), _stream_ptr(stream)))
    losses._hiper_ws = ws
    return losses, S, mo.value


def hiper_coltrast_loss_simulated(q_tokens, q_lens, d_tokens, d_lens, q_pooled, d_pooled_all, *,
                                  world: int, rank: int, n_max: int, tau_li: float = 1.0,
                                  tau_c: float = 0.05, flags: int = 0, want_scores: bool = False,
                                  stream=None):
    """N2 test support: hiper_coltrast_loss for rank `rank` of `world` simulated ranks on one GPU;
    d_pooled_all [world][b][dp] holds every simulated rank's pooled passages."""
    torch = _torch()
    b, q_max_len, dim = q_tokens.shape
    _, d_max_len, _ = d_tokens.shape
    dp = d_pooled_all.shape[-1]
    ql, dl = _host_i32(q_lens), _host_i32(d_lens)
    m = min(n_max, world * b)
    nb = lib().hiper_coltrast_loss_simulated_workspace_size(b, d_max_len, dim, dp, n_max, world)
    ws, wp, wn = _workspace(nb, q_tokens.device)
    _keep(ws, stream)
    losses = torch.empty(3, dtype=torch.float32, device=q_tokens.device)
    S = torch.empty((b, m), dtype=torch.float32, device=q_tokens.device) if want_scores else None
    mo = ctypes.c_int32()
    _check(lib().hiper_coltrast_loss_simulated(
        _dev_ptr(q_tokens), _ptr(ql), q_max_len, _dev_ptr(d_tokens), _ptr(dl), d_max_len, dim,
        _dev_ptr(q_pooled), _dev_ptr(d_pooled_all), dp, b, _dtype_code(q_tokens), flags, n_max,
        float(tau_li), float(tau_c), world, rank, ctypes.c_void_p(wp), wn, _dev_ptr(losses),
        _dev_ptr(S), ctypes.byref(mo), _stream_ptr(stream)))
    return losses, S, mo.value


def hiper_coltrast_scores_loss_grad(q_tokens, q_lens, d_tokens, d_lens, *, pos_idx=None,
                                    temperature: float = 1.0, flags: int = 0, stream=None):
    """NEXT N1: (S [n_q][n_d], loss [1], grad_q like q_tokens (fp32), grad_d like d_tokens (fp32))."""
    torch = _torch()
    n_q, q_max_len, dim = q_tokens.shape
    n_d, d_max_len, _ = d_tokens.shape
    ql, dl = _host_i32(q_lens), _host_i32(d_lens)
    pos = None if pos_idx is None else _host_i32(pos_idx)
    nb = lib().hiper_coltrast_grad_workspace_size(n_q, n_d, d_max_len, dim)
    ws, wp, wn = _workspace(nb, q_tokens.device)
    _keep(ws, stream)
    dev = q_tokens.device
    S = torch.empty((n_q, n_d), dtype=torch.float32, device=dev)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    gq = torch.empty((n_q, q_max_len, dim), dtype=torch.float32, device=dev)
    gd = torch.empty((n_d, d_max_len, dim), dtype=torch.float32, device=dev)
    _check(lib().hiper_coltrast_scores_loss_grad(
        _dev_ptr(q_tokens), _ptr(ql), n_q, q_max_len, _dev_ptr(d_tokens), _ptr(dl), n_d, d_max_len,
        dim, _dtype_code(q_tokens), flags, _ptr(pos) if pos is not None else None,
        float(temperature), ctypes.c_void_p(wp), wn, _dev_ptr(S), _dev_ptr(loss), _dev_ptr(gq),
        _dev_ptr(gd), _stream_ptr(stream)))
    loss._hiper_ws = ws
    return S, loss, gq, gd


def hiper_two_stage_topk(pooled_index: Index, token_index: Index, q_pooled, q_tokens, q_lens,
                         k1: int, k: int, *, flags: int = 0, comm: Comm | None = None, stream=None):
    """NEXT N3: pooled top-k1 then exact MaxSim rerank -> (scores [n_q][k], ids [n_q][k]).
    With comm, every rank passes its shard's two indexes and receives the global result."""
    torch = _torch()
    n_q, q_max_len, _ = q_tokens.shape
    qp = q_pooled.reshape(n_q, -1)
    if qp.dtype != q_tokens.dtype:
        raise HiperError(1, "pooled and token queries must share a dtype")
    ql = _host_i32(q_lens)
    ch = comm.handle if comm else None
    nb = lib().hiper_two_stage_workspace_size(pooled_index.handle, token_index.handle, n_q, k1, ch)
    ws, wp, wn = _workspace(nb, q_tokens.device)
    _keep(ws, stream)
    qp = qp.contiguous()
    _keep(qp, stream)
    s = torch.empty((n_q, k), dtype=torch.float32, device=q_tokens.device)
    i = torch.empty((n_q, k), dtype=torch.int64, device=q_tokens.device)
    _check(lib().hiper_two_stage_topk(pooled_index.handle, token_index.handle, _dev_ptr(qp),
                                      _dev_ptr(q_tokens), _dtype_code(q_tokens), _ptr(ql), n_q,
                                      q_max_len, k1, k, flags, ch, ctypes.c_void_p(wp), wn,
                                      _dev_ptr(s), _dev_ptr(i), _stream_ptr(stream)))
    s._hiper_ws = ws
    return s, i
