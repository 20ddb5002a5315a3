"""Device plumbing shared by the drop-in modules: the CUDA device/stream,
reusable workspaces, pinned host staging, and the uniform stream that
carries the reference's RNG protocol onto the device.

PyTorch is used only for device memory and streams; all compute goes
through `_abi.lib`.
"""

from __future__ import annotations

import threading

import numpy as np
import torch


# algorithmic HBM bytes of the work issued so far (weights + K/V views of every
# forward, K reads + gathers of every retrieval build); bench.py differences it
# around its timed region for the per-token roofline
STATS = {"alg_bytes": 0}


_CUDA_OK = False
# torch's C entry points for the current device / raw stream: torch.cuda.
# current_stream() re-validates the device through Python helpers (~10 us a
# call, several calls per decode round on the host's critical path between a
# round's read-back and its next launch)
_get_device = torch._C._cuda_getDevice
_get_raw_stream = torch._C._cuda_getCurrentRawStream


def device() -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2404_11912_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
        torch.cuda.init()
        _CUDA_OK = True
    return torch.device("cuda", _get_device())


def stream_ptr() -> int:
    """cudaStream_t of this thread's current stream on the current device."""
    if not _CUDA_OK:
        device()
    return _get_raw_stream(_get_device())


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


class _Workspaces:
    """Grow-only scratch buffers keyed by purpose and by the current stream:
    work on one stream is ordered, so reuse is safe; concurrent streams (the
    host threads of a loopback shard group) never share one."""

    def __init__(self):
        self.bufs = {}

    def get(self, key: str, nbytes: int) -> torch.Tensor:
        k = (key, stream_ptr())
        b = self.bufs.get(k)
        if b is None or b.numel() < nbytes:
            b = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device())
            self.bufs[k] = b
        return b


workspaces = _Workspaces()


class _PinnedStaging:
    """Ring of pinned host buffers for the small per-step host->device
    copies (token ids, uniforms).  A copy from pageable memory makes torch
    synchronise the stream -- the GPU would drain and idle while the host
    prepares the next step; a pinned, non-blocking copy is stream-ordered and
    returns at once.  A slot is reused only after its previous copy ran."""

    def __init__(self, slots: int = 32, cap: int = 8192):
        self.slots, self.cap = slots, cap
        self.bufs = {}
        self.events = [None] * slots
        self.i = 0

    _NP = {torch.int32: np.int32, torch.float32: np.float32, torch.float64: np.float64, torch.int64: np.int64}

    def _slot(self) -> int:
        """Next ring slot, once its previous copy has run (events are reused)."""
        slot = self.i
        self.i = (self.i + 1) % self.slots
        ev = self.events[slot]
        if ev is None:
            self.events[slot] = torch.cuda.Event()
        else:
            ev.synchronize()
        return slot

    def copy_into(self, dst: torch.Tensor, arr) -> None:
        """Stream-ordered copy of a small host array into an existing device
        tensor (fixed address: inputs of captured CUDA graphs)."""
        arr = np.ascontiguousarray(arr, dtype=self._NP[dst.dtype])
        slot = self._slot()
        key = (slot, arr.dtype.str)
        buf = self.bufs.get(key)
        if buf is None:
            buf = torch.empty(self.cap, dtype=dst.dtype, pin_memory=True)
            self.bufs[key] = buf
        host = buf[:arr.size]
        host.numpy()[:] = arr.reshape(-1)
        dst.view(-1)[:arr.size].copy_(host, non_blocking=True)
        self.events[slot].record()

    def to_device(self, arr: np.ndarray) -> torch.Tensor:
        arr = np.ascontiguousarray(arr)
        if arr.size > self.cap:
            return torch.from_numpy(arr).to(device())
        slot = self._slot()
        key = (slot, arr.dtype.str)
        buf = self.bufs.get(key)
        if buf is None:
            buf = torch.empty(self.cap, dtype=torch.from_numpy(arr[:0]).dtype, pin_memory=True)
            self.bufs[key] = buf
        host = buf[:arr.size]
        host.numpy()[:] = arr.reshape(-1)
        out = torch.empty(arr.shape, dtype=host.dtype, device=device())
        out.view(-1).copy_(host, non_blocking=True)
        self.events[slot].record()
        return out


class _ThreadStaging:
    """One staging ring per host thread (its events are recorded on that
    thread's current stream)."""

    def __init__(self):
        self._tl = threading.local()

    def _ring(self) -> _PinnedStaging:
        r = getattr(self._tl, "ring", None)
        if r is None:
            r = self._tl.ring = _PinnedStaging()
        return r

    def copy_into(self, dst: torch.Tensor, arr) -> None:
        self._ring().copy_into(dst, arr)

    def to_device(self, arr: np.ndarray) -> torch.Tensor:
        return self._ring().to_device(arr)


staging = _ThreadStaging()


def to_i32_device(tokens) -> torch.Tensor:
    if isinstance(tokens, torch.Tensor):
        if tokens.dtype == torch.int32 and tokens.is_cuda:
            return tokens
        return tokens.to(device=device(), dtype=torch.int32)
    return staging.to_device(np.asarray(tokens, dtype=np.int32))


def as_device_f32(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device())


def as_device_f64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device())


class UniformStream:
    """Uniforms of one numpy PCG64 Generator, in draw order, on the device.

    Kernels consume them through a device cursor (one per sampling event and
    one per verification, speculation.py:9-12).  The host refills by
    compacting [cursor, drawn) and appending a fresh block whenever fewer
    than `margin` remain.  `sync_rng()` rewinds the Generator to its state
    at creation and re-draws exactly the consumed count, so callers that
    keep using the Generator see the reference's stream position.
    """

    def __init__(self, rng: np.random.Generator, block: int = 4096, keep_state: bool = False):
        self.rng = rng
        self.block = block
        self.state0 = rng.bit_generator.state if keep_state else None
        self.consumed_before = 0          # uniforms consumed before the current buffer
        self.buf = staging.to_device(rng.random(block))
        self.drawn = block                # in the current buffer
        self.cursor = torch.zeros(1, dtype=torch.int32, device=device())
        self.host_cursor = 0

    def ensure(self, margin: int, host_cursor: int) -> None:
        """Call with the cursor value read back at the last sync."""
        self.host_cursor = host_cursor
        if self.drawn - host_cursor >= margin:
            return
        rest = self.buf[host_cursor:self.drawn]
        fresh = staging.to_device(self.rng.random(self.block))
        self.consumed_before += host_cursor
        self.buf = torch.cat([rest, fresh])
        self.drawn = self.buf.numel()
        self.cursor.zero_()
        self.host_cursor = 0

    def consumed(self, host_cursor: int) -> int:
        return self.consumed_before + host_cursor

    def sync_rng(self, host_cursor: int) -> None:
        if self.state0 is None:
            return
        self.rng.bit_generator.state = self.state0
        n = self.consumed(host_cursor)
        if n:
            self.rng.random(n)


class Pinned:
    """Small pinned host buffer for per-round readbacks."""

    def __init__(self, n: int, dtype=torch.int32):
        self.t = torch.empty(n, dtype=dtype, pin_memory=True)
