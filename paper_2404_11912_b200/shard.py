"""Sequence sharding of the full KV cache across the GPUs of one node
(the reference never distributes -- hierspec has no
collective -- so this is the one parallel strategy the B200 build adds).

Plan: rank r of G stores the full-cache positions [r*S, (r+1)*S) with S the
context length / G rounded up to a whole number of retrieval chunks; the
last rank also receives every position appended later (it owns
[(G-1)*S, max_seq)).  Weights, the draft lane and the retrieval lane are
replicated and deterministic, so every rank executes the same forwards;
the exchange steps run inside the native code over NCCL:

* per layer of every full-cache forward, the per-rank partial softmax
  states are all-gathered and merged in rank order (hs_forward, HsShard);
* per retrieval build, per-rank fp64 chunk scores are all-gathered (the
  replicated selection is then bit-identical to the unsharded one); each
  rank gathers the chosen chunks it stores and the per-rank slot ranges are
  exchanged with a variable-size all-gather (hs_retrieval_exchange).

The communicator is NCCL's own (hs_comm_init, non-blocking, every call
bounded by a deadline); torch.distributed only ships its unique id from rank
0 to the others.  `SequenceShards.loopback(G)` instead makes G ranks inside
one process on one GPU (one host thread and CUDA stream per rank, exchanges
by device-to-device copies with the same semantics): the G-shard session is
then checked bit for bit against the unsharded one without G GPUs.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import torch

from ._abi import HsShard, check, lib
from .runtime import ptr, stream_ptr

DT_BF16, DT_F32, DT_F64, DT_I32 = 0, 1, 2, 3
_DTYPES = {torch.bfloat16: DT_BF16, torch.float32: DT_F32, torch.float64: DT_F64, torch.int32: DT_I32}


def shard_plan(n_positions: int, world: int, chunk: int) -> List[Tuple[int, Optional[int]]]:
    """[(lo, hi)] per rank; hi is None for the last rank (it owns the tail).
    Shard length = ceil(n / world) rounded up to a multiple of `chunk`, so a
    retrieval chunk never straddles two ranks."""
    if world < 1 or chunk < 1 or n_positions < 1:
        raise ValueError("shard_plan needs world >= 1, chunk >= 1 and a non-empty context")
    per = -(-n_positions // world)
    per = -(-per // chunk) * chunk
    return [(r * per, (r + 1) * per if r < world - 1 else None) for r in range(world)]


def shard_chunk_counts(bounds, upto: int, chunk: int) -> List[int]:
    """Chunks of [0, upto) held by each rank (the last one may be partial)."""
    out = []
    for lo, hi in bounds:
        end = upto if hi is None else min(upto, hi)
        out.append(max(0, -(-(end - lo) // chunk)))
    return out


class SequenceShards:
    """This rank's place in the sequence-sharded full cache plus the NCCL
    communicator used by the native exchange steps."""

    def __init__(self, rank: int, world: int, comm: int, loopback: bool = False):
        self.rank, self.world, self._comm = rank, world, comm
        self.is_loopback = loopback
        d = HsShard()
        d.comm, d.rank, d.world = comm, rank, world
        self.desc = d
        self.ref = C.byref(d)

    @classmethod
    def init(cls, group=None) -> "SequenceShards":
        """Collective over a torch.distributed group (any backend): rank 0
        makes the NCCL id, every rank joins the communicator."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        n = lib.hs_comm_id_bytes()
        payload = [None]
        if rank == 0:
            buf = (C.c_char * n)()
            check(lib.hs_comm_unique_id(buf))
            payload = [bytes(buf)]
        dist.broadcast_object_list(payload, src=0, group=group)
        return cls._join(payload[0], world, rank)

    @classmethod
    def single(cls) -> "SequenceShards":
        """A one-rank communicator: the sharded code path on one GPU."""
        n = lib.hs_comm_id_bytes()
        buf = (C.c_char * n)()
        check(lib.hs_comm_unique_id(buf))
        return cls._join(bytes(buf), 1, 0)

    @classmethod
    def loopback(cls, world: int) -> List["SequenceShards"]:
        """G ranks in this process (hs_loopback_create): rank r's object must
        be used from one host thread with its own current CUDA stream."""
        comms = (C.c_void_p * world)()
        check(lib.hs_loopback_create(world, comms))
        return [cls(r, world, comms[r], loopback=True) for r in range(world)]

    @classmethod
    def _join(cls, uid: bytes, world: int, rank: int) -> "SequenceShards":
        comm = C.c_void_p()
        check(lib.hs_comm_init(C.byref(comm), uid, world, rank))
        return cls(rank, world, comm.value)

    def destroy(self) -> None:
        """NCCL: finalize and destroy this rank's communicator.  Loopback:
        call on any one rank after every rank is done (frees the group)."""
        if self._comm:
            check(lib.hs_loopback_destroy(self._comm) if self.is_loopback else lib.hs_comm_destroy(self._comm))
            self._comm = None

    def abort(self) -> None:
        """Release the peers of a failing rank (their collectives raise)."""
        if self._comm:
            check(lib.hs_comm_abort(self._comm))

    def check(self) -> None:
        """Raise if the communicator carries an asynchronous error (a peer
        failed or timed out)."""
        check(lib.hs_comm_check(self._comm))

    # -- plan ------------------------------------------------------------------------
    def plan(self, n_positions: int, chunk: int):
        return shard_plan(n_positions, self.world, chunk)

    # -- collectives on the current stream ----------------------------------------------
    def all_gather(self, send: torch.Tensor) -> torch.Tensor:
        """[world, *send.shape] in rank order."""
        send = send.contiguous()
        recv = torch.empty((self.world, *send.shape), dtype=send.dtype, device=send.device)
        check(lib.hs_all_gather(self._comm, ptr(send), ptr(recv), send.numel() * send.element_size(),
                                stream_ptr()))
        return recv

    def all_gather_v(self, send: torch.Tensor, counts: List[int]) -> torch.Tensor:
        """1-D concat in rank order of each rank's first counts[r] elements
        (this rank sends send[:counts[rank]])."""
        send = send.contiguous()
        es = send.element_size()
        recv = torch.empty(sum(counts), dtype=send.dtype, device=send.device)
        nb = (C.c_size_t * self.world)(*[c * es for c in counts])
        check(lib.hs_all_gather_v(self._comm, self.rank, self.world, ptr(send), ptr(recv), nb, stream_ptr()))
        return recv

    def all_reduce_sum_(self, buf: torch.Tensor) -> torch.Tensor:
        if not buf.is_contiguous():
            raise ValueError("all_reduce_sum_ needs a contiguous tensor")
        check(lib.hs_all_reduce_sum(self._comm, ptr(buf), buf.numel(), _DTYPES[buf.dtype], stream_ptr()))
        return buf
