"""Multi-GPU sharding of the TVOLAP lanes.

Lanes (channels / sources) are independent (proj/tests/test_engine.cpp:91-102), so
one process per GPU takes a contiguous lane range and no data-path collective is needed. The
only exchange is config C3's stereo mix. Two implementations:
  * MixGroup (the product path): one kernel per rank sums the GPU's sources and stores the
    partial mix straight into every rank's gather buffer over peer memory (cudaIpc-mapped, NVLink
    P2P stores), then each rank sums the slots in rank order — the same bits on every rank
    (tvolap_mix_group_* in the C-ABI; this class only moves the 64-byte handles and runs the
    barriers with torch.distributed);
  * mix_allreduce / tvolap_mix_allreduce: the per-GPU sum + one all-reduce (NCCL; gloo on CPU).
"""
from __future__ import annotations

import ctypes
from typing import Tuple


def weak_lanes(sources_per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling (bench.py): every rank runs its own `sources_per_rank` lanes, seeded lane0 = rank * S."""
    return rank * sources_per_rank, sources_per_rank


def strong_lanes(total_sources: int, rank: int, world: int) -> Tuple[int, int]:
    """Strong scaling: split `total_sources` into contiguous, as-equal-as-possible ranges."""
    base, extra = divmod(total_sources, world)
    lane0 = rank * base + min(rank, extra)
    return lane0, base + (1 if rank < extra else 0)


def mix_allreduce(partial_mix, group=None):
    """Sum the per-rank partial mixes (ears x samples) in place across ranks."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial_mix, op=dist.ReduceOp.SUM, group=group)
    return partial_mix


def max_over_ranks(value: float, device=None) -> float:
    """Max of a timing over ranks (bench.py reports the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class MixGroup:
    """C3's cross-GPU stereo mix over peer memory (tvolap_mix_group_*): create on every rank,
    exchange the IPC handles (torch.distributed all_gather of 64 bytes per rank), open them; then
    per pass scatter() on every rank -> barrier -> gather() -> barrier. world == 1 is a plain
    device-side mix with no handles."""

    def __init__(self, device: int, ears: int, capacity: int, group=None):
        import torch
        import torch.distributed as dist

        from . import tvolap as T

        self.T, self.lib = T, T.lib()
        dist_on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if dist_on else 1
        self.rank = dist.get_rank(group) if dist_on else 0
        self.group, self.device, self.ears, self.capacity = group, device, ears, capacity
        handle = (ctypes.c_char * 64)()
        h = ctypes.c_void_p()
        self._h = None
        if self.world == 1:
            T._check(self.lib.tvolap_mix_group_create(ctypes.byref(h), device, 1, 0, ears, capacity, handle))
            self._h = h.value
            T._check(self.lib.tvolap_mix_group_open(ctypes.c_void_p(self._h), None))
            return
        # every step is agreed by all ranks (a rank that fails must not leave the others waiting):
        # status byte + 64-byte handle travel together through the group's backend
        err = self.lib.tvolap_mix_group_create(ctypes.byref(h), device, self.world, self.rank, ears, capacity, handle)
        self._h = h.value if err == 0 else None
        dev = torch.device("cuda", device) if dist.get_backend(group) == "nccl" else torch.device("cpu")
        mine = torch.tensor([1 if err == 0 else 0] + list(bytes(handle)), dtype=torch.uint8, device=dev)
        every = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(every, mine, group=group)
        rows = [bytes(t.cpu().tolist()) for t in every]
        if not all(r[0] == 1 for r in rows):
            self.close()
            raise T.CudaError("peer-memory mix: a rank could not create its gather buffer")
        err = self.lib.tvolap_mix_group_open(ctypes.c_void_p(self._h), b"".join(r[1:] for r in rows))
        ok = torch.tensor([1 if err == 0 else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if ok.item() != 1:
            self.close()
            raise T.CudaError("peer-memory mix: a rank could not map the peers' gather buffers")

    def _barrier(self, stream):
        import torch
        import torch.distributed as dist

        if stream is None:
            torch.cuda.synchronize(self.device)
        else:
            torch.cuda.ExternalStream(stream, device=self.device).synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)

    def allreduce(self, out, sources: int, samples: int, mix, stream=None):
        """mix (ears x samples, device) = the sum over every rank's `sources` lanes of out
        ((sources * ears) x >= samples, device), bit-identical on every rank."""
        T = self.T
        T._check(self.lib.tvolap_mix_scatter(ctypes.c_void_p(self._h), sources, samples,
                                             ctypes.c_void_p(out.data_ptr()), out.stride(0),
                                             ctypes.c_void_p(stream)))
        self._barrier(stream)  # every rank's partial is in every gather buffer
        T._check(self.lib.tvolap_mix_gather(ctypes.c_void_p(self._h), samples, ctypes.c_void_p(mix.data_ptr()),
                                            mix.stride(0), ctypes.c_void_p(stream)))
        self._barrier(stream)  # every rank has read the slots before the next scatter overwrites them
        return mix

    def close(self):
        if getattr(self, "_h", None):
            self.T._check(self.lib.tvolap_mix_group_destroy(ctypes.c_void_p(self._h)))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
