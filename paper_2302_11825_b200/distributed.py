"""Multi-GPU sharding of the BVC round.

* cache: rank r builds samples [r N / W, (r + 1) N / W); the walks' RNG is keyed by
  the GLOBAL sample index, so the union of shards equals the single-GPU cache
  bitwise (tests/test_gpu_cache.py::test_shard_union_equals_full_cache);
* exchange: one all-gather of the packed 48-byte samples (NCCL over NVLink on the
  GPU box; gloo in the CPU tests);
* gather: query points are split into contiguous ranges; no reduction is needed
  because every point is owned by exactly one rank.

torch.distributed is plumbing here: the collective moves raw bytes of the
library's device buffers, wrapped without copies through __cuda_array_interface__.
"""
from __future__ import annotations

import ctypes as C

SAMPLE_BYTES = 48  # struct CacheSample (csrc/internal.h)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [begin, end) of n units for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * n // world, (rank + 1) * n // world


def shard_sizes(n: int, world: int) -> list[int]:
    return [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]


class _DeviceBytes:
    """Zero-copy view of a device buffer for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes // 4,), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3}


def allgather_bytes(dist, torch, local, sizes_bytes):
    """All-gather variable-size int32 shards (padded to the largest) and concatenate."""
    words = max(sizes_bytes) // 4
    if all(s == sizes_bytes[0] for s in sizes_bytes) and local.numel() == words:  # equal shards: one buffer
        out = torch.empty(words * len(sizes_bytes), dtype=torch.int32, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    buf = torch.zeros(words, dtype=torch.int32, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in sizes_bytes]
    dist.all_gather(parts, buf)
    return torch.cat([p[: s // 4] for p, s in zip(parts, sizes_bytes)])


def generate_and_allgather(B, dist, torch, scene, problem, region, cfg, seed, rnd, rank, world, stats=None,
                           points=None, gradients=False):
    """The rank's shard of the cache, all-gathered; with `points`, the rank's fallback-band
    walks run during the shard's walks (bvc_generate_boundary_cache_shard_fallback)."""
    N = max(1, cfg.nBoundary)
    s0, s1 = shard_range(N, rank, world)
    if points is not None:
        shard = B.generate_boundary_cache_with_fallback(scene, problem, region, cfg, seed, rnd, s0, s1, points,
                                                        gradients, stats=stats)
    else:
        shard = B.generate_boundary_cache(scene, problem, region, cfg, seed, rnd, begin=s0, end=s1, stats=stats)
    ptr, nbytes = shard.packed()
    local = torch.as_tensor(_DeviceBytes(ptr, nbytes), device="cuda") if nbytes else \
        torch.empty(0, dtype=torch.int32, device="cuda")
    full = allgather_bytes(dist, torch, local, [s * SAMPLE_BYTES for s in shard_sizes(N, world)])
    torch.cuda.synchronize()
    h = C.c_void_p()
    B.api._check(B.lib().bvc_boundary_cache_from_packed(C.c_void_p(full.data_ptr()), N, shard.dim, 0,
                                                        C.c_double(0.0), C.byref(h)))
    # the library copies from `full` on its own stream; finish before torch may recycle it
    B.synchronize()
    cache = B.BoundaryCache(h)
    if cfg.voronoi:  # the weights need the whole round's samples
        cache.assign_voronoi(region)
    return cache


# --- the library's own communicator (bvc_comm; the sharded round runs in C++) ---------

def library_comm(B, dist, rank: int, world: int):
    """An NCCL bvc_comm over the torch.distributed job: rank 0's ncclUniqueId reaches
    the other ranks through torch.distributed (bootstrap only; the round's all-gather
    is the library's own ncclAllGather on its stream)."""
    box = [B.comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(box, src=0)
    return B.Communicator.nccl(box[0], world, rank)


def host_staged_comm(B, dist, torch, rank: int, world: int):
    """A bvc_comm whose all-gather is host-staged over a CPU (gloo) process group: the
    rank's device shard is copied to the host, all-gathered, and copied back into the
    library's receive buffer. For tests and hosts without NCCL between the ranks (e.g.
    several ranks sharing one GPU, where NCCL refuses duplicate devices)."""

    def fn(send_ptr, recv_ptr, nbytes):
        words = nbytes // 4
        dev = torch.device("cuda", torch.cuda.current_device())
        send = torch.as_tensor(_DeviceBytes(send_ptr, nbytes), device=dev) if nbytes else \
            torch.empty(0, dtype=torch.int32, device=dev)
        host = send.cpu()
        parts = [torch.empty(words, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, host)
        recv = torch.as_tensor(_DeviceBytes(recv_ptr, nbytes * world), device=dev)
        recv.copy_(torch.cat(parts).to(dev))
        torch.cuda.synchronize()

    return B.Communicator.from_allgather(world, rank, fn)
