"""Multi-GPU sharding of the BP image (H7): one process per GPU, torch.distributed.

Two decompositions of the same sum P(p) = sum_m sum_n (...)  (Alg. 2 L12):
  * pixel rows  -- rank r owns grid rows [row0, row0 + nrow); every rank range-compresses
    all chirps (cheap, HBM-bound) and back-projects its rows; the image is assembled with
    one all_gather_into_tensor over NVLink (rows are contiguous in the row-major image).
  * chirps      -- rank r owns chirps [c0, c0 + nc); it range-compresses only those and
    back-projects ALL pixels into a partial image; one reduce(SUM) to the root adds the
    partial images (complex addition is component-wise on the float32 view).
  * pixel rows, gather fused (NEXT-4) -- ``FusedRowGather``: every rank's full image lives in
    symmetric memory; the BP epilogue stores each finished tile into all ranks' images over
    NVLink (P2P stores, or one multimem.st to the NVSwitch multicast address), so the gather
    overlaps the compute and no collective runs afterwards (one symmetric-memory barrier).
The compute calls go through libsar (``sar.Plan``); the other helpers only partition and
move bytes, so they also run with the gloo backend on CPU tensors in the tests.
"""
from __future__ import annotations


def row_partition(ny: int, world: int, rank: int):
    """Contiguous, balanced row blocks; equal sizes when world divides ny (all_gather
    needs equal chunks, so callers with ragged splits pad to ceil(ny/world))."""
    base, rem = divmod(ny, world)
    row0 = rank * base + min(rank, rem)
    return row0, base + (1 if rank < rem else 0)


def tile_partition(n_tiles: int, world: int, rank: int):
    """Contiguous, balanced (+-1 tile) blocks of absolute BP tiles (tile = ty * tiles_x + tx):
    SURVEY 8(e) "rank r owns a contiguous block of tiles"; with the per-tile anchors every
    pixel is computed exactly as in the unsharded image."""
    return row_partition(n_tiles, world, rank)


def tile_row_partition(tiles_y: int, tile_y: int, ny: int, world: int, rank: int):
    """Row blocks made of whole tile rows (balanced +-1 tile row), as (row0, nrow): the row
    shards of the NCCL all-gather leg, each a contiguous block of tiles."""
    t0, nt = row_partition(tiles_y, world, rank)
    row0 = min(ny, t0 * tile_y)
    return row0, min(ny, (t0 + nt) * tile_y) - row0


def weighted_partition(weights, world: int, rank: int):
    """Contiguous blocks of items with about equal total weight, as (first, count): block r ends
    at the item boundary nearest to (r + 1)/world of the total, every block keeps at least one item
    when there are at least ``world`` items.  With equal weights it is ``row_partition``'s split."""
    import bisect

    n = len(weights)
    cum = [0.0]
    for w in weights:
        cum.append(cum[-1] + max(float(w), 0.0))
    if cum[-1] <= 0.0 or n < world:
        return row_partition(n, world, rank)
    cuts = [0]
    for k in range(1, world):
        target = cum[-1] * k / world
        i = bisect.bisect_left(cum, target)
        if i > n or (i > 0 and target - cum[i - 1] <= cum[i] - target):
            i -= 1
        cuts.append(min(max(i, cuts[-1] + 1), n - (world - k)))
    cuts.append(n)
    return cuts[rank], cuts[rank + 1] - cuts[rank]


def rebalance(blocks, times, world: int, rank: int):
    """Measured load balance: re-cut contiguous blocks (``blocks`` = every rank's (first, count) over
    the same item sequence, ``times`` = every rank's measured time for its block) so that each rank
    gets an equal share of the measured cost, the cost spread uniformly over each measured block.
    Used by ``bench.py`` between warm-up steps (tile costs depend on the geometry: near-field tiles,
    derived-leg series terms), converging in a couple of iterations."""
    w = []
    for (_, n), t in sorted(zip(blocks, times)):
        w += [max(float(t), 0.0) / n] * n if n > 0 else []
    return weighted_partition(w, world, rank)


def chirp_partition(n_chirps: int, world: int, rank: int):
    return row_partition(n_chirps, world, rank)


def gather_rows(local, ny: int, group=None, parts=None):
    """Assemble the full [ny][nx] complex image from per-rank row blocks.

    ``parts`` lists every rank's (row0, nrow) (default: ``row_partition``).  Uses
    all_gather_into_tensor on the float32 view when blocks are equal, else pads every block to
    the largest block and trims.  Works for NCCL (CUDA tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    nx = local.shape[1]
    parts = parts or [row_partition(ny, world, r) for r in range(world)]
    per = max(n for _, n in parts)
    if local.shape[0] != per:
        pad = torch.zeros((per, nx), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        local = pad
    full = torch.empty((per * world, nx), dtype=local.dtype, device=local.device)
    src = torch.view_as_real(local).reshape(-1)
    dst = torch.view_as_real(full).reshape(-1)
    if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(dst, src, group=group)
    else:
        dist.all_gather(list(dst.chunk(world)), src, group=group)   # chunks are views of dst
    if all(n == per for _, n in parts):
        return full
    # drop the padding rows of every ragged block
    return torch.cat([full[r * per: r * per + n] for r, (_, n) in enumerate(parts)])


def reduce_partials(partial, dst: int = 0, group=None):
    """Sum per-rank partial images (chirp sharding) into rank ``dst`` (in place there)."""
    import torch
    import torch.distributed as dist

    dist.reduce(torch.view_as_real(partial).reshape(-1), dst=dst, op=dist.ReduceOp.SUM, group=group)
    return partial


class FusedRowGather:
    """Full [ny][nx] complex64 image in symmetric memory on every rank (torch
    ``_symmetric_memory``) + the device addresses the BP scatter epilogue writes to.

    ``ptrs`` are the P2P-mapped buffers of all ranks (``multicast=False``) or the single
    multicast address (``multicast=True``, when the NVSwitch supports it and
    ``prefer_multicast``).  ``root_ptrs`` addresses rank ``root``'s buffer only (the fused
    chirp-shard reduction).  After the scatter launch, ``barrier()`` orders every rank's
    stores before any rank reads ``image``."""

    def __init__(self, ny: int, nx: int, device, group=None, prefer_multicast: bool = True):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        group = group or dist.group.WORLD
        self.world = dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("the scatter epilogue addresses at most 8 ranks")
        self.buf = symm_mem.empty((ny, 2 * nx), dtype=torch.float32, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, group.group_name)
        self.image = torch.view_as_complex(self.buf.view(ny, nx, 2))
        self.multicast = bool(prefer_multicast and self.hdl.multicast_ptr)   # 0 without NVLS multicast
        self.ptrs = [int(self.hdl.multicast_ptr)] if self.multicast else [int(p) for p in self.hdl.buffer_ptrs]

    def root_ptrs(self, root: int = 0):
        return [int(self.hdl.buffer_ptrs[root])]

    def publish_ptrs(self, rank: int):
        """The P2P buffers with the calling rank's own first (``SAR_SCATTER_PUBLISH``: compute into
        the own image, then copy the finished tiles to the peers)."""
        ptrs = [int(p) for p in self.hdl.buffer_ptrs]
        return [ptrs[rank]] + ptrs[:rank] + ptrs[rank + 1:]

    def barrier(self, channel: int = 0):
        self.hdl.barrier(channel=channel)
