"""Block-range sharding across GPUs (one process per GPU).

Blocks are independent — every block is filtered with its own padding and no
data crosses tile seams (image.hpp:205-209) — so an image is partitioned into
contiguous block-row bands and a video into contiguous frame ranges, one per
rank, with no data-path collective. The only collective is the optional
gather of the u8 result to a root rank (torch.distributed: NCCL over
NVLink/NVSwitch on the GPU box, gloo in the CPU tests).

The per-shard compute is a callable so the partition/gather logic is the same
for the CUDA path (`plan.filter_image` on the rank's device) and for the CPU
oracle the tests plug in.
"""
from __future__ import annotations

from typing import Callable, Sequence


def balanced_ranges(count: int, world: int) -> list[tuple[int, int]]:
    """Split [0, count) into `world` contiguous ranges whose sizes differ by
    at most one (earlier ranks take the remainder)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(count, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((start, start + n))
        start += n
    return out


def block_row_bands(height: int, n: int, world: int) -> list[tuple[int, int]]:
    """Pixel-row bands [y0, y1) per rank, aligned to block rows of side n. The
    last band carries the image's ragged bottom edge (if any), which keeps the
    reference's edge replication (tile(), image.hpp:175-176) local to it."""
    bh = (height + n - 1) // n
    return [(min(height, a * n), min(height, b * n)) for a, b in balanced_ranges(bh, world)]


def filter_image_sharded(img, n: int, rank: int, world: int,
                         compute: Callable, gather: bool = True, group=None):
    """Filter rank's band of `img` ((h, w) array/tensor, identical on every
    rank or at least valid on the rank's band) with `compute(band) -> band`;
    with `gather`, rank 0 receives the full (h, w) result (others get None).
    Without `gather`, every rank returns only its own band."""
    h = img.shape[0]
    y0, y1 = block_row_bands(h, n, world)[rank]
    band = compute(img[y0:y1]) if y1 > y0 else img[y0:y1]
    if not gather or world == 1:
        return band
    return _gather_rows(band, h, n, rank, world, group)


def filter_frames_sharded(frames, rank: int, world: int, compute: Callable,
                          gather: bool = False, group=None):
    """Video: rank r filters frames [f0, f1) of (F, h, w) `frames` with
    `compute(frames_slice, first_frame_index) -> out_slice`."""
    f0, f1 = balanced_ranges(frames.shape[0], world)[rank]
    out = compute(frames[f0:f1], f0)
    if not gather or world == 1:
        return out
    return _gather_leading(out, frames.shape[0], rank, world, group)


def _as_tensor(x):
    import numpy as np
    import torch
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x)), True
    return x.contiguous(), False


def _gather_rows(band, h: int, n: int, rank: int, world: int, group):
    return _gather_ranges(band, [b - a for a, b in block_row_bands(h, n, world)], rank, world,
                          group)


def _gather_leading(part, total: int, rank: int, world: int, group):
    return _gather_ranges(part, [b - a for a, b in balanced_ranges(total, world)], rank, world,
                          group)


def _gather_ranges(part, sizes: Sequence[int], rank: int, world: int, group):
    """all_gather of equal-size (padded) slabs along dim 0, concatenated in rank
    order on rank 0. Equal sizes keep it a single NCCL all_gather."""
    import torch
    import torch.distributed as dist
    t, was_numpy = _as_tensor(part)
    cap = max(sizes)
    pad_shape = (cap,) + tuple(t.shape[1:])
    slab = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
    slab[: t.shape[0]] = t
    slabs = torch.empty((world * cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(slabs, slab, group=group)
    if rank != 0:
        return None
    full = torch.cat([slabs[r * cap: r * cap + sizes[r]] for r in range(world)], dim=0)
    return full.cpu().numpy() if was_numpy else full
