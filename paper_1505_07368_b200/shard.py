"""Row-band sharding of one Mandelbrot request across ranks / devices.

SURVEY.md §8e: contiguous bands of the config-3 zoom carry up to 1.15x the
mean work, so bands of `band_rows` rows are dealt cyclically (band b goes to
rank b % world). Each band is an independent tile; no data-path collective.
"""
from __future__ import annotations

from .cafxg import MandelDesc


def cyclic_bands(height: int, world: int, rank: int, band_rows: int) -> list[tuple[int, int]]:
    """(row0, nrows) of the bands rank `rank` owns."""
    out = []
    for b, r0 in enumerate(range(0, height, band_rows)):
        if b % world == rank:
            out.append((r0, min(band_rows, height - r0)))
    return out


def band_tiles(d: MandelDesc, world: int, rank: int, band_rows: int,
               global_offsets: bool) -> list[MandelDesc]:
    """Sub-tiles of the full-width request `d` for `rank`. With
    global_offsets the counts land at their place in the full image (one
    shared host buffer); otherwise they are packed rank-locally."""
    tiles, local = [], 0
    for r0, n in cyclic_bands(d.nrows, world, rank, band_rows):
        t = MandelDesc.from_buffer_copy(d)
        t.row0 = d.row0 + r0
        t.nrows = n
        t.out_offset = d.out_offset + (r0 * d.ncols if global_offsets else local)
        local += n * d.ncols
        tiles.append(t)
    return tiles
