"""Plain-IEEE numpy statement of the partition-invariant reduction of the
device (csrc/gks_reduce.cuh): the specification the device reductions are
tested against bit for bit, and the proof that a partition into whole
reduction groups leaves every sum unchanged.

fold(values): position i -> lane i % 256, accumulator (i // 256) % 4 (each a
sequential sum from +0.0); lane = (a0 + a1) + (a2 + a3); lanes combined by
the warp shuffle tree (offsets 16, 8, 4, 2, 1 inside each of the 8 warps,
then 4, 2, 1 over the warp sums).  A sum over cells: segments of 768 cells
(3840 vector entries), groups of G segments (G from the global cell count),
each level the same fold.
"""

import numpy as np

SEG_CELLS = 768


def group_segments(nc_global):
    nseg = -(-nc_global // SEG_CELLS)
    g = 1
    while -(-nseg // g) > 1024:
        g *= 2
    return g


def _tree(lane):
    w = lane.reshape(8, 32).copy()
    for o in (16, 8, 4, 2, 1):
        w[:, :o] = w[:, :o] + w[:, o:2 * o]
    v = w[:, 0].copy()
    for o in (4, 2, 1):
        v[:o] = v[:o] + v[o:2 * o]
    return float(v[0])


def fold(values):
    values = np.asarray(values, dtype=np.float64)
    acc = np.zeros((4, 256))
    for k in range(-(-len(values) // 256)):
        seg = values[k * 256:(k + 1) * 256]
        acc[k % 4, :len(seg)] = acc[k % 4, :len(seg)] + seg
    lane = (acc[0] + acc[1]) + (acc[2] + acc[3])
    return _tree(lane)


def cell_sum(values, per_cell, nc_global=None, cell_first=0):
    """Group partials of `values` (per_cell entries per cell, the rank's
    cells starting at canonical cell `cell_first`) -> dict group -> partial."""
    nc = len(values) // per_cell
    ncg = nc if nc_global is None else nc_global
    g = group_segments(ncg)
    sv = SEG_CELLS * per_cell
    nseg = -(-nc // SEG_CELLS)
    segp = [fold(values[s * sv:(s + 1) * sv]) for s in range(nseg)]
    g0 = cell_first // (SEG_CELLS * g)
    return {g0 + k: fold(segp[k * g:(k + 1) * g]) for k in range(-(-nseg // g))}


def total(groups, nc_global):
    g = group_segments(nc_global)
    ng = -(-(-(-nc_global // SEG_CELLS)) // g)
    return fold([groups.get(k, 0.0) for k in range(ng)])


def dot(x, y, nc_global=None):
    """Device GMRES dot of two (nc, 5) vectors on one rank."""
    p = (np.asarray(x, np.float64) * np.asarray(y, np.float64)).ravel()
    ncg = len(p) // 5 if nc_global is None else nc_global
    return total(cell_sum(p, 5, ncg), ncg)
