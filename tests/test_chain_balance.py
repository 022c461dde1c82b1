"""CPU: the host-balanced chain work split (stack.balanced_work) is a valid assignment -- every (K-chunk,
first row tile) item of every stage exactly once, the rest of the grid idle -- and it lowers the units a
CTA carries across a decoder layer's prefix-input stages (qkv -> o, gate_up -> down)."""

import numpy as np

from paper_2603_27914_b200.stack import balanced_work

LLAMA2_7B = [(12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008)]


def carried(tab, shapes, grid):
    """Per stage: the max over CTAs of the units carried since the last stage with a full-output input."""
    load = np.zeros(grid)
    out = []
    for s, (rows, cols) in enumerate(shapes):
        nb, rt = cols // 256, -(-rows // 16)
        nch = -(-nb // 16)
        gc = grid // nch
        if not (s > 0 and cols < shapes[s - 1][0]):
            load[:] = 0
        for c in range(grid):
            v = tab[s, c]
            if v >= 0:
                ch, r0 = divmod(int(v), gc)
                n = (rt - 1 - r0) // gc + 1 if r0 < rt else 0
                load[c] += n * min(16, nb - 16 * ch) / 16
        out.append(load.max())
    return out


def test_balanced_work_is_a_permutation():
    shapes = LLAMA2_7B * 3 + [(700, 512), (512, 256), (70000, 512)]
    for grid in (148, 132, 17):
        tab = balanced_work(shapes, grid)
        for s, (rows, cols) in enumerate(shapes):
            nch = -(-(cols // 256) // 16)
            gc = grid // nch
            got = sorted(int(v) for v in tab[s] if v >= 0)
            assert got == list(range(nch * gc)), (grid, s)
            assert (tab[s] < 0).sum() == grid - nch * gc


def test_balanced_work_lowers_carried_units():
    shapes = LLAMA2_7B * 4
    grid = 148
    tab = balanced_work(shapes, grid)
    rr = np.full_like(tab, -1)
    for s, (rows, cols) in enumerate(shapes):  # the kernel's default split
        nch = -(-(cols // 256) // 16)
        gc = grid // nch
        for c in range(grid):
            if c // nch < gc:
                rr[s, c] = (c % nch) * gc + (c // nch + 7 * s) % gc
    b, d = carried(tab, shapes, grid), carried(rr, shapes, grid)
    assert b[1] == 7 and d[1] == 8          # qkv + o
    assert b[3] == 15 and d[3] >= 15        # gate_up + down
    assert all(x <= y for x, y in zip(b, d))
