"""Host logic of the symmetric kernels' work lists (CPU; the C library's
ncgp_debug_sym_items runs the same walks tc_prepare uploads).  For every
flavour, item length and tile count the items must cover each tile on or
above the diagonal exactly once (K(X, X) is symmetric, the transposed
products supply the rest).  For the blocked K1-sym2 the tile order inside an
item is restated from kop_sym2_kernel's Tile2 (column-major over the block's
four row tiles) and its invariants checked: every active row meets the
item's last column (the O flush), each column's transposed tiles form one
contiguous run (the D_T flush), and the item's tile count is what the
multi-GPU split balances on (sym2_item_tiles)."""

import ctypes
from collections import Counter

import pytest

from paper_2310_20285_b200 import _native

RB = 4


def items(flavour, nb, item):
    lib = _native.load()
    fn = lib.ncgp_debug_sym_items
    fn.restype = ctypes.c_int64
    fn.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]
    k = fn(flavour, nb, item, None, 0)
    assert k > 0
    buf = (ctypes.c_int32 * (3 * k))()
    assert fn(flavour, nb, item, ctypes.addressof(buf), k) == k
    return [tuple(buf[3 * i:3 * i + 3]) for i in range(k)]


def tile2(b, c0, c1, nb):
    """kop_sym2_kernel's Tile2: column-major over the block's row tiles r <= ct."""
    rlo, rend = RB * b, min(RB * b + RB, nb)
    for ct in range(c0, c1):
        for r in range(rlo, min(rend, ct + 1)):
            yield r, ct


NBS = [1, 2, 3, 4, 5, 7, 16, 21, 40, 157, 300]


@pytest.mark.parametrize("item", [16, 48, 128])
@pytest.mark.parametrize("nb", NBS)
def test_blocked_worklist_covers_upper_triangle_once(nb, item):
    tab = items(3, nb, item)
    seen = Counter()
    for b, c0, c1 in tab:
        rlo, rend = RB * b, min(RB * b + RB, nb)
        assert rlo < nb and rlo <= c0 < c1 <= nb
        tiles = list(tile2(b, c0, c1, nb))
        seen.update(tiles)
        rows = {r for r, _ in tiles}
        # every row of the block that the item touches meets its last column
        assert rows == set(range(rlo, rend)) & {r for r in range(rlo, rend) if r <= c1 - 1}
        assert all(any(r == rr and ct == c1 - 1 for rr, ct in tiles) for r in rows)
        # a column's transposed tiles (r < ct) are consecutive in the order
        for ct in range(c0, c1):
            idx = [i for i, (r, c) in enumerate(tiles) if c == ct and r < ct]
            assert idx == list(range(idx[0], idx[0] + len(idx))) if idx else True
    want = Counter({(r, c): 1 for c in range(nb) for r in range(c + 1)})
    assert seen == want


@pytest.mark.parametrize("item", [16, 128])
@pytest.mark.parametrize("nb", NBS)
def test_single_cta_worklist_covers_upper_triangle_once(nb, item):
    seen = Counter()
    for r, c0, c1 in items(1, nb, item):
        assert r <= c0 < c1 <= nb
        seen.update((r, c) for c in range(c0, c1))
    assert seen == Counter({(r, c): 1 for c in range(nb) for r in range(c + 1)})


@pytest.mark.parametrize("nb", NBS)
def test_pair_worklist_covers_each_pair_row_once(nb):
    """CTA pairs: row-tile pair a covers column tiles [2a, nb) exactly once."""
    seen = Counter()
    for a, c0, c1 in items(2, nb, 16):
        assert 2 * a <= c0 < c1 <= nb
        seen.update((a, c) for c in range(c0, c1))
    assert seen == Counter({(a, c): 1 for a in range((nb + 1) // 2) for c in range(2 * a, nb)})


def test_blocked_items_are_block_major():
    """Column blocks of L tiles in order (the L2 locality of the accumulator
    rows and column records the running CTAs share)."""
    tab = items(3, 300, 16)
    starts = [c0 // 16 for _, c0, _ in tab]
    assert starts == sorted(starts)
