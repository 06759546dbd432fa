"""The shared-memory bank-conflict model (tools/smem_layout.py) on the kernel's layouts: the
n = 4 and n = 8 swizzles are conflict free for every access of the pencil kernel, every layout
is injective on its box (no two points share a word), and the model reproduces the ncu
conflict fractions it was validated against."""
import itertools
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import smem_layout as S  # noqa: E402


@pytest.mark.parametrize("n", [4, 8])
def test_swizzled_layouts_conflict_free(n):
    tpc, p, c = S.CFG[n]
    tot, ideal = S.evaluate(n, tpc, p, c, *S.lay_source(n), *S.flay_source(n))
    assert tot == ideal


@pytest.mark.parametrize("n", [4, 5, 6, 7, 8, 9, 10, 11])
def test_layouts_injective(n):
    lay, slot = S.lay_source(n)
    words = {lay(x, y, z) for x, y, z in itertools.product(range(n), repeat=3)}
    assert len(words) == n ** 3 and min(words) >= 0 and max(words) < slot
    flay, fslot = S.flay_source(n)
    fw = {flay(a, i, j) for a in range(12) for i, j in itertools.product(range(n), repeat=2)}
    assert len(fw) == 12 * n * n and min(fw) >= 0 and max(fw) < fslot


def test_model_matches_ncu_for_the_old_layouts():
    # padded linear layouts the kernel used before: ncu measured 53 % (n = 4) and 28 % (n = 6,
    # 32 threads x 2 pencils) of the shared-memory wavefronts as bank conflicts
    tot, ideal = S.evaluate(4, 16, 1, 4, lambda x, y, z: x + 4 * y + 18 * z, 73,
                            lambda a, i1, i2: 21 * a + i1 + 5 * i2, 12 * 21)
    assert 0.50 < (tot - ideal) / tot < 0.58
    tot, ideal = S.evaluate(6, 32, 2, 1, lambda x, y, z: x + 9 * y + 54 * z, 324,
                            lambda a, i1, i2: 43 * a + i1 + 7 * i2, 12 * 43)
    assert 0.22 < (tot - ideal) / tot < 0.32
