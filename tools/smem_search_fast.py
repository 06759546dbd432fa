"""Vectorised layout search on top of tools/smem_layout.py's access model (development aid).

    python tools/smem_search_fast.py N [--tpc T --p P --c C]
"""
import argparse
import itertools
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import smem_layout as S  # noqa: E402


def lane_table(n, tpc, p, c):
    threads = c * tpc
    warps = (threads + 31) // 32
    rows = []   # per (warp, k): arrays lane, slot, pa, pb (active only)
    for w in range(warps):
        for k in range(p):
            L, SL, PA, PB = [], [], [], []
            for l in range(32):
                tid = 32 * w + l
                if tid >= threads:
                    continue
                slot, lane = divmod(tid, tpc)
                pc = lane + k * tpc
                if pc >= n * n:
                    continue
                L.append(l); SL.append(slot); PA.append(pc % n); PB.append(pc // n)
            if L:
                rows.append((np.array(L), np.array(SL), np.array(PA), np.array(PB)))
    return rows


def waves(lanes, addr):
    tot = 0
    for half in (0, 1):
        m = (lanes >= 16) == bool(half)
        if not m.any():
            continue
        a = np.unique(addr[m])
        tot += np.bincount(a % 16, minlength=16).max()
    return tot


# occurrences of each (array, direction) pencil access per cell in the kernel (smem_layout.accesses)
COUNTS = {("A0", "X"): 3, ("A1", "X"): 1, ("A0", "Y"): 4, ("A1", "Y"): 3, ("A0", "Z"): 3, ("A1", "Z"): 2}


def vol_cost(n, rows, lay, lslot, per_cell):
    tot = 0
    for (arr, d), cnt in COUNTS.items():
        base = 0 if arr == "A0" else lslot
        for L, SL, PA, PB in rows:
            for e in range(n):
                E = np.full_like(PA, e)
                x, y, z = {"X": (E, PA, PB), "Y": (PA, E, PB), "Z": (PA, PB, E)}[d]
                addr = SL * per_cell + base + lay(x, y, z)
                tot += cnt * waves(L, addr)
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("--tpc", type=int)
    ap.add_argument("--p", type=int)
    ap.add_argument("--c", type=int)
    a = ap.parse_args()
    n = a.n
    tpc, p, c = S.CFG[n]
    tpc, p, c = a.tpc or tpc, a.p or p, a.c or c
    rows = lane_table(n, tpc, p, c)
    lay0, lslot0 = S.lay_source(n)
    fl0, fslot0 = S.flay_source(n)
    lay0v = np.vectorize(lay0)
    base = vol_cost(n, rows, lambda x, y, z: lay0v(x, y, z), lslot0, 2 * lslot0 + fslot0)
    ideal = vol_cost(n, rows, lambda x, y, z: np.zeros_like(x) + (x + n * y + n * n * z) * 0 + np.arange(len(x)) if False else x * 0 + 0, lslot0, 0)
    print("n=%d source volume cost %d" % (n, base))
    best = None
    for sy in range(n, n + 4):
        for szp in range(0, 9):
            sz = n * sy + szp
            lslot = sz * n
            per_cell = 2 * lslot + fslot0
            for a1, a2, b in itertools.product(range(n), range(n), range(n)):
                lay = (lambda x, y, z: ((x + a1 * z + a2 * y) % n) + sy * ((y + b * z) % n) + sz * z)
                t = vol_cost(n, rows, lay, lslot, per_cell)
                key = (t, lslot)
                if best is None or key < best[0]:
                    best = (key, (sy, sz, a1, a2, b))
        print("  sy=%d best so far %s" % (sy, best), flush=True)
    print("BEST", best)


if __name__ == "__main__":
    main()


def face_rows(n, tpc, c):
    """(lanes, slot, arr_offset_index, line) for the tangential-stage instructions and the
    per-point instructions (pencil rows)."""
    threads = c * tpc
    warps = (threads + 31) // 32
    tang = []
    rounds = (4 * n + tpc - 1) // tpc
    for w in range(warps):
        for rr in range(rounds):
            L, SL, AR, LN = [], [], [], []
            for l in range(32):
                tid = 32 * w + l
                if tid >= threads:
                    continue
                slot, lane = divmod(tid, tpc)
                tk = lane + rr * tpc
                if tk >= 4 * n:
                    continue
                L.append(l); SL.append(slot); AR.append(tk // n); LN.append(tk % n)
            if L:
                tang.append((np.array(L), np.array(SL), np.array(AR), np.array(LN)))
    return tang


def face_cost(n, rows, tang, flay, lslot, fslot):
    per_cell = 2 * lslot + fslot
    tot = 0
    # per-point accesses: 12 arrays written once (normal-first) and read once (roles): 2 each
    for arr in range(12):
        for L, SL, PA, PB in rows:
            addr = SL * per_cell + 2 * lslot + flay(np.full_like(PA, arr), PA, PB)
            tot += 2 * waves(L, addr)
    # tangential stages: for q in 0..2, dim 0 and 1, read + write per element
    for q in range(3):
        for dim in (0, 1):
            for L, SL, AR, LN in tang:
                A = 4 * q + AR
                for e in range(n):
                    E = np.full_like(LN, e)
                    a = flay(A, E, LN) if dim == 0 else flay(A, LN, E)
                    tot += 2 * waves(L, SL * per_cell + 2 * lslot + a)
    return tot


def search_face(n, tpc, p, c, lslot):
    rows = lane_table(n, tpc, p, c)
    tang = face_rows(n, tpc, c)
    fl0, fslot0 = S.flay_source(n)
    base = face_cost(n, rows, tang, np.vectorize(fl0), lslot, fslot0)
    print("n=%d source face cost %d" % (n, base))
    best = None
    for rs in range(n, n + 3):
        for ap_ in range(0, 9):
            arr = n * rs + ap_
            for c1, d1 in itertools.product(range(n), range(n)):
                fl = (lambda A, i1, i2: arr * A + ((i1 + c1 * A) % n) + rs * ((i2 + d1 * A) % n))
                t = face_cost(n, rows, tang, fl, lslot, 12 * arr)
                key = (t, arr)
                if best is None or key < best[0]:
                    best = (key, (rs, arr, c1, d1))
    print("FACE BEST", best)


def ideal_costs(n, tpc, p, c):
    rows = lane_table(n, tpc, p, c)
    tang = face_rows(n, tpc, c)
    z = lambda *args: args[0] * 0 + np.arange(len(args[0])) * 0
    # a distinct word per lane with distinct residues: conflict-free lower bound = nonempty halves
    def halves(L):
        return int((L < 16).any()) + int((L >= 16).any())
    vol = sum(cnt * n * halves(L) for cnt in COUNTS.values() for L, _, _, _ in rows)
    face = sum(2 * halves(L) for _ in range(12) for L, _, _, _ in rows) + sum(
        2 * n * halves(L) for _ in range(6) for L, _, _, _ in tang)
    return vol, face


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "all":
    pass
