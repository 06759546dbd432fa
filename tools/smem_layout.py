"""Shared-memory bank-conflict model of the pencil kernel (dg_cell.cuh) and a layout search.

    python tools/smem_layout.py N [--search] [--tpc T --p P --c C]

Enumerates the kernel's shared-memory accesses per phase (volume arrays A0/A1 along x-, y- and
z-pencils, the neighbour-trace arrays NT: normal-first writes, tangential stages, the roles'
per-point reads) for the launch configuration of Cfg<N> (or the one given), and counts 8-byte
wavefronts with the half-warp model (lanes 0-15 and 16-31 are separate 128-byte phases; in a
phase, distinct 8-byte words with the same index mod 16 serialise). Prints the wavefronts per
cell against the conflict-free minimum for the layout in the source (generic padded linear Lay /
FLay, or the n = 4 / n = 8 swizzles) and, with --search, the best rotation layout
    at(x, y, z)      = ((x + a z + a2 y) mod N) + SY ((y + b z) mod N) + SZ z
    at(arr, i1, i2)  = ARR arr + ((i1 + c arr) mod N) + RS ((i2 + d arr) mod N)
over small parameter ranges. A development aid; the kernel's layouts are what ships.
"""
import argparse
import itertools

CFG = {2: (8, 1, 16), 3: (16, 1, 8), 4: (16, 1, 4), 5: (32, 1, 1), 6: (36, 1, 4), 7: (64, 1, 1), 8: (64, 1, 1),
       9: (96, 1, 1), 10: (64, 2, 1), 11: (128, 1, 1)}
GEN_LAY = {2: (2, 5, 9), 3: (3, 9, 27), 5: (5, 25, 125), 6: (9, 54, 321), 7: (7, 55, 379),
           9: (9, 89, 793), 10: (10, 106, 1054), 11: (11, 123, 1351)}
GEN_FLAY = {5: (5, 25), 6: (6, 41), 7: (7, 56), 9: (9, 81), 10: (10, 101), 11: (11, 121)}


def lay_source(n):
    if n == 4:
        return (lambda x, y, z: (x ^ z) + 4 * (y ^ z) + 16 * z), 64
    if n == 8:
        return (lambda x, y, z: (x ^ ((y >> 1) | ((z & 1) << 2))) + 8 * (y ^ (z & 1)) + 64 * z), 512
    sy, sz, slot = GEN_LAY[n]
    return (lambda x, y, z: x + sy * y + sz * z), slot


def flay_source(n):
    if n == 4:
        return (lambda a, i1, i2: 16 * a + (i1 ^ (a & 3)) + 4 * (i2 ^ (a & 3))), 12 * 16
    if n == 8:
        return (lambda a, i1, i2: 64 * a + 8 * (i2 ^ (a & 1)) + (i1 ^ ((i2 >> 1) | ((a & 1) << 2)))), 12 * 64
    rs, arr = GEN_FLAY.get(n, (n + 1, n * (n + 1) + 1))
    return (lambda a, i1, i2: a * arr + i1 + rs * i2), 12 * arr


def accesses(n, tpc, p, c, lay, lslot, flay, fslot, pw=None, tw=None):
    """Yield, per warp instruction, the list of (lane, word address) of the active lanes.
    pw: width of the pencil grid (pencil pc = a + pw b; lanes with a or b >= n idle), tw: lines per
    face array in the tangential-stage lane mapping (both n by default, as in the kernel)."""
    pw = pw or n
    tw = tw or n
    per_cell = 2 * lslot + fslot
    threads = c * tpc
    warps = (threads + 31) // 32
    nn = n * n

    def lanes_info(w):
        out = []
        for l in range(32):
            tid = 32 * w + l
            if tid >= threads:
                continue
            slot, lane = divmod(tid, tpc)
            out.append((l, slot, lane))
        return out

    def pencil_acc(w, base_of, coords):
        # one instruction per (pencil slot k, element e)
        info = lanes_info(w)
        for k in range(p):
            for e in range(n):
                acc = []
                for l, slot, lane in info:
                    pc = lane + k * tpc
                    pa, pb = pc % pw, pc // pw
                    if pa >= n or pb >= n:
                        continue
                    acc.append((l, slot * per_cell + base_of + lay(*coords(e, pa, pb))))
                yield acc

    def face_point_acc(w, arr):
        info = lanes_info(w)
        for k in range(p):
            acc = []
            for l, slot, lane in info:
                pc = lane + k * tpc
                pa, pb = pc % pw, pc // pw
                if pa >= n or pb >= n:
                    continue
                acc.append((l, slot * per_cell + 2 * lslot + flay(arr, pa, pb)))
            yield acc

    def tangential_acc(w, q, dim):
        info = lanes_info(w)
        rounds = (4 * tw + tpc - 1) // tpc
        for rr in range(rounds):
            for e in range(n):
                acc = []
                for l, slot, lane in info:
                    tk = lane + rr * tpc
                    if tk >= 4 * tw:
                        continue
                    arr, line = 4 * q + tk // tw, tk % tw
                    if line >= n:
                        continue
                    a = flay(arr, e, line) if dim == 0 else flay(arr, line, e)
                    acc.append((l, slot * per_cell + 2 * lslot + a))
                yield acc   # read
                yield acc   # write

    X = lambda e, a, b: (e, a, b)
    Y = lambda e, a, b: (a, e, b)
    Z = lambda e, a, b: (a, b, e)
    for w in range(warps):
        A0, A1 = 0, lslot
        seq = []
        # phase 1: x-stage writes A0, normal-first writes of the x-neighbour traces
        seq += list(pencil_acc(w, A0, X))
        for arr in range(4):
            seq += list(face_point_acc(w, arr))
        # phase 2
        seq += list(pencil_acc(w, A0, Y)) + list(pencil_acc(w, A1, Y))
        seq += list(tangential_acc(w, 0, 0))
        for arr in range(4, 8):
            seq += list(face_point_acc(w, arr))
        # phase 3
        seq += list(pencil_acc(w, A1, Z)) + list(pencil_acc(w, A0, Z))
        seq += list(tangential_acc(w, 1, 0)) + list(tangential_acc(w, 0, 1))
        for arr in range(8, 12):
            seq += list(face_point_acc(w, arr))
        # phase 4: x role
        seq += list(pencil_acc(w, A0, X))
        for arr in range(4):
            seq += list(face_point_acc(w, arr))
        seq += list(pencil_acc(w, A1, X))
        seq += list(tangential_acc(w, 2, 0)) + list(tangential_acc(w, 1, 1))
        # phase 5: y role
        seq += list(pencil_acc(w, A0, Y))
        for arr in range(4, 8):
            seq += list(face_point_acc(w, arr))
        seq += list(pencil_acc(w, A1, Y)) + list(pencil_acc(w, A1, Y))
        seq += list(tangential_acc(w, 2, 1))
        # phase 6: z role
        seq += list(pencil_acc(w, A0, Z))
        for arr in range(8, 12):
            seq += list(face_point_acc(w, arr))
        seq += list(pencil_acc(w, A1, Z)) + list(pencil_acc(w, A0, Z))
        # phases 7, 8
        seq += list(pencil_acc(w, A0, Y)) + list(pencil_acc(w, A0, Y)) + list(pencil_acc(w, A0, X))
        for acc in seq:
            yield acc


def wavefronts(acc):
    tot, ideal = 0, 0
    for half in (0, 1):
        words = {a for l, a in acc if (l >= 16) == bool(half)}
        if not words:
            continue
        ideal += 1
        cnt = {}
        for a in words:
            cnt[a % 16] = cnt.get(a % 16, 0) + 1
        tot += max(cnt.values())
    return tot, ideal


def evaluate(n, tpc, p, c, lay, lslot, flay, fslot, pw=None, tw=None):
    tot = ideal = 0
    for acc in accesses(n, tpc, p, c, lay, lslot, flay, fslot, pw, tw):
        t, i = wavefronts(acc)
        tot += t
        ideal += i
    return tot, ideal


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("--search", action="store_true")
    ap.add_argument("--tpc", type=int)
    ap.add_argument("--p", type=int)
    ap.add_argument("--c", type=int)
    a = ap.parse_args()
    n = a.n
    tpc, p, c = CFG[n]
    tpc, p, c = a.tpc or tpc, a.p or p, a.c or c
    lay, lslot = lay_source(n)
    flay, fslot = flay_source(n)
    tot, ideal = evaluate(n, tpc, p, c, lay, lslot, flay, fslot)
    print("n=%d cfg=(%d,%d,%d) source layout: %d wavefronts, conflict-free %d (%.0f %% conflicts)"
          % (n, tpc, p, c, tot, ideal, 100.0 * (tot - ideal) / tot))
    if not a.search:
        return
    best = None
    # volume layout first (face layout fixed), then the face layout
    for sy, a1, a2, b in itertools.product(range(n, n + 4), range(n), range(n), range(n)):
        for szp in range(0, 9):
            sz = n * sy + szp
            lslot2 = sz * n
            lay2 = (lambda x, y, z, sy=sy, sz=sz, a1=a1, a2=a2, b=b: ((x + a1 * z + a2 * y) % n) + sy * ((y + b * z) % n) + sz * z)
            t, i = evaluate(n, tpc, p, c, lay2, lslot2, flay, fslot)
            key = (t, lslot2)
            if best is None or key < best[0]:
                best = (key, (sy, sz, a1, a2, b), i)
    (t, lslot2), (sy, sz, a1, a2, b), i = best
    print("best volume layout: SY=%d SZ=%d a=%d a2=%d b=%d slot=%d: %d wavefronts (%.0f %% conflicts)"
          % (sy, sz, a1, a2, b, lslot2, t, 100.0 * (t - i) / t))
    lay2 = (lambda x, y, z: ((x + a1 * z + a2 * y) % n) + sy * ((y + b * z) % n) + sz * z)
    bestf = None
    for rs, c1, d1 in itertools.product(range(n, n + 3), range(n), range(n)):
        for ap_ in range(0, 9):
            arr = n * rs + ap_
            fl = (lambda A, i1, i2, rs=rs, arr=arr, c1=c1, d1=d1: arr * A + ((i1 + c1 * A) % n) + rs * ((i2 + d1 * A) % n))
            t2, i2 = evaluate(n, tpc, p, c, lay2, lslot2, fl, 12 * arr)
            key = (t2, arr)
            if bestf is None or key < bestf[0]:
                bestf = (key, (rs, arr, c1, d1), i2)
    (t2, arr), (rs, arr, c1, d1), i2 = bestf
    print("best face layout: RS=%d ARR=%d c=%d d=%d: %d wavefronts (%.0f %% conflicts)"
          % (rs, arr, c1, d1, t2, 100.0 * (t2 - i2) / t2))


if __name__ == "__main__":
    main()
