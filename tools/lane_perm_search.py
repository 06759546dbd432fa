"""Shared-memory layout + lane-to-pencil permutation search for the fast kernel's volume arrays
(development aid; the bank-conflict model of tools/smem_layout.py, restricted to the pencil
accesses, per role).

Per role q (x-, y-, z-pencils) a warp instruction touches, for fixed element e, the addresses
A_q(e, pencil(lane)) of its lanes; the 8-byte words of a 16-lane phase conflict when equal mod 16.
The element only shifts every address of the instruction by the same constant, so a phase is
conflict free iff its lanes' pencil keys  key_x = SY a + SZ b,  key_y = a + SZ b,  key_z = a + SY b
(mod 16, plus the cell's base for several cells per CTA) are distinct. The lane -> pencil map is
free per role (each phase only needs every pencil covered once), so for each padded linear layout
(SY, SZ) the search anneals one permutation per role, and reports the best layout.

    python tools/lane_perm_search.py N [--out file.json]
"""
import argparse
import json
import random

CFG = {5: (32, 1, 1), 6: (36, 1, 4), 7: (64, 1, 1), 9: (48, 2, 2), 10: (64, 2, 1), 11: (128, 1, 1)}
FARR = {5: 25, 6: 41, 7: 56, 9: 81, 10: 101, 11: 121}


def slot_size(N, SY, SZ):
    return SZ * (N - 1) + SY * (N - 1) + N


def key(N, SY, SZ, q, pc):
    a, b = pc % N, pc // N
    return (SY * a + SZ * b) if q == 0 else ((a + SZ * b) if q == 1 else (a + SY * b))


def groups(N):
    TPC, P, C = CFG[N]
    n = TPC * C
    G = []
    for k in range(P):
        for w0 in range(0, ((n + 31) // 32) * 32, 32):
            for h in (0, 16):
                g = [(tid - (tid // TPC) * TPC + k * TPC, tid // TPC) for tid in range(w0 + h, w0 + h + 16) if tid < n]
                if g:
                    G.append(g)
    return G


def cost(N, SY, SZ, q, perm, G, percell):
    tot = 0
    for g in G:
        cnt = {}
        for idx, slot in g:
            pc = perm[idx] if idx < len(perm) else None
            if pc is None:
                continue
            bk = (slot * percell + key(N, SY, SZ, q, pc)) % 16
            cnt[bk] = cnt.get(bk, 0) + 1
        if cnt:
            tot += max(cnt.values())
    return tot


def anneal(N, SY, SZ, q, G, percell, iters, seed):
    TPC, P, C = CFG[N]
    ns = TPC * P
    rnd = random.Random(seed)
    perm = list(range(N * N)) + [None] * (ns - N * N)
    cur = best = cost(N, SY, SZ, q, perm, G, percell)
    bestp = perm[:]
    T = 1.0
    for _ in range(iters):
        i, j = rnd.randrange(ns), rnd.randrange(ns)
        if i == j:
            continue
        perm[i], perm[j] = perm[j], perm[i]
        c = cost(N, SY, SZ, q, perm, G, percell)
        if c <= cur or rnd.random() < 2.718 ** (-(c - cur) / max(T, 1e-3)):
            cur = c
            if c < best:
                best, bestp = c, perm[:]
        else:
            perm[i], perm[j] = perm[j], perm[i]
        T *= 0.9995
    return best, bestp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("N", type=int)
    ap.add_argument("--iters", type=int, default=4000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    N = a.N
    G = groups(N)
    ideal = sum(1 for g in G if any(idx < N * N for idx, _ in g))
    best = None
    for SY in range(N, N + 4):
        for SZ in range(SY * (N - 1) + N, SY * (N - 1) + N + 18):
            percell = 2 * slot_size(N, SY, SZ) + 12 * FARR[N]
            tot, perms = 0, []
            for q in range(3):
                c, p = anneal(N, SY, SZ, q, G, percell, a.iters, 7 * q + 1)
                tot += c
                perms.append(p)
            if best is None or tot < best[0] or (tot == best[0] and slot_size(N, SY, SZ) < slot_size(N, best[1], best[2])):
                best = (tot, SY, SZ, perms)
                print("N=%d SY=%d SZ=%d cost %d (ideal %d)" % (N, SY, SZ, tot, 3 * ideal), flush=True)
    tot, SY, SZ, perms = best
    res = {"N": N, "SY": SY, "SZ": SZ, "cost": tot, "ideal": 3 * ideal,
           "perm": [[-1 if v is None else v for v in p] for p in perms]}
    if a.out:
        json.dump(res, open(a.out, "w"))
    print(json.dumps({k: res[k] for k in ("N", "SY", "SZ", "cost", "ideal")}))


if __name__ == "__main__":
    main()
