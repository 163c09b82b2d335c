"""Search the C3 interior kernel's staging layout (fourier2d.cu, kF2iSlot) and check it.

A (line, matrix) run of two staged rows is 98 doubles; element s (= run element + shift sh, sh = 1
when the run starts 8 bytes off a 16-byte boundary) lives in 16-byte slot slot[sh][s >> 1].
Shared-memory accesses are served per half-warp for 8-byte and per quarter-warp for 16-byte
accesses; a phase costs one wavefront per distinct address in its busiest bank.
  * x-stage writes: lane (g, t), g < 7 writes elements g + 14 t + 7 j + 49 i + sh (j = 1: t < 3);
  * run reads: lane reads 16-byte pairs lane + sh and lane + 32 + sh (< 49).
The reads force slot = 8 * ((P - sh) // 8) + b(P) with b a permutation of 0..7 in every window of
8 pairs; the search permutes within windows until every write phase hits 16 distinct banks.

    python tools/staging_layout.py            # search (seeded) and print the tables
    python tools/staging_layout.py --check    # wavefronts of the natural and the committed layout
"""
import random
import sys

COMMITTED = [
    [5, 3, 2, 1, 6, 7, 0, 4, 14, 15, 13, 10, 11, 12, 9, 8, 19, 16, 20, 21, 17, 18, 23, 22, 28,
     25, 30, 31, 26, 24, 27, 29, 39, 34, 35, 37, 33, 36, 38, 32, 44, 40, 47, 46, 41, 42, 43, 45, 49, 48],
    [51, 7, 3, 1, 0, 2, 5, 6, 4, 8, 12, 15, 9, 11, 10, 13, 14, 23, 22, 19, 20, 16, 17, 18, 21,
     25, 28, 31, 26, 27, 24, 30, 29, 34, 37, 32, 33, 39, 36, 38, 35, 41, 46, 44, 42, 45, 40, 47, 43, 52]]


def writes(sh):
    for i in (0, 1):
        for j in (0, 1):
            yield [(4 * g + t, g + 14 * t + 7 * j + 49 * i + sh) for g in range(7) for t in range(4 if j == 0 else 3)]


def wavefronts(pairs, per_phase, key):
    tot = 0
    for ph in range(32 // per_phase):
        banks = {}
        for lane, a in pairs:
            if lane // per_phase == ph:
                banks.setdefault(key(a), set()).add(a)
        tot += max([len(v) for v in banks.values()] + [0])
    return tot


def cost(slot, sh):
    addr = lambda s: 2 * slot[s >> 1] + (s & 1)
    w = [wavefronts([(l, addr(s)) for l, s in pat], 16, lambda a: a % 16) for pat in writes(sh)]
    r1 = wavefronts([(l, 2 * slot[l + sh]) for l in range(32)], 8, lambda a: (a // 2) % 8)
    r2 = wavefronts([(l, 2 * slot[l + 32 + sh]) for l in range(32) if l + 32 < 49 - sh], 8, lambda a: (a // 2) % 8)
    return w, r1, r2


def search(sh, seed=0, iters=200000):
    rnd = random.Random(seed)
    starts = [sh + 8 * k for k in range(7)]
    b = {}
    for st in starts:
        perm = list(range(8))
        rnd.shuffle(perm)
        for l in range(8):
            b[st + l] = perm[l]
    if sh == 1:
        b[0] = b[50]          # pair 0 (element 0 of a shifted run) takes a spare slot of the last window

    def slots():
        return [(6 * 8 + b[P]) if P < sh else ((P - sh) // 8) * 8 + b[P] for P in range(50)]

    def c():
        return sum(x - 2 for x in cost(slots(), sh)[0])
    cur = c()
    for _ in range(iters):
        if cur == 0:
            break
        st = rnd.choice(starts)
        x, y = rnd.sample(range(8), 2)
        b[st + x], b[st + y] = b[st + y], b[st + x]
        if sh == 1:
            b[0] = b[50]
        new = c()
        if new <= cur or rnd.random() < 0.01:
            cur = new
        else:
            b[st + x], b[st + y] = b[st + y], b[st + x]
            if sh == 1:
                b[0] = b[50]
    return cur, slots()


if __name__ == "__main__":
    if "--check" in sys.argv:
        for name, tab in (("natural", [list(range(50))] * 2), ("committed", COMMITTED)):
            for sh in (0, 1):
                assert len(set(tab[sh])) == 50
                print(name, "sh", sh, "x-stage write wavefronts", *cost(tab[sh], sh))
    else:
        for sh in (0, 1):
            print(sh, search(sh))
