"""Search the row -> fiber map of the DMMA super-tile (8 fibers, rows r = lane/4)
that minimises shared-memory wavefronts of one axis pass (A-fragment loads,
delta-column loads, in-place stores), per (d, p, axis).  Model: LDS/STS.128,
a warp in 4 phases of 8 lanes (rows 2q, 2q+1 x lane%4); a phase costs the
largest number of distinct 16-byte addresses that share a bank group
(address mod 8 in 16-byte units).  Averaged over the super-tile's start fiber."""
import itertools
import sys


def shape(P, tail_dmma9=True):
    H = (P - 1) // 2
    K = 2 * H
    NK = (K + 3) // 4
    TAIL = (P % 4 == 1) and not (tail_dmma9 and P == 9)
    NM = P - 1 if TAIL else P
    NT = (2 * NM + 7) // 8
    return H, K, NK, NM, NT, TAIL


def cost(D, P, AX, rfib):
    H, K, NK, NM, NT, TAIL = shape(P)
    PD = P ** D
    STR = P ** (D - 1 - AX)
    SH = D - 1 - AX
    PF = PD // P
    C1 = (1 << SH) * PD

    def ebase(f):
        return (f // STR) * STR * P + f % STR

    total = 0
    for f0 in range(0, PF, 8):  # super-tiles aligned to tasks (tau = st*8 + rfib; tasks of PF fibers)
        fib = [(f0 + rfib[r]) % PF for r in range(8)]
        accesses = []  # list of per-lane address lists (one LDS/STS instruction each)
        for kk in range(NK):
            addr = []
            for lane in range(32):
                r, c = lane >> 2, lane & 3
                k = 4 * kk + c
                b, l = (k // H, 2 * (k % H) + 1) if k < K else (0, 0)
                addr.append(ebase(fib[r]) + l * STR + b * C1)
            accesses.append(addr)
        for n in range(NT):
            a0, a1 = [], []
            for lane in range(32):
                r, c = lane >> 2, lane & 3
                m = 4 * n + c
                a0.append(ebase(fib[r]) + min(2 * m, P - 1) * STR)
                a1.append(C1 + ebase(fib[r]) + min(max(2 * m - (P - 1), 0), P - 1) * STR)
            accesses += [a0, a1]
        for n in range(NT):  # stores of m = 4n + c (< NM) to both outputs
            s0, s1 = [], []
            for lane in range(32):
                r, c = lane >> 2, lane & 3
                m = min(4 * n + c, NM - 1)
                s0.append(ebase(fib[r]) + m * STR)
                s1.append(C1 + ebase(fib[r]) + m * STR)
            accesses += [s0, s1]
        for addr in accesses:
            for ph in range(4):
                lanes = addr[8 * ph:8 * ph + 8]
                groups = {}
                for a in set(lanes):
                    groups.setdefault(a % 8, set()).add(a)
                total += max(len(v) for v in groups.values())
    return total


def current(r):
    return (r >> 1) + 4 * (r & 1)


if __name__ == "__main__":
    cases = [(2, 5), (2, 7), (2, 9), (3, 5), (3, 7)]
    for D, P in cases:
        for AX in range(D):
            cur = [current(r) for r in range(8)]
            c0 = cost(D, P, AX, cur)
            best, bp = c0, cur
            for perm in itertools.permutations(range(8)):
                if perm[0] != 0:
                    continue  # rotations equivalent enough; fix row 0 -> fiber 0
                cc = cost(D, P, AX, perm)
                if cc < best:
                    best, bp = cc, list(perm)
            print(D, P, AX, "current", c0, "best", best, bp, flush=True)
