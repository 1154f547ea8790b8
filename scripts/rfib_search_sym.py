"""Row -> fiber map of the symmetric DMMA super-tile (8 fibers, rows r = lane/4)
minimising shared-memory wavefronts of one axis pass, per (d, p, axis, G).

Access model of consumer_pass (translate.cu, symmetric form): lane (r, c)
of a super-tile loads, for its fiber, child-0 element 2c+1 and child-1 element
p-2-2c (A fragments of the s/t GEMMs), child-0 element 2c and child-1 element
p-1-2c (delta columns; clamped to p-1 / 0 for c > H), for p = 9 also child-0
element p-1 and child-1 element 0 (centre delta), and stores outputs m = c and
m' = p-1-c into both slots (in-place passes).  LDS/STS.128: a warp in 4 phases
of 8 lanes (rows 2q, 2q+1); a phase costs the largest number of distinct
16-byte addresses sharing a bank group (address mod 8, 16-byte units).  The
child-1 slot is (1 << (d-1-ax)) * G * p^d elements after child 0 (slot-major
stage); averaged over task-aligned super-tiles of one group."""
import itertools
import sys


def cost(D, P, AX, G, rfib):
    H = (P - 1) // 2
    PD = P ** D
    STR = P ** (D - 1 - AX)
    SH = D - 1 - AX
    PF = PD // P
    C1 = (1 << SH) * PD * G

    def ebase(f):
        return (f // STR) * STR * P + f % STR

    total = 0
    for f0 in range(0, PF, 8):
        fib = [(f0 + rfib[r]) % PF for r in range(8)]
        acc = []

        def lanes(fn):
            return [fn(l >> 2, l & 3) for l in range(32)]
        acc.append(lanes(lambda r, c: ebase(fib[r]) + min(2 * c + 1, P - 2) * STR))
        acc.append(lanes(lambda r, c: C1 + ebase(fib[r]) + max(P - 2 - 2 * c, 1) * STR))
        acc.append(lanes(lambda r, c: ebase(fib[r]) + min(2 * c, P - 1) * STR))
        acc.append(lanes(lambda r, c: C1 + ebase(fib[r]) + max(P - 1 - 2 * c, 0) * STR))
        if P == 9:
            acc.append(lanes(lambda r, c: ebase(fib[r]) + (P - 1) * STR))
            acc.append(lanes(lambda r, c: C1 + ebase(fib[r])))
        for base in (0, C1):
            acc.append(lanes(lambda r, c: base + ebase(fib[r]) + min(c, H) * STR))
            acc.append(lanes(lambda r, c: base + ebase(fib[r]) + max(P - 1 - c, H) * STR))
        for addr in acc:
            for ph in range(4):
                ls = addr[8 * ph:8 * ph + 8]
                groups = {}
                for a in set(ls):
                    groups.setdefault(a % 8, set()).add(a)
                total += max(len(v) for v in groups.values())
    return total


def default(r):
    return (r >> 1) + 4 * (r & 1)


if __name__ == "__main__":
    cases = [(2, 5, 8), (2, 7, 4), (2, 9, 4), (3, 5, 2), (3, 7, 1), (3, 7, 2), (3, 9, 1)]
    for D, P, G in cases:
        for AX in range(D):
            cur = [default(r) for r in range(8)]
            c0 = cost(D, P, AX, G, cur)
            ident = cost(D, P, AX, G, list(range(8)))
            best, bp = c0, cur
            for perm in itertools.permutations(range(8)):
                if perm[0] != 0:
                    continue
                cc = cost(D, P, AX, G, perm)
                if cc < best:
                    best, bp = cc, list(perm)
            code = sum(v << (4 * r) for r, v in enumerate(bp))
            print(D, P, G, AX, "default", c0, "identity", ident, "best", best, bp, hex(code), flush=True)
