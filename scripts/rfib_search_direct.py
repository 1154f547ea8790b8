"""Row -> fiber map of the direct-form (p = 5) super-tile, per (d, axis, G),
minimising modelled shared-memory wavefronts, with the slot-major stage
(child-1 slot (1 << (d-1-axis)) * (G * p^d + pad) elements after child 0; pad =
SlotPad, 1 element).

Access model of direct_math (translate.cu): lane (r, c) loads child (c >> 1)'s
element 2 (c & 1) + 1 (A fragment), child 0's element min(2c, 4) and child 1's
element max(2c - 4, 0) (delta columns), child 1's element 4 (tail delta), and
(in-place passes) stores element c of both children plus one scalar half of
element 4.  LDS/STS.128 in 4 phases of 8 lanes (rows 2q, 2q+1); a phase costs
the largest number of distinct 16-byte addresses sharing a bank group.  For the
last (global) pass only the loads count, and consecutive fibers in rows 2q,
2q+1 fill whole sectors -- reported separately ("identity")."""
import itertools


def phase(addrs):
    g = {}
    for a in set(x for x in addrs if x is not None):
        g.setdefault(a % 8, set()).add(a)
    return max((len(v) for v in g.values()), default=0)


def cost(D, AX, G, rfib, stores=True, pad=1):
    P = 5
    PD = P ** D
    STR = P ** (D - 1 - AX)
    PF = PD // P
    C1 = (1 << (D - 1 - AX)) * (PD * G + pad)  # slot-major stage with SlotPad
    tot = 0
    for f0 in range(0, PF, 8):
        fib = [(f0 + rfib[r]) % PF for r in range(8)]
        eb = [(f // STR) * STR * P + f % STR for f in fib]
        ins = []
        ins.append([eb[l >> 2] + ((C1 if (l & 3) >> 1 else 0) + (2 * (l & 1) + 1) * STR) for l in range(32)])
        ins.append([eb[l >> 2] + min(2 * (l & 3), P - 1) * STR for l in range(32)])
        ins.append([C1 + eb[l >> 2] + max(2 * (l & 3) - (P - 1), 0) * STR for l in range(32)])
        ins.append([C1 + eb[l >> 2] + (P - 1) * STR for l in range(32)])
        if stores:
            ins.append([eb[l >> 2] + (l & 3) * STR for l in range(32)])
            ins.append([C1 + eb[l >> 2] + (l & 3) * STR for l in range(32)])
            ins.append([(C1 if (l & 3) >> 1 else 0) + eb[l >> 2] + (P - 1) * STR for l in range(32)])
        for a in ins:
            for ph in range(4):
                tot += phase(a[8 * ph:8 * ph + 8])
    return tot


if __name__ == "__main__":
    for D, G in [(3, 2), (2, 8)]:
        for AX in range(D):
            ident = list(range(8))
            best = None
            for perm in itertools.permutations(range(8)):
                if perm[0] != 0:
                    continue
                c = cost(D, AX, G, perm)
                if best is None or c < best[0]:
                    best = (c, perm)
            code = sum(v << (4 * r) for r, v in enumerate(best[1]))
            print(D, G, AX, "identity", cost(D, AX, G, ident), "identity loads-only", cost(D, AX, G, ident, False),
                  "best", best[0], list(best[1]), hex(code), flush=True)
