"""Shared-memory wavefront model of the symmetric pass as implemented
(translate.cu consumer_pass / sym_math): identity row map (rows 2q, 2q+1 =
consecutive fibers), lanes c = 0..3 of a row load child 0's odd element 2c+1
and child 1's p-2-2c, the even pair 2c / p-1-2c (p = 9: also the centre pair),
and store m = c and m' = p-1-c; one row of each 16-byte phase stores m' in the
instruction where the other stores m (swap).  Prints, per (d, p, axis), the
modelled wavefronts with the odd rows swapped and with the even rows swapped,
against the conflict-free minimum.  LDS/STS.128: 4 phases of 8 lanes; a phase
costs the largest number of distinct 16-byte addresses sharing a bank group."""


def phase(addrs):
    g = {}
    for a in set(x for x in addrs if x is not None):
        g.setdefault(a % 8, set()).add(a)
    return max((len(v) for v in g.values()), default=0)


def rows(D, P, AX, G, f, swapped):
    H = (P - 1) // 2
    PD = P ** D
    STR = P ** (D - 1 - AX)
    C1 = (1 << (D - 1 - AX)) * PD * G
    eb = (f // STR) * STR * P + f % STR
    L = {}
    L["a0"] = [eb + min(2 * c + 1, P - 2) * STR for c in range(4)]
    L["a1"] = [C1 + eb + max(P - 2 - 2 * c, 1) * STR for c in range(4)]
    L["e0"] = [eb + min(2 * c, P - 1) * STR for c in range(4)]
    L["e1"] = [C1 + eb + max(P - 1 - 2 * c, 0) * STR for c in range(4)]
    if P == 9:
        L["c0"] = [eb + (P - 1) * STR] * 4
        L["c1"] = [C1 + eb] * 4
    m = [min(c, H) for c in range(4)]
    mp = [max(P - 1 - c, H) for c in range(4)]
    f_el = mp if swapped else m
    s_el = m if swapped else mp
    L["f0"] = [eb + f_el[c] * STR if c <= H else None for c in range(4)]
    L["f1"] = [C1 + eb + f_el[c] * STR if c <= H else None for c in range(4)]
    L["s0"] = [eb + s_el[c] * STR if c < H else None for c in range(4)]
    L["s1"] = [C1 + eb + s_el[c] * STR if c < H else None for c in range(4)]
    return L


def cost(D, P, AX, G, swap_odd):
    PF = P ** (D - 1)
    tot = mn = 0
    for f0 in range(0, PF, 8):
        for q in range(4):
            A = rows(D, P, AX, G, (f0 + 2 * q) % PF, not swap_odd)
            B = rows(D, P, AX, G, (f0 + 2 * q + 1) % PF, swap_odd)
            for k in A:
                tot += phase(A[k] + B[k])
                mn += 1
    return tot, mn


if __name__ == "__main__":
    for D, P, G in [(2, 7, 4), (2, 9, 4), (3, 7, 1), (3, 9, 1)]:
        for AX in range(D):
            (co, mn), (ce, _) = cost(D, P, AX, G, True), cost(D, P, AX, G, False)
            print(D, P, AX, "swap odd rows", co, "swap even rows", ce, "minimum", mn)
