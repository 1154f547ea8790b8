"""Bank-conflict model of the symmetric pass with per-row role choices.

Rows 2q, 2q+1 of a super-tile share a 16-byte-access phase.  Besides the row
-> fiber map, the second row of a phase may (a) load its children in the
opposite order (child 1 in the instruction where the first row loads child
0), separately for the odd and the even element pairs, and (b) store its
outputs in a different order (m' before m, and/or z_1 before z_0).  The signs
these swaps introduce fold into the existing FMAs.  For each (d, p, axis, G)
this finds the row map and per-phase choices minimising the modelled
wavefronts (LDS/STS.128: a phase of 8 lanes costs the largest number of
distinct 16-byte addresses that share a bank group, address mod 8)."""
import itertools
import sys


def phase_cost(addrs):
    groups = {}
    for a in set(addrs):
        groups.setdefault(a % 8, set()).add(a)
    return max(len(v) for v in groups.values())


def instr_sets(D, P, AX, G, f):
    """per row: dict name -> list of 4 lane addresses (c = 0..3) for fiber f"""
    H = (P - 1) // 2
    PD = P ** D
    STR = P ** (D - 1 - AX)
    SH = D - 1 - AX
    C1 = (1 << SH) * PD * G
    eb = (f // STR) * STR * P + f % STR
    cs = range(4)
    d = {}
    d["a0"] = [eb + min(2 * c + 1, P - 2) * STR for c in cs]
    d["a1"] = [C1 + eb + max(P - 2 - 2 * c, 1) * STR for c in cs]
    d["e0"] = [eb + min(2 * c, P - 1) * STR for c in cs]
    d["e1"] = [C1 + eb + max(P - 1 - 2 * c, 0) * STR for c in cs]
    if P == 9:
        d["c0"] = [eb + (P - 1) * STR] * 4
        d["c1"] = [C1 + eb] * 4
    m = [min(c, H) for c in cs]
    mp = [max(P - 1 - c, H) for c in cs]
    d["s0m"] = [eb + x * STR for x in m]
    d["s0p"] = [eb + x * STR for x in mp]
    d["s1m"] = [C1 + eb + x * STR for x in m]
    d["s1p"] = [C1 + eb + x * STR for x in mp]
    return d


# instruction slots and, per option, which named access a row performs in each
LOAD_ODD = [("a0", "a1"), ("a1", "a0")]
LOAD_EVEN = [("e0", "e1"), ("e1", "e0")]
STORES = [("s0m", "s1m", "s0p", "s1p"), ("s0p", "s1p", "s0m", "s1m"), ("s1m", "s0m", "s1p", "s0p"),
          ("s1p", "s0p", "s1m", "s0m")]


def cost_pair(D, P, AX, G, fa, fb, ob):
    """cost of one phase: row A fiber fa (default roles), row B fiber fb with option ob"""
    A = instr_sets(D, P, AX, G, fa)
    B = instr_sets(D, P, AX, G, fb)
    lo, le, st = ob
    tot = 0
    for i in range(2):
        tot += phase_cost(A[LOAD_ODD[0][i]] + B[LOAD_ODD[lo][i]])
        tot += phase_cost(A[LOAD_EVEN[0][i]] + B[LOAD_EVEN[le][i]])
    for i in range(4):
        tot += phase_cost(A[STORES[0][i]] + B[STORES[st][i]])
    if P == 9:
        tot += phase_cost(A["c0"] + B["c0"]) + phase_cost(A["c1"] + B["c1"])
    return tot


OPTS = [(lo, le, st) for lo in range(2) for le in range(2) for st in range(4)]


def best_map(D, P, AX, G):
    PF = P ** (D - 1)
    starts = list(range(0, PF, 8))
    best = None
    for perm in itertools.permutations(range(8)):
        if perm[0] != 0:
            continue
        tot = 0
        choice = []
        for q in range(4):
            ra, rb = perm[2 * q], perm[2 * q + 1]
            costs = [sum(cost_pair(D, P, AX, G, (f0 + ra) % PF, (f0 + rb) % PF, o) for f0 in starts) for o in OPTS]
            k = min(range(len(OPTS)), key=lambda i: costs[i])
            tot += costs[k]
            choice.append(OPTS[k])
        if best is None or tot < best[0]:
            best = (tot, list(perm), choice)
    # lower bound: 4 wavefronts per access instruction
    nins = 4 + 4 + (2 if P == 9 else 0)
    return best, 4 * nins * 4 * len(starts)


if __name__ == "__main__":
    cases = [(2, 7, 4), (2, 9, 4), (3, 7, 1), (3, 9, 1)]
    for D, P, G in cases:
        for AX in range(D):
            (tot, perm, choice), lb = best_map(D, P, AX, G)
            ident = sum(cost_pair(D, P, AX, G, (f0 + 2 * q) % P ** (D - 1), (f0 + 2 * q + 1) % P ** (D - 1), (0, 0, 0))
                        for q in range(4) for f0 in range(0, P ** (D - 1), 8))
            print(D, P, G, AX, "best", tot, "lower bound", lb, "identity/no swaps", ident, perm, choice, flush=True)
