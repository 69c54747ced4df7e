"""Shared-memory wavefront model for the HexHelm stages (FP64 accesses:
each half-warp of 16 lanes is one 128-byte wavefront when its addresses hit
distinct 8-byte bank pairs; identical addresses broadcast)."""
import itertools
import sys

def wavefronts(addrs):
    """addrs: list of 32 double-indices (None = inactive lane)."""
    total = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in half:
            if a is None:
                continue
            banks.setdefault(a % 16, set()).add(a)
        total += max((len(v) for v in banks.values()), default=0)
    return total

def stage_cost(items, nt, accesses):
    """items: list of work items; accesses(item) -> list of addresses (one per
    instruction, same count for every item).  Returns (wavefronts, ideal)."""
    wf = ideal = 0
    for w0 in range(0, len(items), nt):
        for warp0 in range(w0, min(w0 + nt, len(items)), 32):
            lanes = items[warp0:warp0 + 32]
            acc = [accesses(it) for it in lanes]
            for k in range(len(acc[0])):
                addrs = [a[k] for a in acc] + [None] * (32 - len(acc))
                wf += wavefronts(addrs)
                ideal += (2 if len(acc) > 16 else 1)
    return wf, ideal

def hexhelm(M, Q, NE, NT, QK, SW_fn, CSpad):
    SW = SW_fn(M, Q, QK)
    CS = CSpad
    M3 = M ** 3
    res = {}
    it = [(e, pq) for e in range(NE) for pq in range(M * M)]
    res["S1 r"] = stage_cost(it, NT, lambda x: [x[0] * M3 + x[1] * M + r for r in range(M)] +
                                               [x[0] * SW + x[1] * QK + k for k in range(Q)])
    it = [(e, p, k) for e in range(NE) for p in range(M) for k in range(Q)]
    res["S2 q"] = stage_cost(it, NT, lambda x: [x[0] * SW + x[1] * M * QK + q * QK + x[2] for q in range(M)] +
                                               [x[0] * SW + x[1] * Q * QK + j * QK + x[2] for j in range(Q)])
    it = [(e, j, k) for e in range(NE) for j in range(Q) for k in range(Q)]
    res["S3 p"] = stage_cost(it, NT, lambda x: [x[0] * SW + p * Q * QK + x[1] * QK + x[2] for p in range(M)] +
                                               [x[0] * SW + i * Q * QK + x[1] * QK + x[2] for i in range(Q)] * 2)
    it = [(e, i, j) for e in range(NE) for i in range(Q) for j in range(Q)]
    res["S4 k"] = stage_cost(it, NT, lambda x: [x[0] * SW + (x[1] * Q + x[2]) * QK + k for k in range(Q)] * 2)
    it = [(e, i, k) for e in range(NE) for i in range(Q) for k in range(Q)]
    res["S5 j"] = stage_cost(it, NT, lambda x: [x[0] * SW + x[1] * Q * QK + j * QK + x[2] for j in range(Q)] * 6 +
                             [x[0] * 7 * CS + c * CS + (x[1] * Q + j) * Q + x[2] for c in range(7) for j in range(Q)])
    it = [(e, i, j) for e in range(NE) for i in range(Q) for j in range(Q)]
    res["S6 k"] = stage_cost(it, NT, lambda x: [x[0] * SW + (x[1] * Q + x[2]) * QK + k for k in range(Q)] * 3)
    it = [(e, j, k) for e in range(NE) for j in range(Q) for k in range(Q)]
    res["S7 i"] = stage_cost(it, NT, lambda x: [x[0] * SW + i * Q * QK + x[1] * QK + x[2] for i in range(Q)] * 2 +
                                               [x[0] * SW + p * Q * QK + x[1] * QK + x[2] for p in range(M)])
    it = [(e, p, k) for e in range(NE) for p in range(M) for k in range(Q)]
    res["S8 j"] = stage_cost(it, NT, lambda x: [x[0] * SW + x[1] * Q * QK + j * QK + x[2] for j in range(Q)] +
                                               [x[0] * SW + x[1] * M * QK + q * QK + x[2] for q in range(M)])
    it = [(e, pq) for e in range(NE) for pq in range(M * M)]
    res["S9 k"] = stage_cost(it, NT, lambda x: [x[0] * SW + x[1] * QK + k for k in range(Q)] +
                                               [x[0] * M3 + x[1] * M + r for r in range(M)])
    return res

if __name__ == "__main__":
    M, Q, NE, NT = 5, 6, 3, 128
    for QK in (Q, Q + 1):
        for swname, swf in (("odd", lambda M, Q, QK: (Q * Q * QK) | 1), ("plain", lambda M, Q, QK: Q * Q * QK),
                            ("+4", lambda M, Q, QK: Q * Q * QK + 4)):
            r = hexhelm(M, Q, NE, NT, QK, swf, 216)
            tot = sum(v[0] for v in r.values()); ideal = sum(v[1] for v in r.values())
            print(f"QK={QK} SW={swname}: wavefronts {tot} ideal {ideal} ratio {tot/ideal:.2f}  " +
                  " ".join(f"{k}:{v[0]/v[1]:.2f}" for k, v in r.items()))
