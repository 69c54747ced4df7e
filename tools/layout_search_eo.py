"""Search shared-memory pitches of the K-row even-odd Helmholtz (HexHelmEO)
for odd Q: element stride SE, dense-tensor plane pitch SI, T1/T2 plane
pitches PP1/PP2 and the staged geometry element stride GEO_S (even), each
free mod 16.  Wavefront model: tools/bank_sim.py (FP64 accesses, one
wavefront per half-warp per distinct address per bank pair).  Stage access
lists mirror hex_ops.cuh:HexHelmEO::compute.  Prints the best combination
and its per-stage ratios against the current layout."""
import itertools
import sys

from bank_sim import stage_cost


def rowrot(M, R):
    g = 16 if M % 16 == 0 else 8 if M % 8 == 0 else 4 if M % 4 == 0 else 2 if M % 2 == 0 else 1
    per = 16 // g
    nv = 16 // per
    return (R // per) & (nv - 1)


def stages(M, Q, NE, NT, SE, SI, PP1, PP2, GS, CS):
    QK = Q | 1  # odd_up(Q), as HexHelmEO
    M3 = M ** 3
    OUT0 = NE * SE  # output block staged in W1 (OUT_OFF)
    W0, W1, W2 = 0, NE * SE, 2 * NE * SE
    st = {}
    it = [(e, p, q) for e in range(NE) for p in range(M) for q in range(M)]
    rr = lambda x: rowrot(M, x[0] * M * M + x[1] * M + x[2])
    st["S1"] = (it, lambda x: [x[0] * M3 + (x[1] * M + x[2]) * M + (r + rr(x)) % M for r in range(M)] +
                [W0 + x[0] * SE + x[1] * PP1 + x[2] * QK + k for k in range(Q)], ("SE", "PP1"))
    it = [(e, p, k) for e in range(NE) for p in range(M) for k in range(Q)]
    st["S2"] = (it, lambda x: [W0 + x[0] * SE + x[1] * PP1 + q * QK + x[2] for q in range(M)] +
                [W1 + x[0] * SE + x[1] * PP2 + j * Q + x[2] for j in range(Q)], ("SE", "PP1", "PP2"))
    it = [(e, j, k) for e in range(NE) for j in range(Q) for k in range(Q)]
    st["S3"] = (it, lambda x: [W1 + x[0] * SE + p * PP2 + x[1] * Q + x[2] for p in range(M)] +
                [W0 + x[0] * SE + i * SI + x[1] * Q + x[2] for i in range(Q)] +
                [W2 + x[0] * SE + i * SI + x[1] * Q + x[2] for i in range(Q)], ("SE", "PP2", "SI"))
    it = [(e, i, k) for e in range(NE) for i in range(Q) for k in range(Q)]
    st["S4"] = (it, lambda x: [W0 + x[0] * SE + x[1] * SI + j * Q + x[2] for j in range(Q)] +
                [W1 + x[0] * SE + x[1] * SI + j * Q + x[2] for j in range(Q)], ("SE", "SI"))
    it = [(e, i, j) for e in range(NE) for i in range(Q) for j in range(Q)]
    st["S5"] = (it, lambda x: [W + x[0] * SE + x[1] * SI + x[2] * Q + k for W in (W0, W2, W1) for k in range(Q)] +
                [x[0] * GS + c * CS + (x[1] * Q + x[2]) * Q + k for c in range(7) for k in range(Q)] +
                [W + x[0] * SE + x[1] * SI + x[2] * Q + k for W in (W0, W2, W1) for k in range(Q)],
                ("SE", "SI", "GS"))
    it = [(e, i, k) for e in range(NE) for i in range(Q) for k in range(Q)]
    st["S6"] = (it, lambda x: [W + x[0] * SE + x[1] * SI + j * Q + x[2] for W in (W1, W0, W0) for j in range(Q)],
                ("SE", "SI"))
    it = [(e, j, k) for e in range(NE) for j in range(Q) for k in range(Q)]
    st["S7"] = (it, lambda x: [W + x[0] * SE + i * SI + x[1] * Q + x[2] for W in (W0, W2) for i in range(Q)] +
                [W1 + x[0] * SE + p * PP2 + x[1] * Q + x[2] for p in range(M)], ("SE", "SI", "PP2"))
    it = [(e, p, k) for e in range(NE) for p in range(M) for k in range(Q)]
    st["S8"] = (it, lambda x: [W1 + x[0] * SE + x[1] * PP2 + j * Q + x[2] for j in range(Q)] +
                [W0 + x[0] * SE + x[1] * PP1 + q * QK + x[2] for q in range(M)], ("SE", "PP1", "PP2"))
    it = [(e, p, q) for e in range(NE) for p in range(M) for q in range(M)]
    st["S9"] = (it, lambda x: [W0 + x[0] * SE + x[1] * PP1 + x[2] * QK + k for k in range(Q)] +
                [OUT0 + x[0] * M3 + (x[1] * M + x[2]) * M + (r + rr(x)) % M for r in range(M)], ("SE", "PP1"))
    return st


def total(M, Q, NE, NT, prm, CS):
    st = stages(M, Q, NE, NT, prm["SE"], prm["SI"], prm["PP1"], prm["PP2"], prm["GS"], CS)
    out = {}
    for k, (it, acc, _) in st.items():
        out[k] = stage_cost(it, NT, acc)
    return out


def main(M, Q, NE, NT):
    CS = Q ** 3 + (Q ** 3) % 2
    def up(lo, r):  # smallest v >= lo with v = r mod 16
        v = lo
        while v % 16 != r % 16:
            v += 1
        return v
    cur_pp1 = up(M * Q, Q)
    cur_pp2 = up(Q * Q, Q)
    cur = dict(SI=Q * Q, PP1=cur_pp1, PP2=cur_pp2, GS=7 * CS,
               SE=max(Q ** 3, M * cur_pp1, M * cur_pp2) + (max(Q ** 3, M * cur_pp1, M * cur_pp2) % 2))
    base = total(M, Q, NE, NT, cur, CS)
    bt = sum(v[0] for v in base.values())
    ideal = sum(v[1] for v in base.values())
    print(f"M={M} Q={Q} NE={NE} NT={NT} current {cur}: {bt} wavefronts (ideal {ideal}, {bt/ideal:.2f}x)")
    print("   ", {k: round(v[0] / v[1], 2) for k, v in base.items()})
    # coordinate search: each parameter over its 16 residues, repeat
    best = dict(cur)
    best_t = bt
    ranges = {"SI": range(Q * Q, Q * Q + 16), "PP1": range(M * Q, M * Q + 16),
              "PP2": range(Q * Q, Q * Q + 16), "GS": range(7 * CS, 7 * CS + 16, 2)}
    for rnd in range(3):
        for key in ("SI", "PP1", "PP2", "GS", "SE"):
            cands = ranges.get(key)
            if key == "SE":
                lo = max(Q * best["SI"], M * best["PP1"], M * best["PP2"])
                cands = range(lo, lo + 16)
            for v in cands:
                trial = dict(best)
                trial[key] = v
                if key != "SE":
                    lo = max(Q * trial["SI"], M * trial["PP1"], M * trial["PP2"])
                    if trial["SE"] < lo:
                        trial["SE"] = up(lo, trial["SE"])
                t = sum(x[0] for x in total(M, Q, NE, NT, trial, CS).values())
                if t < best_t:
                    best_t, best = t, trial
        print(f"  round {rnd}: {best} {best_t} ({best_t/ideal:.2f}x)", flush=True)
    fin = total(M, Q, NE, NT, best, CS)
    print("   ", {k: round(v[0] / v[1], 2) for k, v in fin.items()})


if __name__ == "__main__":
    M, Q, NE, NT = (int(v) for v in sys.argv[1:5])
    main(M, Q, NE, NT)
