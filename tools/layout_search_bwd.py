"""Wavefront-model search (tools/bank_sim.py) of the work-tensor pitches of
HexBwd / HexIprod: A[p][q][k] (row RA, plane PA, element SA) and
B[p][j][k] (row RB, plane PB, element SB).  Coordinate descent from the
current layout (RA = RB = odd_up(Q), PA = M*RA, PB = Q*RB, SA/SB odd)."""
import sys

from bank_sim import stage_cost


def cost(M, Q, NE, NT, prm, iprod=False):
    RA, PA, SA, RB, PB, SB = (prm[k] for k in ("RA", "PA", "SA", "RB", "PB", "SB"))
    M3, Q3 = M ** 3, Q ** 3
    A0, B0, O0 = 0, NE * SA, NE * SA + NE * SB + 100000
    tot = 0
    ideal = 0
    it = [(e, p, q) for e in range(NE) for p in range(M) for q in range(M)]
    if not iprod:
        acc = lambda x: [O0 + x[0] * M3 + (x[1] * M + x[2]) * M + r for r in range(M)] + \
                        [A0 + x[0] * SA + x[1] * PA + x[2] * RA + k for k in range(Q)]
    else:
        acc = lambda x: [A0 + x[0] * SA + x[1] * PA + x[2] * RA + k for k in range(Q)] + \
                        [O0 + x[0] * M3 + (x[1] * M + x[2]) * M + r for r in range(M)]
    w, i = stage_cost(it, NT, acc); tot += w; ideal += i
    it = [(e, p, k) for e in range(NE) for p in range(M) for k in range(Q)]
    acc = lambda x: [A0 + x[0] * SA + x[1] * PA + q * RA + x[2] for q in range(M)] + \
                    [B0 + x[0] * SB + x[1] * PB + j * RB + x[2] for j in range(Q)]
    w, i = stage_cost(it, NT, acc); tot += w; ideal += i
    it = [(e, j, k) for e in range(NE) for j in range(Q) for k in range(Q)]
    acc = lambda x: [B0 + x[0] * SB + p * PB + x[1] * RB + x[2] for p in range(M)] + \
                    [O0 + x[0] * Q3 + ii * Q * Q + x[1] * Q + x[2] for ii in range(Q)]
    w, i = stage_cost(it, NT, acc); tot += w; ideal += i
    return tot, ideal


def main(M, Q, NE, NT, iprod):
    odd = lambda v: v | 1
    QK = odd(Q)
    cur = dict(RA=QK, PA=M * QK, SA=odd(M * M * QK), RB=QK, PB=Q * QK, SB=odd(M * Q * QK))
    t0, ideal = cost(M, Q, NE, NT, cur, iprod)
    print(f"{'iprod' if iprod else 'bwd'} M={M} Q={Q} NE={NE} NT={NT} current {cur}: {t0} ({t0/ideal:.2f}x)")
    best, bt = dict(cur), t0
    for rnd in range(3):
        for key in ("RA", "RB", "PA", "PB", "SA", "SB"):
            lo = {"RA": Q, "RB": Q, "PA": M * best["RA"], "PB": Q * best["RB"],
                  "SA": M * best["PA"], "SB": M * best["PB"]}[key]
            for v in range(lo, lo + 16):
                tr = dict(best)
                tr[key] = v
                tr["PA"] = max(tr["PA"], M * tr["RA"])
                tr["PB"] = max(tr["PB"], Q * tr["RB"])
                tr["SA"] = max(tr["SA"], M * tr["PA"])
                tr["SB"] = max(tr["SB"], M * tr["PB"])
                t, _ = cost(M, Q, NE, NT, tr, iprod)
                if t < bt:
                    bt, best = t, tr
        print(f"  round {rnd}: {best} {bt} ({bt/ideal:.2f}x)", flush=True)


if __name__ == "__main__":
    M, Q, NE, NT = (int(v) for v in sys.argv[1:5])
    main(M, Q, NE, NT, len(sys.argv) > 5 and sys.argv[5] == "iprod")
