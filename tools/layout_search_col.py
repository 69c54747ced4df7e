"""Wavefront-model search of the shared-memory pitches and lane orders of
the i-column Helmholtz plan (HexHelmCol, hex_ops.cuh):

  S1 r->k  lanes (e,p,q): writes A tensors T1, T1d   [p][q][k]
  S2 q->j  lanes over (e,p,k): reads T1, T1d along q, writes B tensors T2, T2e, T2f
  S5 i     lanes over (e,j,k): reads B columns along p, geometry columns
                               along i, writes B columns
  B1 j->q  lanes as S2: reads B along j, writes A tensors V0, V1
  B2 k->r  lanes as S1: reads V0, V1 along k

A tensors: addr = e*SEA + p*PA + q*RA + k.  B tensors: addr = e*SEB + p*PB +
j*Q + k.  Geometry: e*GS + c*CS + i*Q^2 + j*Q + k.
Lane orders: 'nat' = element-major, last index fastest; 'ef' = element
fastest; 'pf' = element-major, p fastest (S2 / B1 only).
Model: tools/bank_sim.py (a half-warp is one wavefront when its addresses
fall on distinct 8-byte bank pairs).  The three address families are
independent given the lane orders, so each is minimised on its own.

usage: layout_search_col.py M Q NE NT
"""
import sys
from bank_sim import stage_cost


def items(order, NE, n1, n2):
    if order == "nat":
        return [(e, a, b) for e in range(NE) for a in range(n1) for b in range(n2)]
    if order == "ef":
        return [(e, a, b) for a in range(n1) for b in range(n2) for e in range(NE)]
    if order == "pf":
        return [(e, a, b) for e in range(NE) for b in range(n2) for a in range(n1)]
    raise ValueError(order)


def cost_a(M, Q, NE, NT, RA, PA, SEA, o2):
    it1 = items("nat", NE, M, M)
    rows = lambda x: [x[0] * SEA + x[1] * PA + x[2] * RA + k for k in range(Q)]
    c1 = stage_cost(it1, NT, lambda x: rows(x) * 4)  # S1 writes 2, B2 reads 2
    it2 = items(o2, NE, M, Q)
    colq = lambda x: [x[0] * SEA + x[1] * PA + q * RA + x[2] for q in range(M)]
    c2 = stage_cost(it2, NT, lambda x: colq(x) * 4)  # S2 reads 2, B1 writes 2
    return c1[0] + c2[0], c1[1] + c2[1]


def cost_b(M, Q, NE, NT, PB, SEB, o2, o5):
    it2 = items(o2, NE, M, Q)
    colj = lambda x: [x[0] * SEB + x[1] * PB + j * Q + x[2] for j in range(Q)]
    c2 = stage_cost(it2, NT, lambda x: colj(x) * 6)  # S2 writes 3, B1 reads 3
    it5 = items(o5, NE, Q, Q)
    colp = lambda x: [x[0] * SEB + p * PB + x[1] * Q + x[2] for p in range(M)]
    c5 = stage_cost(it5, NT, lambda x: colp(x) * 6)
    return c2[0] + c5[0], c2[1] + c5[1]


def cost_g(M, Q, NE, NT, GS, o5):
    it5 = items(o5, NE, Q, Q)
    col = lambda x: [x[0] * GS + i * Q * Q + x[1] * Q + x[2] for i in range(Q)]
    c = stage_cost(it5, NT, lambda x: col(x) * 7)
    return c


def with_res(lo, res):
    v = lo
    while v % 16 != res:
        v += 1
    return v


def search(M, Q, NE, NT, verbose=True):
    CS = (Q ** 3 + 1) & ~1
    out = []
    for o2 in ("nat", "ef", "pf"):
        # A family
        bestA = None
        for RA in range(Q, Q + 5):
            for PA in range(M * RA, M * RA + 16):
                for res in range(16):
                    SEA = with_res(2 * M * PA, res)
                    c = cost_a(M, Q, NE, NT, RA, PA, SEA, o2)
                    key = (c[0], SEA)
                    if bestA is None or key < bestA[0]:
                        bestA = (key, dict(RA=RA, PA=PA, SEA=SEA), c)
        for o5 in ("nat", "ef"):
            bestB = None
            for PB in range(Q * Q, Q * Q + 16):
                for res in range(16):
                    SEB = with_res(3 * M * PB, res)
                    c = cost_b(M, Q, NE, NT, PB, SEB, o2, o5)
                    key = (c[0], SEB)
                    if bestB is None or key < bestB[0]:
                        bestB = (key, dict(PB=PB, SEB=SEB), c)
            bestG = None
            for res in range(0, 16, 2):
                GS = with_res(7 * CS, res)
                c = cost_g(M, Q, NE, NT, GS, o5)
                key = (c[0], GS)
                if bestG is None or key < bestG[0]:
                    bestG = (key, dict(GS=GS), c)
            tot = bestA[2][0] + bestB[2][0] + bestG[2][0]
            ideal = bestA[2][1] + bestB[2][1] + bestG[2][1]
            foot = bestA[1]["SEA"] + bestB[1]["SEB"] + bestG[1]["GS"]
            out.append((tot / NE, round(tot / ideal, 3), foot, o2, o5, bestA[1], bestB[1], bestG[1],
                        "A %.2f B %.2f G %.2f" % (bestA[2][0] / bestA[2][1], bestB[2][0] / bestB[2][1],
                                                   bestG[2][0] / bestG[2][1])))
    out.sort(key=lambda t: (t[0], t[2]))
    return out


if __name__ == "__main__":
    M, Q = int(sys.argv[1]), int(sys.argv[2])
    NE = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    NT = int(sys.argv[4]) if len(sys.argv) > 4 else 128
    for b in search(M, Q, NE, NT):
        print(b)
