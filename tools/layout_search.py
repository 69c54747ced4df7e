"""Brute-force search of shared-memory pitches for the Q^3 work tensors of
HexHelm: address(i,j,k) = i*SI + j*SJ + k.  Access patterns (lanes over
work items, items ordered as in the kernel):
  pencil-i stages (S3/S7): lanes (j,k) k fastest, scalar loads over i
  pencil-j stage  (S5):    lanes (i,k) k fastest, scalar loads over j
  pencil-k stages (S4/S6): lanes (i,j) j fastest, loads over k, scalar or
                           128-bit pairs (needs SI, SJ even, Q even)
Cost = wavefronts / ideal, weighted by how many accesses each stage makes."""
import sys

def wf64(addrs):
    t = 0
    for h in (addrs[:16], addrs[16:]):
        b = {}
        for a in h:
            b.setdefault(a % 16, set()).add(a)
        t += max((len(v) for v in b.values()), default=0)
    return t

def wf128(addrs):
    # addrs are double indices (even); 8-lane phases of 16B
    t = 0
    for p in range(0, len(addrs), 8):
        b = {}
        for a in addrs[p:p + 8]:
            b.setdefault((a // 2) % 8, set()).add(a)
        t += max((len(v) for v in b.values()), default=0)
    return t

def cost(Q, NE, SI, SJ, SE, vec):
    items_jk = [(e, j, k) for e in range(NE) for j in range(Q) for k in range(Q)]
    items_ik = items_jk
    items_ij = items_jk
    tot = ideal = 0
    def run(items, addr_fn, nacc, weight, vec128=False):
        nonlocal tot, ideal
        for w0 in range(0, len(items), 32):
            lanes = items[w0:w0 + 32]
            if vec128:
                for s in range(0, Q, 2):
                    addrs = [addr_fn(x, s) for x in lanes]
                    tot += weight * wf128(addrs)
                    ideal += weight * ((len(lanes) + 7) // 8)
            else:
                for s in range(nacc):
                    addrs = [addr_fn(x, s) for x in lanes]
                    tot += weight * wf64(addrs)
                    ideal += weight * (2 if len(lanes) > 16 else 1)
    # pencil-i: lanes (j,k)
    run(items_jk, lambda x, s: x[0] * SE + s * SI + x[1] * SJ + x[2], Q, 4)
    # pencil-j: lanes (i,k)
    run(items_ik, lambda x, s: x[0] * SE + x[1] * SI + s * SJ + x[2], Q, 6)
    # pencil-k: lanes (i,j)
    run(items_ij, lambda x, s: x[0] * SE + x[1] * SI + x[2] * SJ + s, Q, 5, vec128=vec)
    return tot / ideal

if __name__ == "__main__":
    Q = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    NE = 3
    best = []
    for SJ in range(Q, Q + 12):
        for SI in range(Q * SJ, Q * SJ + 24):
            for vec in ((False, True) if Q % 2 == 0 and SJ % 2 == 0 and SI % 2 == 0 else (False,)):
                SE = Q * SI + 1
                for pad in range(0, 8):
                    c = cost(Q, NE, SI, SJ, SE + pad, vec)
                    best.append((c, SJ, SI, SE + pad, vec))
    best.sort()
    for b in best[:8]:
        print("cost %.3f SJ=%d SI=%d SE=%d vec128=%s" % b)
    print("current (QK odd):", cost(Q, NE, Q * (Q | 1), Q | 1, (Q * Q * (Q | 1)) | 1, False))
