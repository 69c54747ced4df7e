// Periodic structured hex numbering by entity (shared by the fused kernels
// and the standalone scatter): assembly.py:89-133 generalised, identical to
// oracle/assembly.py hex_periodic + build_map for uniform order.
#pragma once
#include <stdint.h>

namespace sphp {

// ---------------------------------------------------------------------------
// Periodic hex numbering by entity (assembled modes): every local mode maps
// to one of 27 entities of its element (8 vertices, 12 edges, 6 faces, the
// interior) plus an offset; the per-mode (entity, offset) table is built
// once per CTA, the 27 entity bases once per element, so a gather/scatter
// index costs one shared load and one add.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int mode_code(int M, int nl) {
  const int b = M - 2;  // bubbles per edge (P - 1)
  const int p = nl / (M * M), q = (nl / M) % M, r = nl % M;
  const int idx[3] = {p, q, r};
  const int nb = (p >= 2) + (q >= 2) + (r >= 2);
  int cls, off;
  if (nb == 0) {
    cls = p * 4 + q * 2 + r;
    off = 0;
  } else if (nb == 1) {
    const int d = (p >= 2) ? 0 : ((q >= 2) ? 1 : 2);
    int o[2], c = 0;
    for (int a = 0; a < 3; ++a)
      if (a != d) o[c++] = idx[a];
    cls = 8 + d * 4 + o[0] * 2 + o[1];
    off = idx[d] - 2;
  } else if (nb == 2) {
    const int d = (p < 2) ? 0 : ((q < 2) ? 1 : 2);
    int k[2], c = 0;
    for (int a = 0; a < 3; ++a)
      if (a != d) k[c++] = idx[a];
    cls = 20 + d * 2 + idx[d];
    off = (k[0] - 2) * b + (k[1] - 2);
  } else {
    cls = 26;
    off = ((p - 2) * b + (q - 2)) * b + (r - 2);
  }
  return cls | (off << 5);
}

// ---------------------------------------------------------------------------
// Entity classes in closed form: class k of element (x, y, z) is the entity
// R + size * vid(x + dx, y + dy, z + dz) (periodic wrap), the form that the
// class-range kernels (periodic_ops.cu, pipeline MODE 5) evaluate per
// segment / tile with a few integer ops.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int class_size(int k, int b) {
  return k < 8 ? 1 : (k < 20 ? b : (k < 26 ? b * b : b * b * b));
}
// does class k's entity sit at x + 1 (the element's high-x side)?
__host__ __device__ __forceinline__ int class_dx(int k) {
  return k < 8    ? (k >> 2)
         : k < 20 ? ((((k - 8) >> 2) != 0) ? ((k - 8) >> 1) & 1 : 0)  // edge off the x axis
         : k < 26 ? ((((k - 20) >> 1) == 0) ? (k - 20) & 1 : 0)       // x-normal face
                  : 0;
}
// class k's entity of element (x, y, z) is gid = R + size * vid(x + dx,
// y + dy, z + dz) (periodic wrap): the closed form of entity_base
// (periodic.cuh) that per-segment code evaluates with a few integer ops
struct ClassGeom {
  int R, s, d;  // region base, entity size, dx | dy << 1 | dz << 2
};
__host__ __device__ __forceinline__ ClassGeom class_geom(int k, int n, int P) {
  const int N3 = n * n * n, b = P - 1;
  if (k < 8) return {0, 1, ((k >> 2) & 1) | (((k >> 1) & 1) << 1) | ((k & 1) << 2)};
  if (k < 20) {
    const int j = k - 8, dir = j >> 2, s0 = (j >> 1) & 1, s1 = j & 1;
    // the two shifts go to the axes other than dir, in order
    const int d = dir == 0 ? (s0 << 1) | (s1 << 2) : (dir == 1 ? s0 | (s1 << 2) : s0 | (s1 << 1));
    return {N3 + dir * N3 * b, b, d};
  }
  if (k < 26) {
    const int j = k - 20, dir = j >> 1, side = j & 1;
    return {N3 + 3 * N3 * b + dir * N3 * b * b, b * b, side << dir};
  }
  return {N3 * (1 + 3 * b + 3 * b * b), b * b * b, 0};
}
__host__ __device__ __forceinline__ int class_gid(const ClassGeom& g, int n, int x, int y, int z) {
  x += g.d & 1;
  y += (g.d >> 1) & 1;
  z += (g.d >> 2) & 1;
  x -= x >= n ? n : 0;
  y -= y >= n ? n : 0;
  z -= z >= n ? n : 0;
  return g.R + g.s * (x + n * (y + n * z));
}
__host__ __device__ __forceinline__ int entity_base(int n, int P, int ex, int ey, int ez, int k) {
  const int N3 = n * n * n, b = P - 1;
  auto wrap = [n](int i) { return i >= n ? i - n : i; };
  auto vid = [&](int i, int j, int l) { return wrap(i) + n * (wrap(j) + n * wrap(l)); };
  const int base[3] = {ex, ey, ez};
  if (k < 8) return vid(ex + (k >> 2), ey + ((k >> 1) & 1), ez + (k & 1));
  if (k < 20) {
    const int j = k - 8, d = j >> 2;
    const int st[2] = {(j >> 1) & 1, j & 1};
    int c[3], m = 0;
    for (int a = 0; a < 3; ++a) c[a] = base[a] + (a == d ? 0 : st[m++]);
    return N3 + (d * N3 + vid(c[0], c[1], c[2])) * b;
  }
  if (k < 26) {
    const int j = k - 20, d = j >> 1, side = j & 1;
    int c[3] = {ex, ey, ez};
    c[d] += side;
    return N3 + 3 * N3 * b + (d * N3 + vid(c[0], c[1], c[2])) * b * b;
  }
  return N3 * (1 + 3 * b + 3 * b * b) + (ex + n * (ey + n * ez)) * b * b * b;
}

}  // namespace sphp
