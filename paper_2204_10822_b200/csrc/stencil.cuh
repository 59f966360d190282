// stencil.cuh — symmetric storage of the finest-level Jacobian and its row access.
//
// J is exactly symmetric: the sv linearisation with the modification of eq:modification
// is symmetric by construction, the mass / drag / std / Picard terms are symmetric,
// and the Dirichlet rows/columns are eliminated symmetrically with a unit diagonal.  So
// each node stores only the "upper" half of its 9-point 2x2-block stencil row, slot-major SoA
// (Jst[e * Nn + node], every load of a warp coalesced, no index arrays), 19 values per node:
//
//   e = 4u + 2k + m, u = 0..3:  block J_(node,k),(nb_u,m) toward the upper neighbours
//                               nb_u = node + off_u, off = (1, s-1, s, s+1) = E, NW, N, NE
//                               (stencil slots 5..8, slot = (dj+1)*3 + (di+1));
//   e = 16, 17, 18:             J_xx, J_xy (= J_yx), J_yy of the node's own block.
//
// The lower half of row `node` is the transpose of the upper blocks of its lower neighbours:
// slot sl = 0..3 (SW, S, SE, W) is block u = 3 - sl of node - off_u, transposed.  Dirichlet
// nodes store the identity (J_xx = J_yy = 1, all else 0) and interior nodes store 0 toward them,
// so the lower-half reconstruction is exact everywhere in the interior.  152 B per node instead
// of 288 B for the full stencil: every finest-level SpMV / smoother pass reads 47 % fewer bytes.
#pragma once

namespace seaice {

constexpr int kJS = 19;  // stored values per node
constexpr int kJDxx = 16, kJDxy = 17, kJDyy = 18;
constexpr double kJBytesNode = 8.0 * kJS;                         // 152
constexpr double kAsmBytesNode = kJBytesNode + 64.0;              // + v, v_o, F read; R written
constexpr double kSpmvBytesNode = kJBytesNode + 32.0;             // + x read, y written

__host__ __device__ constexpr int stencil_off(int u, int s) { return u == 0 ? 1 : (u == 1 ? s - 1 : (u == 2 ? s : s + 1)); }

// Full 36-value row (old slot layout Jr[sl*4 + 2k + m]) of an interior node.
__device__ __forceinline__ void stencil_row(const double* __restrict__ J, long long Nn, int s, int node,
                                            double (&Jr)[36]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double* up = J + (long long)(4 * u) * Nn + node;
    const double* lo = J + (long long)(4 * u) * Nn + (node - stencil_off(u, s));
    const int su = 5 + u, sl = 3 - u;
#pragma unroll
    for (int e = 0; e < 4; ++e) Jr[su * 4 + e] = __ldg(up + e * Nn);
    // transpose: J_(node,k),(lo,m) = J_(lo,m),(node,k) = lo's value at 2m + k
    Jr[sl * 4 + 0] = __ldg(lo);
    Jr[sl * 4 + 1] = __ldg(lo + 2 * Nn);
    Jr[sl * 4 + 2] = __ldg(lo + Nn);
    Jr[sl * 4 + 3] = __ldg(lo + 3 * Nn);
  }
  Jr[16] = __ldg(J + kJDxx * Nn + node);
  Jr[17] = __ldg(J + kJDxy * Nn + node);
  Jr[18] = Jr[17];
  Jr[19] = __ldg(J + kJDyy * Nn + node);
}

// Own 2x2 block (xx, xy, yx, yy) of any node.
__device__ __forceinline__ double4 stencil_diag(const double* __restrict__ J, long long Nn, int node) {
  const double xy = J[kJDxy * Nn + node];
  return make_double4(J[kJDxx * Nn + node], xy, xy, J[kJDyy * Nn + node]);
}

// (J x)_node for an interior node, straight from the symmetric storage.
__device__ __forceinline__ double2 stencil_apply(const double* __restrict__ J, long long Nn, int s, int node,
                                                 const double2* __restrict__ x) {
  const double2 xc = __ldg(x + node);
  const double xy = __ldg(J + kJDxy * Nn + node);
  double y0 = __ldg(J + kJDxx * Nn + node) * xc.x + xy * xc.y;
  double y1 = xy * xc.x + __ldg(J + kJDyy * Nn + node) * xc.y;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int off = stencil_off(u, s);
    const double* up = J + (long long)(4 * u) * Nn + node;
    const double2 xu = __ldg(x + node + off);
    y0 += __ldg(up) * xu.x + __ldg(up + Nn) * xu.y;
    y1 += __ldg(up + 2 * Nn) * xu.x + __ldg(up + 3 * Nn) * xu.y;
    const double* lo = up - off;
    const double2 xl = __ldg(x + node - off);
    y0 += __ldg(lo) * xl.x + __ldg(lo + 2 * Nn) * xl.y;
    y1 += __ldg(lo + Nn) * xl.x + __ldg(lo + 3 * Nn) * xl.y;
  }
  return make_double2(y0, y1);
}

}  // namespace seaice
