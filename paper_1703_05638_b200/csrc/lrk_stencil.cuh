// lrk_stencil.cuh — node-level evaluation of the matrix-free operator L
// (box stencil + per-node upwind or Galerkin Q1 convection), shared by the
// stencil kernels (lrk_misc.cu) and the persistent step-solve kernel
// (lrk_rich.cu).
#pragma once
#include "lrk_misc.h"

namespace lrk {

// Local wind at interior node (i1, i2, i3): w0 + (2 x2 (1 - x1^2), -2 x1 (1 - x2^2), 0).
__device__ __forceinline__ double wind_at(const StencilArgs& a, int ax, int i1, int i2) {
  const double x1 = a.h * (i1 + 1), x2 = a.h * (i2 + 1);
  if (ax == 0) return a.w0[0] + 2.0 * x2 * (1.0 - x1 * x1);
  if (ax == 1) return a.w0[1] - 2.0 * x1 * (1.0 - x2 * x2);
  return a.w0[2];
}

// Per-node first-order upwind (row i of W, or of W^T for the adjoint):
// row q: diag += |w_a(q)|/h; entry (q, q - e_a) = -w_a(q)/h if w_a(q) > 0,
// entry (q, q + e_a) = +w_a(q)/h if w_a(q) < 0.
template <typename Ld>
__device__ __forceinline__ double var_upwind(const StencilArgs& a, const double* x, int64_t i,
                                             int i1, int i2, int i3, int64_t plane, Ld ld) {
  const int n = a.n;
  const double ih = 1.0 / a.h;
  double acc = 0.0;
  const int idx[3] = {i1, i2, i3};
  const int64_t stride[3] = {1, n, plane};
  for (int ax = 0; ax < a.dim; ++ax) {
    const double w = wind_at(a, ax, i1, i2);
    acc += fabs(w) * ih * ld(x + i);
    if (!a.adjoint) {
      if (w > 0.0 && idx[ax] > 0) acc -= w * ih * ld(x + i - stride[ax]);
      if (w < 0.0 && idx[ax] < n - 1) acc += w * ih * ld(x + i + stride[ax]);
    } else {
      // column i of W: rows i + e_a (their lower neighbour is i) and i - e_a
      if (idx[ax] < n - 1) {
        const double wp = wind_at(a, ax, i1 + (ax == 0), i2 + (ax == 1));
        if (wp > 0.0) acc -= wp * ih * ld(x + i + stride[ax]);
      }
      if (idx[ax] > 0) {
        const double wm = wind_at(a, ax, i1 - (ax == 0), i2 - (ax == 1));
        if (wm < 0.0) acc += wm * ih * ld(x + i - stride[ax]);
      }
    }
  }
  return acc;
}

// Galerkin Q1 convection row (or column, for the adjoint) at interior node
// (i1, i2) from its 3 x 3 neighbourhood v[(d2+1)*3 + (d1+1)] (zero outside the
// domain).  Element (p1, p2) spans nodes p..p+1 per axis (node -1 and n are
// the Dirichlet boundary); with the wind (wx, wy) of its centre,
//   N^e_ab = h [ wx (s_b1 / 2) m(a2, b2) + wy m(a1, b1) (s_b2 / 2) ],
//   s_0 = -1, s_1 = +1, m(equal) = 1/3, m(different) = 1/6.
// Returns (N v)_i / h^2 (lumped mass h^2), i.e. the term added to L v.
__device__ __forceinline__ double galerkin_nb(const StencilArgs& a, int i1, int i2, const double (&v)[9]) {
  double acc = 0.0;
#pragma unroll
  for (int e2 = 0; e2 < 2; ++e2)
#pragma unroll
    for (int e1 = 0; e1 < 2; ++e1) {
      const int p1 = i1 - 1 + e1, p2 = i2 - 1 + e2;       // lower-left node of the element
      const double xc = a.h * (p1 + 1.5), yc = a.h * (p2 + 1.5);
      const double wx = a.w0[0] + (a.rotating ? 2.0 * yc * (1.0 - xc * xc) : 0.0);
      const double wy = a.w0[1] - (a.rotating ? 2.0 * xc * (1.0 - yc * yc) : 0.0);
      const int l1 = 1 - e1, l2 = 1 - e2;                 // local index of node i in the element
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
        for (int q1 = 0; q1 < 2; ++q1) {
          // forward: a = (l1, l2) is the test node, b = (q1, q2); adjoint: swapped
          const int a1 = a.adjoint ? q1 : l1, a2 = a.adjoint ? q2 : l2;
          const int b1 = a.adjoint ? l1 : q1, b2 = a.adjoint ? l2 : q2;
          const double m1 = a1 == b1 ? (1.0 / 3.0) : (1.0 / 6.0);
          const double m2 = a2 == b2 ? (1.0 / 3.0) : (1.0 / 6.0);
          const double ne = wx * (b1 ? 0.5 : -0.5) * m2 + wy * m1 * (b2 ? 0.5 : -0.5);
          const int d1 = p1 + q1 - i1, d2 = p2 + q2 - i2;
          acc += ne * v[(d2 + 1) * 3 + (d1 + 1)];
        }
    }
  return acc / a.h;
}

// (L x)_i at node i = (i1, i2, i3) of column x, neighbours read with the
// loader `ld` (plain loads, or L2 loads where another CTA of the same launch
// wrote x).
template <typename Ld>
__device__ __forceinline__ double stencil_lx(const StencilArgs& a, const double* x, int64_t i, int i1,
                                             int i2, int i3, Ld ld) {
  const int n = a.n;
  const int64_t plane = (int64_t)n * n;
  double lx = 0.0;
  const int d3lo = a.dim == 3 ? -1 : 0, d3hi = a.dim == 3 ? 1 : 0;
  for (int d3 = d3lo; d3 <= d3hi; ++d3) {
    if (i3 + d3 < 0 || i3 + d3 >= (a.dim == 3 ? n : 1)) continue;
#pragma unroll
    for (int d2 = -1; d2 <= 1; ++d2) {
      if (i2 + d2 < 0 || i2 + d2 >= n) continue;
#pragma unroll
      for (int d1 = -1; d1 <= 1; ++d1) {
        const double cf = a.coef[(d3 + 1) * 9 + (d2 + 1) * 3 + (d1 + 1)];
        if (cf == 0.0 || i1 + d1 < 0 || i1 + d1 >= n) continue;
        lx += cf * ld(x + i + d1 + (int64_t)d2 * n + (int64_t)d3 * plane);
      }
    }
  }
  if (a.wind_field) lx += var_upwind(a, x, i, i1, i2, i3, plane, ld);
  if (a.galerkin) {
    double v[9];
#pragma unroll
    for (int d2 = -1; d2 <= 1; ++d2)
#pragma unroll
      for (int d1 = -1; d1 <= 1; ++d1) {
        const bool in = i1 + d1 >= 0 && i1 + d1 < n && i2 + d2 >= 0 && i2 + d2 < n;
        v[(d2 + 1) * 3 + (d1 + 1)] = in ? ld(x + i + d1 + (int64_t)d2 * n) : 0.0;
      }
    lx += galerkin_nb(a, i1, i2, v);
  }
  return lx;
}

}  // namespace lrk
