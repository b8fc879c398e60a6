// cito_node.cuh — node relations of the transcription and their Jacobians (K3).
//
// Replaces cito.ocp.Transcription.node_constraints / node_jacobians
// (/root/reference/pkg/src/cito/ocp.py:272-365):
//   psi_fn     ocp.py:277-287   (integral cross-complementarity, FB on y increments)
//   theta_fn   ocp.py:289-296 -> impact_residuals cito/contact_dynamics.py:134-172
//   impulse_fn ocp.py:298-303 -> impact_map       cito/contact_dynamics.py:111-124
// One thread per (node item, input direction): the function is evaluated in
// forward-mode dual arithmetic seeded on that direction, giving one Jacobian
// column; direction 0 also writes the values.
#pragma once

#include "cito_kernels.cuh"

struct Dn {
  double v, d;
};
__device__ __forceinline__ Dn dn(double v) { return {v, 0.0}; }
__device__ __forceinline__ Dn operator+(Dn a, Dn b) { return {a.v + b.v, a.d + b.d}; }
__device__ __forceinline__ Dn operator-(Dn a, Dn b) { return {a.v - b.v, a.d - b.d}; }
__device__ __forceinline__ Dn operator-(Dn a) { return {-a.v, -a.d}; }
__device__ __forceinline__ Dn operator*(Dn a, Dn b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
__device__ __forceinline__ Dn operator*(double c, Dn a) { return {c * a.v, c * a.d}; }
__device__ __forceinline__ Dn operator/(Dn a, Dn b) {
  const double r = a.v / b.v;
  return {r, (a.d - r * b.d) / b.v};
}
__device__ __forceinline__ Dn dsqrt(Dn a) {
  const double r = sqrt(a.v);
  return {r, a.d * 0.5 / r};
}
__device__ __forceinline__ Dn dsabs(Dn x) { return dsqrt(x * x + dn(1.0)) - dn(1.0); }
__device__ __forceinline__ Dn dfb(Dn a, Dn b, double delta) {  // smoothmath.py:90-92
  return a + b - dsqrt(a * a + b * b + dn(delta));
}
__device__ __forceinline__ Dn dsng(Dn x) { return x / dsqrt(x * x + dn(1.0)); }  // contact_dynamics.py:50-52

// Node input [q-, v-, v+, Phi, Gamma] seeded on direction `dir`, read lazily from
// its three source segments (z or a packed vector): a dual is formed at each use
// instead of materialising all of them (their seeds alone would take 2 x NV
// registers per thread).
struct NodeIn {
  const double *p0, *p1, *p2;  // [q-, v-] | [v+] | [Phi, Gamma]
  int nq2, nq3, dir;
  __device__ __forceinline__ Dn at(int k) const {
    const double v = k < nq2 ? p0[k] : (k < nq3 ? p1[k - nq2] : p2[k - nq3]);
    return {v, dir == k ? 1.0 : 0.0};
  }
};
struct NodeView {  // NodeIn shifted by a segment offset
  const NodeIn& in;
  int off;
  __device__ __forceinline__ Dn operator[](int k) const { return in.at(off + k); }
};

// contact point, frame and signed distance in dual arithmetic (multibody.py:264-269, 384-411)
template <class M, class Q>
__device__ __forceinline__ void contact_geom(const KParams& P, const Q& q, int i, Dn* dPdth, Dn* n, Dn* t, Dn& sd) {
  const int l = M::clink(i);
  double sv, cv;
  sincos(q[3 * l + 2].v, &sv, &cv);
  const Dn c = {cv, -sv * q[3 * l + 2].d}, s = {sv, cv * q[3 * l + 2].d};
  const Dn rx = P.cr[i][0] * c - P.cr[i][1] * s;
  const Dn rz = P.cr[i][0] * s + P.cr[i][1] * c;
  const Dn Px = q[3 * l] + rx, Pz = q[3 * l + 1] + rz;
  dPdth[0] = -rz;
  dPdth[1] = rx;
  if constexpr (M::IMPLICIT) {
    T2 t2 = surface_t2(P, Px.v, Pz.v);
    const Dn h = {t2.v, t2.gx * Px.d + t2.gz * Pz.d};
    const Dn gx = {t2.gx, t2.hxx * Px.d + t2.hxz * Pz.d};
    const Dn gz = {t2.gz, t2.hxz * Px.d + t2.hzz * Pz.d};
    const Dn gn = dsqrt(gx * gx + gz * gz);
    n[0] = gx / gn;
    n[1] = gz / gn;
    sd = h / gn;
  } else {
    n[0] = dn(0.0);
    n[1] = dn(1.0);
    sd = Pz - dn(P.height);
  }
  t[0] = n[1];
  t[1] = -n[0];
}

template <class M>
__device__ __forceinline__ void node_psi(const KParams& P, const double* ya, const double* yb, int dir, double delta,
                                         double eps, double* val, double* jcol, int jstride) {
  constexpr int NC = M::NC, NY = 5 * NC + M::NGO;
  auto Y = [&](int k) -> Dn { return {k < NY ? ya[k] : yb[k - NY], dir == k ? 1.0 : 0.0}; };  // [y+_k, y-_{k+1}]
  int r = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    Dn d[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) d[k] = Y(NY + 5 * i + k) - Y(5 * i + k);
    const Dn rows[3] = {dfb(d[0], d[4], delta), dfb(d[0], d[1], delta), dfb(d[2], d[3], delta)};
#pragma unroll
    for (int k = 0; k < 3; ++k, ++r) {
      if (val) val[r] = rows[k].v;
      jcol[r * jstride] = rows[k].d;
    }
  }
#pragma unroll
  for (int o = 0; o < M::NGO; ++o, ++r) {
    const Dn v = Y(NY + 5 * NC + o) - Y(5 * NC + o) - dn(eps);
    if (val) val[r] = v.v;
    jcol[r * jstride] = v.d;
  }
}

template <class M>
__device__ __forceinline__ void node_theta(const KParams& P, const NodeIn& x, double delta, double* val,
                                           double* jcol, int jstride) {
  constexpr int NL = M::NL, NC = M::NC, NQ = 3 * NL;
  const NodeView q{x, 0}, vm{x, NQ}, vp{x, 2 * NQ}, Phi{x, 3 * NQ}, Gam{x, 3 * NQ + 2 * NC};
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int l = M::clink(i);
    Dn dP[2], n[2], t[2], sd;
    contact_geom<M>(P, q, i, dP, n, t, sd);
    Dn va[3], vb[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      va[k] = vp[3 * l + k] + P.crest[i] * vm[3 * l + k];
      vb[k] = vp[3 * l + k];
    }
    const Dn Ja0 = va[0] + dP[0] * va[2], Ja1 = va[1] + dP[1] * va[2];
    const Dn Jb0 = vb[0] + dP[0] * vb[2], Jb1 = vb[1] + dP[1] * vb[2];
    const Dn vn_rest = n[0] * Ja0 + n[1] * Ja1;
    const Dn vt_plus = t[0] * Jb0 + t[1] * Jb1;
    const Dn Pt = Phi[2 * i], Pn = Phi[2 * i + 1];
    const Dn cone = dsabs(P.mu[i] * Pn) - dsabs(Pt);
    const Dn rows[6] = {Pn * vn_rest, Pn * (vt_plus + Gam[i] * dsng(Pt)), dfb(Pn, sd, delta),
                        dfb(Gam[i], cone, delta), -sd, -vn_rest};
    const int ro[6] = {2 * i, 2 * i + 1, 2 * NC + 4 * i, 2 * NC + 4 * i + 1, 2 * NC + 4 * i + 2,
                       2 * NC + 4 * i + 3};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      if (val) val[ro[k]] = rows[k].v;
      jcol[ro[k] * jstride] = rows[k].d;
    }
  }
}

// The block pattern of the joint Gram matrix in joint order (joints coupled iff they
// share a link) and of its Cholesky factor with fill come from the generated
// topology (M::jfill_g / M::jfill_l, gen_models.py::joint_fill): constexpr bit tests
// that fold away in the unrolled loops, so the factor lives in registers.  Skipping
// the structural zeros leaves every computed value bit-identical to the dense
// factorisation (the skipped terms are exact zeros).
// Entry (2j+al, 2k+be) of the joint Gram matrix J M^-1 J^T in dual arithmetic
// (contact_dynamics.py:91-92), from the rotated joint anchors R[joint][side][xz].
template <class M, int NJP>
__device__ __forceinline__ Dn gram_entry(const KParams& P, const Dn (&R)[NJP][2][2], int j, int k, int al, int be) {
  Dn g = dn(0.0);
#pragma unroll
  for (int sa = 0; sa < 2; ++sa)
#pragma unroll
    for (int sb = 0; sb < 2; ++sb) {
      const int la = sa == 0 ? M::jparent(j) : M::jchild(j);
      const int lb = sb == 0 ? M::jparent(k) : M::jchild(k);
      if (la < 0 || la != lb) continue;
      const double sg = (sa == sb) ? 1.0 : -1.0;
      const Dn dA = al == 0 ? -R[j][sa][1] : R[j][sa][0], dB = be == 0 ? -R[k][sb][1] : R[k][sb][0];
      Dn v = P.minv_I[la] * (dA * dB);
      if (al == be) v = v + dn(P.minv_m[la]);
      g = g + sg * v;
    }
  return g;
}

template <class M>
__device__ __forceinline__ void node_impulse(const KParams& P, const NodeIn& x, double* val, double* jcol,
                                             int jstride) {
  constexpr int NL = M::NL, NJ = M::NJ, NC = M::NC, NQ = 3 * NL;
  const NodeView q{x, 0}, vm{x, NQ}, vp{x, 2 * NQ}, Phi{x, 3 * NQ};
  Dn w[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) w[k] = dn(0.0);
#pragma unroll
  for (int i = 0; i < NC; ++i) {  // _contact_wrench with impulses
    const int l = M::clink(i);
    Dn dP[2], n[2], t[2], sd;
    contact_geom<M>(P, q, i, dP, n, t, sd);
    const Dn F0 = t[0] * Phi[2 * i] + n[0] * Phi[2 * i + 1];
    const Dn F1 = t[1] * Phi[2 * i] + n[1] * Phi[2 * i + 1];
    w[3 * l] = w[3 * l] + F0;
    w[3 * l + 1] = w[3 * l + 1] + F1;
    w[3 * l + 2] = w[3 * l + 2] + (dP[0] * F0 + dP[1] * F1);
  }
  Dn out[NQ];
  if constexpr (NJ == 0) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      out[3 * l] = vm[3 * l] + P.minv_m[l] * w[3 * l];
      out[3 * l + 1] = vm[3 * l + 1] + P.minv_m[l] * w[3 * l + 1];
      out[3 * l + 2] = vm[3 * l + 2] + P.minv_I[l] * w[3 * l + 2];
    }
  } else {
    constexpr int NJ2 = 2 * NJ;
    Dn cth[NL], sth[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      double sv, cv;
      sincos(q[3 * l + 2].v, &sv, &cv);
      cth[l] = {cv, -sv * q[3 * l + 2].d};
      sth[l] = {sv, cv * q[3 * l + 2].d};
    }
    Dn R[Pos<NJ>::v][2][2];  // [joint][side][xz]
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int sa = 0; sa < 2; ++sa) {
        const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
        if (l < 0) continue;
        const double ax = sa == 0 ? P.jrp[j][0] : P.jrc[j][0], az = sa == 0 ? P.jrp[j][1] : P.jrc[j][1];
        R[j][sa][0] = ax * cth[l] - az * sth[l];
        R[j][sa][1] = ax * sth[l] + az * cth[l];
      }
    // Gram matrix G = J M^-1 J^T, packed lower triangle in joint order (values; the
    // tangent along this thread's direction, nonzero for link angles only, is
    // recomputed where the solve needs it)
    constexpr int NPK = NJ2 * (NJ2 + 1) / 2;
    double Lv[NPK];
#pragma unroll
    for (int e = 0; e < NPK; ++e) Lv[e] = 0.0;  // fill entries start at 0
    auto gram = [&](int j, int k, int al, int be) -> Dn { return gram_entry<M>(P, R, j, k, al, be); };
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int k = 0; k <= j; ++k)
#pragma unroll
        for (int al = 0; al < 2; ++al)
#pragma unroll
          for (int be = 0; be < 2; ++be) {
            if ((j == k && be > al) || !M::jfill_g(j, k)) continue;
            Lv[LI(2 * j + al, 2 * k + be)] = gram(j, k, al, be).v;
          }
    // rhs = J (v- + M^-1 w)
    Dn a[NQ];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      a[3 * l] = vm[3 * l] + P.minv_m[l] * w[3 * l];
      a[3 * l + 1] = vm[3 * l + 1] + P.minv_m[l] * w[3 * l + 1];
      a[3 * l + 2] = vm[3 * l + 2] + P.minv_I[l] * w[3 * l + 2];
    }
    double xv[NJ2], dx[NJ2];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int al = 0; al < 2; ++al) {
        Dn acc = dn(0.0);
#pragma unroll
        for (int sa = 0; sa < 2; ++sa) {
          const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
          if (l < 0) continue;
          const double sgn = sa == 0 ? 1.0 : -1.0;
          const Dn dPa = al == 0 ? -R[j][sa][1] : R[j][sa][0];
          acc = acc + sgn * (a[3 * l + al] + dPa * a[3 * l + 2]);
        }
        xv[2 * j + al] = acc.v;
        dx[2 * j + al] = acc.d;
      }
    // G x = rhs: Cholesky in joint order (the elimination order decides which
    // mathematically-zero Jacobian entries come out as exact zeros, and joint
    // order reproduces the reference's pattern; cito/contact_dynamics.py:117-121),
    // reciprocal pivots; the tangent reuses the factor: G dx = d(rhs) - dG x
    double Li[NJ2];
#pragma unroll
    for (int cc = 0; cc < NJ2; ++cc) {
      double d = Lv[LI(cc, cc)];
#pragma unroll
      for (int k = 0; k < cc; ++k)
        if (M::jfill_l(cc / 2, k / 2)) d = d - Lv[LI(cc, k)] * Lv[LI(cc, k)];
      Lv[LI(cc, cc)] = sqrt(d);
      Li[cc] = 1.0 / Lv[LI(cc, cc)];
#pragma unroll
      for (int r = cc + 1; r < NJ2; ++r) {
        if (!M::jfill_l(r / 2, cc / 2)) continue;
        double x2 = Lv[LI(r, cc)];
#pragma unroll
        for (int k = 0; k < cc; ++k)
          if (M::jfill_l(r / 2, k / 2) && M::jfill_l(cc / 2, k / 2)) x2 = x2 - Lv[LI(r, k)] * Lv[LI(cc, k)];
        Lv[LI(r, cc)] = x2 * Li[cc];
      }
    }
#pragma unroll
    for (int r = 0; r < NJ2; ++r) {
      double x2 = xv[r];
#pragma unroll
      for (int k = 0; k < r; ++k)
        if (M::jfill_l(r / 2, k / 2)) x2 = x2 - Lv[LI(r, k)] * xv[k];
      xv[r] = x2 * Li[r];
    }
#pragma unroll
    for (int r = NJ2 - 1; r >= 0; --r) {
      double x2 = xv[r];
#pragma unroll
      for (int k = r + 1; k < NJ2; ++k)
        if (M::jfill_l(k / 2, r / 2)) x2 = x2 - Lv[LI(k, r)] * xv[k];
      xv[r] = x2 * Li[r];
    }
    if (x.dir < NQ && x.dir % 3 == 2) {  // only link angles move G
#pragma unroll
    for (int r = 0; r < NJ2; ++r)
#pragma unroll
      for (int c = 0; c < NJ2; ++c)
        if (M::jfill_g(r / 2, c / 2)) {
          const Dn g = r >= c ? gram(r / 2, c / 2, r % 2, c % 2) : gram(c / 2, r / 2, c % 2, r % 2);
          dx[r] = __dsub_rn(dx[r], __dmul_rn(g.d, xv[c]));
        }
    }
#pragma unroll
    for (int r = 0; r < NJ2; ++r) {
      double x2 = dx[r];
#pragma unroll
      for (int k = 0; k < r; ++k)
        if (M::jfill_l(r / 2, k / 2)) x2 = __dsub_rn(x2, __dmul_rn(Lv[LI(r, k)], dx[k]));
      dx[r] = x2 * Li[r];
    }
#pragma unroll
    for (int r = NJ2 - 1; r >= 0; --r) {
      double x2 = dx[r];
#pragma unroll
      for (int k = r + 1; k < NJ2; ++k)
        if (M::jfill_l(k / 2, r / 2)) x2 = __dsub_rn(x2, __dmul_rn(Lv[LI(k, r)], dx[k]));
      dx[r] = x2 * Li[r];
    }
    Dn z[NJ2];
#pragma unroll
    for (int r = 0; r < NJ2; ++r) z[r] = {xv[r], dx[r]};
    // v+ = v- + M^-1 (w + J^T Phi_j)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int sa = 0; sa < 2; ++sa) {
        const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
        if (l < 0) continue;
        const double sgn = sa == 0 ? 1.0 : -1.0;
        const Dn l0 = -z[2 * j], l1 = -z[2 * j + 1];
        w[3 * l] = w[3 * l] + sgn * l0;
        w[3 * l + 1] = w[3 * l + 1] + sgn * l1;
        w[3 * l + 2] = w[3 * l + 2] + sgn * ((-R[j][sa][1]) * l0 + R[j][sa][0] * l1);
      }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      out[3 * l] = vm[3 * l] + P.minv_m[l] * w[3 * l];
      out[3 * l + 1] = vm[3 * l + 1] + P.minv_m[l] * w[3 * l + 1];
      out[3 * l + 2] = vm[3 * l + 2] + P.minv_I[l] * w[3 * l + 2];
    }
  }
#pragma unroll
  for (int k = 0; k < NQ; ++k) {
    const Dn r = vp[k] - out[k];
    if (val) val[k] = r.v;
    jcol[k * jstride] = r.d;
  }
}

#ifndef CITO_K3_MINB
#define CITO_K3_MINB 1
#endif
template <class M>
__global__ void __launch_bounds__(64, CITO_K3_MINB) k_node(const KParams P, int64_t Np, int64_t Nn, const double* __restrict__ y_pairs,
                                             const double* __restrict__ theta_vecs, double delta, double eps,
                                             double* __restrict__ psi, double* __restrict__ psi_jac,
                                             double* __restrict__ th, double* __restrict__ th_jac,
                                             double* __restrict__ imp, double* __restrict__ imp_jac, const ZSrc zs) {
  constexpr int NL = M::NL, NC = M::NC, NQ = 3 * NL, NY = 5 * NC + M::NGO;
  constexpr int NPSI = 3 * NC + M::NGO, NV = 3 * NQ + 3 * NC, NI = 3 * NQ + 2 * NC;
  constexpr int NXT = 2 * NQ + NY;
  if (zs.de) {  // relaxation parameters from device memory (CUDA-graph replays)
    delta = zs.de[0];
    eps = zs.de[1];
  }
  // item space: [Np * 2NY psi columns][Nn * NV theta columns][Nn * NI impulse columns]
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_psi = Np * (2 * NY), n_th = Nn * NV, n_imp = Nn * NI;
  if (t < n_psi) {
    constexpr int NY2 = Pos<2 * NY>::v;
    const int64_t k = t / NY2;
    const int d = (int)(t % NY2);
    const double* ya = y_pairs + k * 2 * NY;
    const double* yb = ya + NY;
    if (zs.z) {  // [y+_k, y-_{k+1}] straight from z (Transcription._node_inputs, ocp.py:316-318)
      const double* zb = zs.z + (k / zs.n_int) * zs.zstride;
      const int64_t kk = k % zs.n_int;
      ya = zb + (2 * kk + 1) * NXT + 2 * NQ;
      yb = zb + (2 * kk + 2) * NXT + 2 * NQ;
    }
    node_psi<M>(P, ya, yb, d, delta, eps, d == 0 ? psi + k * NPSI : nullptr, psi_jac + k * NPSI * 2 * NY + d, 2 * NY);
  } else if (t < n_psi + n_th + n_imp) {
    const bool is_th = t < n_psi + n_th;
    const int64_t e = is_th ? t - n_psi : t - n_psi - n_th;
    const int64_t k = is_th ? e / NV : e / NI;
    const int d = is_th ? (int)(e % NV) : (int)(e % NI);
    NodeIn x{theta_vecs + k * NV, theta_vecs + k * NV + 2 * NQ, theta_vecs + k * NV + 3 * NQ, 2 * NQ, 3 * NQ, d};
    if (zs.z) {  // [q-, v-, v+, Phi, Gamma] of node k straight from z (ocp.py:319-333)
      const double* zb = zs.z + (k / zs.n_node) * zs.zstride;
      const int64_t kk = k % zs.n_node;
      x.p0 = zb + 2 * kk * NXT;
      x.p1 = zb + (2 * kk + 1) * NXT + NQ;
      x.p2 = zb + zs.base_p + 3 * NC * kk;
    }
    if (is_th) {
      if (NC > 0)
        node_theta<M>(P, x, delta, d == 0 ? th + k * 6 * NC : nullptr, th_jac + k * 6 * NC * NV + d, NV);
    } else {
      node_impulse<M>(P, x, d == 0 ? imp + k * NQ : nullptr, imp_jac + k * NQ * NI + d, NI);
    }
  }
}

// ---------------------------------------------------------------------------
// K3, warp per node item (default): the same dual-number code as k_node, but a warp
// owns one item (an interval's psi block, a node's theta or impulse block) and its
// lanes evaluate only the input directions whose column can be nonzero for the
// topology (NodeDirs below: e.g. HalfCheetah impulse map 32 of 67, theta 24 of 69).
// The other columns are structural: zero, or the identity of v+ in the impulse
// defect v+ - impact_map(...).  Columns are assembled in a shared-memory tile and
// the warp writes the item's whole Jacobian block row by row (contiguous,
// coalesced, every sector written once) instead of 67 scattered column writes.
// Every computed entry is bit-identical to k_node's (same operations per direction).
template <class M>
struct NodeDirs {
  static constexpr int NL = M::NL, NC = M::NC, NQ = 3 * NL;
  static constexpr int NV = 3 * NQ + 3 * NC, NI = 3 * NQ + 2 * NC;
  static constexpr bool contact_link(int l) {
    for (int i = 0; i < NC; ++i)
      if (M::clink(i) == l) return true;
    return false;
  }
  // impulse map (contact_dynamics.py:111-124): link angles move the anchors, the Gram
  // matrix and the contact lever arms; contact-link positions move the contact frame
  // (implicit terrain only); v- and the impulses enter the solve; v+ only as identity
  static constexpr bool imp_live(int d) {
    if (d < NQ) return d % 3 == 2 || (M::IMPLICIT && contact_link(d / 3));
    if (d < 2 * NQ) return true;
    if (d < 3 * NQ) return false;
    return true;
  }
  // impact residuals (contact_dynamics.py:134-172): only the contact links' q, v-, v+
  // and the contact impulses / Gamma
  static constexpr bool th_live(int d) {
    if (d < 3 * NQ) return contact_link((d % NQ) / 3);
    return true;
  }
  int imp[NI > 0 ? NI : 1], th[NV > 0 ? NV : 1];
  int n_imp, n_th;
  constexpr NodeDirs() : imp(), th(), n_imp(0), n_th(0) {
    for (int d = 0; d < NI; ++d)
      if (imp_live(d)) imp[n_imp++] = d;
    for (int d = 0; d < NV; ++d)
      if (th_live(d)) th[n_th++] = d;
  }
};

// the live-direction tables in constant memory (indexed by lane at run time)
template <class M>
__constant__ const NodeDirs<M> kNodeDirs = NodeDirs<M>();

template <class M>
struct NodeTile {
  static constexpr int NL = M::NL, NC = M::NC, NQ = 3 * NL, NY = 5 * NC + M::NGO;
  static constexpr int NPSI = 3 * NC + M::NGO, NV = 3 * NQ + 3 * NC, NI = 3 * NQ + 2 * NC;
  static constexpr int A = NPSI * 2 * NY, B = 6 * NC * NV, C = NQ * NI;
  static constexpr int N = A > B ? (A > C ? A : C) : (B > C ? B : C);  // doubles per warp
};

#define K3W_WARPS 4
template <class M>
__global__ void __launch_bounds__(32 * K3W_WARPS) k_node_w(const KParams P, int64_t Np, int64_t Nn,
                                                          const double* __restrict__ y_pairs,
                                                          const double* __restrict__ theta_vecs, double delta, double eps,
                                                          double* __restrict__ psi, double* __restrict__ psi_jac,
                                                          double* __restrict__ th, double* __restrict__ th_jac,
                                                          double* __restrict__ imp, double* __restrict__ imp_jac,
                                                          const ZSrc zs) {
  using T = NodeTile<M>;
  constexpr int NC = M::NC, NQ = T::NQ, NY = T::NY, NPSI = T::NPSI, NV = T::NV, NI = T::NI;
  constexpr int NXT = 2 * NQ + NY;
  constexpr NodeDirs<M> DIRC{};  // compile-time counts
  const NodeDirs<M>& DIRS = kNodeDirs<M>;
  extern __shared__ __align__(16) double k3_tile[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* tile = k3_tile + (size_t)wib * T::N;
  if (zs.de) {  // relaxation parameters from device memory (CUDA-graph replays)
    delta = zs.de[0];
    eps = zs.de[1];
  }
  // warp order: impulse items, theta items, psi items -- the heaviest first, so the
  // light ones fill the tail of the launch
  const int64_t w = (int64_t)blockIdx.x * K3W_WARPS + wib;
  if (w >= 2 * Nn) {  // psi of interval k: 2 NY directions, all live (ocp.py:277-287)
    const int64_t k = w - 2 * Nn;
    if (k >= Np) return;
    const double* ya = y_pairs + k * 2 * NY;
    const double* yb = ya + NY;
    if (zs.z) {
      const double* zb = zs.z + (k / zs.n_int) * zs.zstride;
      const int64_t kk = k % zs.n_int;
      ya = zb + (2 * kk + 1) * NXT + 2 * NQ;
      yb = zb + (2 * kk + 2) * NXT + 2 * NQ;
    }
    for (int d = lane; d < 2 * NY; d += 32)
      node_psi<M>(P, ya, yb, d, delta, eps, d == 0 ? psi + k * NPSI : nullptr, tile + d, 2 * NY);
    __syncwarp();
    double* dst = psi_jac + k * T::A;
    for (int e = lane; e < T::A; e += 32) dst[e] = tile[e];
    return;
  }
  const bool is_th = w >= Nn;
  const int64_t k = is_th ? w - Nn : w;
  NodeIn x{theta_vecs + k * NV, theta_vecs + k * NV + 2 * NQ, theta_vecs + k * NV + 3 * NQ, 2 * NQ, 3 * NQ, 0};
  if (zs.z) {
    const double* zb = zs.z + (k / zs.n_node) * zs.zstride;
    const int64_t kk = k % zs.n_node;
    x.p0 = zb + 2 * kk * NXT;
    x.p1 = zb + (2 * kk + 1) * NXT + NQ;
    x.p2 = zb + zs.base_p + 3 * NC * kk;
  }
  if (is_th) {
    if constexpr (NC > 0) {
      constexpr int NCOL = NV, NROW = 6 * NC;
      for (int e = lane; e < NROW * NCOL; e += 32) tile[e] = 0.0;  // structural zeros
      __syncwarp();
      for (int i = lane; i < DIRC.n_th; i += 32) {
        x.dir = DIRS.th[i];
        node_theta<M>(P, x, delta, i == 0 ? th + k * NROW : nullptr, tile + x.dir, NCOL);
      }
      __syncwarp();
      double* dst = th_jac + k * T::B;
      for (int e = lane; e < T::B; e += 32) dst[e] = tile[e];
    }
  } else {
    constexpr int NCOL = NI, NROW = NQ;
    for (int e = lane; e < NROW * NCOL; e += 32) {
      const int r = e / NCOL, c = e % NCOL;
      tile[e] = (c == 2 * NQ + r) ? 1.0 : 0.0;  // d(v+ - impact_map)/dv+ = I; other dead columns 0
    }
    __syncwarp();
    for (int i = lane; i < DIRC.n_imp; i += 32) {
      x.dir = DIRS.imp[i];
      node_impulse<M>(P, x, i == 0 ? imp + k * NQ : nullptr, tile + x.dir, NCOL);
    }
    __syncwarp();
    double* dst = imp_jac + k * T::C;
    for (int e = lane; e < T::C; e += 32) dst[e] = tile[e];
  }
}
