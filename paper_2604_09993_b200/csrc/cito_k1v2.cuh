// cito_k1v2.cuh — K1 v2: the fused interval linearization with a short primal
// critical chain (one CTA per interval, fp64, sm_100a).
//
// Same mathematics as k_linearize (cito_kernels.cuh; reference
// cito.augmentation.Discretizer.linearize_batch, augmentation.py:180-242), but
// the per-stage work is split so that only the dependent chain of the RK stage
// recursion sits on the critical path:
//
//   warp 0          stage t   critical chain only: stage input (lanes own state
//                             coordinates, stage slopes in registers), sin/cos and
//                             FOH control (lane per link / control), then ONE lane
//                             runs kinematics -> forces -> Gram -> straight-line
//                             block LDL^T (generated per topology) -> joint
//                             reactions -> vdot, all in registers.
//   warps 1..NCW    stage t-3 tangent columns (one thread per column).
//   warp NCW+1      stage t-2 rate Jacobian: one lane per input direction (q, v and
//                             u; generic forward-mode tangent code, one code path).
//   warp NCW+2      stage t-1 everything off the chain: contact frames, signed
//                             distances, Omega and path rows, the y accumulators,
//                             the dS terms of the q-row stage inputs.
// (CITO_JAC_ONE_WARP=0 restores round 1's layout: separate q/v and u Jacobian warps
// with direction-kind-specialised code.)
//
// A 4-slot ring of per-stage records in shared memory carries the stage from
// role to role; one __syncthreads per tick.
#pragma once

#include "cito_kernels.cuh"


// ---------------------------------------------------------------------------
// Rate-Jacobian column of one input direction, specialised on the direction
// kind (1: q, 2: v, 3: u): the derivative of prim_rate restricted to the seed
// terms that kind can make nonzero (cito/contact_dynamics.py:86-108,
// multibody.py:285-392, augmentation.py:100-153).  Same arithmetic as tan_rate
// for the surviving terms.
template <class M, int KIND>
__device__ __forceinline__ void tan_rate_k(const KParams& P, const Prim<M>& pr, const double* v, int dir, double* out) {
  constexpr int NL = M::NL, NJ = M::NJ, NC = M::NC, NA = M::NA, NQ = 3 * NL, NX = 2 * NQ;
  constexpr bool HQ = (KIND & 1) != 0, HV = (KIND & 2) != 0, HU = (KIND & 4) != 0;
  (void)NL;
#define SQ(k) ((dir) == (k) ? 1.0 : 0.0)
#define SV(k) ((dir) == NQ + (k) ? 1.0 : 0.0)
#define SU(m) ((dir) == NX + (m) ? 1.0 : 0.0)
  double dW[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) dW[k] = 0.0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p = M::jparent(j), c = M::jchild(j), a = M::jact(j);
    double dm = 0.0;
    bool any = false;
    if constexpr (HU) {
      if (a >= 0) {
        dm = SU(a);
        any = true;
      }
    }
    if constexpr (HQ) {
      if (P.jspring[j]) {
        const double dth_p = p >= 0 ? SQ(3 * p + 2) : 0.0;
        dm = dm - P.jk[j] * (SQ(3 * c + 2) - dth_p);
        any = true;
      }
    }
    if constexpr (HV) {
      if (P.jspring[j]) {
        const double dom_p = p >= 0 ? SV(3 * p + 2) : 0.0;
        dm = dm - P.jd[j] * (SV(3 * c + 2) - dom_p);
        any = true;
      }
    }
    if (any) {
      dW[3 * c + 2] += dm;
      if (p >= 0) dW[3 * p + 2] -= dm;
    }
  }
  double dP[Pos<NC>::v][2], dn[Pos<NC>::v][2], dsd[Pos<NC>::v];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int l = M::clink(i);
    const double rx = pr.rr[i][0], rz = pr.rr[i][1];
    dP[i][0] = dP[i][1] = dn[i][0] = dn[i][1] = dsd[i] = 0.0;
    if constexpr (HQ) {
      const double dth = SQ(3 * l + 2);
      dP[i][0] = SQ(3 * l) + dth * (-rz);
      dP[i][1] = SQ(3 * l + 1) + dth * rx;
      if constexpr (M::IMPLICIT) {
        const double Hd0 = pr.H[i][0] * dP[i][0] + pr.H[i][1] * dP[i][1];
        const double Hd1 = pr.H[i][1] * dP[i][0] + pr.H[i][2] * dP[i][1];
        const double gn = pr.gn[i], g0 = pr.g[i][0], g1 = pr.g[i][1];
        const double gHd = g0 * Hd0 + g1 * Hd1;
        const double ign3 = pr.ign3[i];
        dn[i][0] = Hd0 / gn - g0 * gHd * ign3;
        dn[i][1] = Hd1 / gn - g1 * gHd * ign3;
        dsd[i] = (g0 * dP[i][0] + g1 * dP[i][1]) / gn - pr.hv[i] * gHd * ign3;
      } else {
        dsd[i] = dP[i][1];
      }
      const double ft = pr.u[NA + 2 * i], fn = pr.u[NA + 2 * i + 1];
      double dF0 = 0.0, dF1 = 0.0;
      if constexpr (M::IMPLICIT) {
        const double dt0 = dn[i][1], dt1 = -dn[i][0];
        dF0 = dt0 * ft + dn[i][0] * fn;
        dF1 = dt1 * ft + dn[i][1] * fn;
        dW[3 * l] += dF0;
        dW[3 * l + 1] += dF1;
      }
      dW[3 * l + 2] += -dth * (rx * pr.F[i][0] + rz * pr.F[i][1]) + (-rz) * dF0 + rx * dF1;
    }
    if constexpr (HU) {
      const double dft = SU(NA + 2 * i), dfn = SU(NA + 2 * i + 1);
      const double dF0 = pr.t[i][0] * dft + pr.n[i][0] * dfn;
      const double dF1 = pr.t[i][1] * dft + pr.n[i][1] * dfn;
      dW[3 * l] += dF0;
      dW[3 * l + 1] += dF1;
      dW[3 * l + 2] += (-rz) * dF0 + rx * dF1;
    }
  }
  if constexpr (NJ == 0) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      out[3 * l] = P.minv_m[l] * dW[3 * l];
      out[3 * l + 1] = P.minv_m[l] * dW[3 * l + 1];
      out[3 * l + 2] = P.minv_I[l] * dW[3 * l + 2];
    }
  } else {
    constexpr int NJ2 = 2 * NJ;
    if constexpr (HQ) {  // g = dW + dJ^T lam (theta coordinates only)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int sa = 0; sa < 2; ++sa) {
          const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
          if (l < 0) continue;
          const double sgn = sa == 0 ? 1.0 : -1.0;
          const double* R = sa == 0 ? pr.rp[j] : pr.rc[j];
          dW[3 * l + 2] += sgn * (-SQ(3 * l + 2)) * (R[0] * pr.lam[2 * j] + R[1] * pr.lam[2 * j + 1]);
        }
    }
    // rhs' = dJ vdot + J M^-1 g + dcurv, directly in elimination order
    double zp[NJ2];
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      const int j = M::jperm(a);
#pragma unroll
      for (int al = 0; al < 2; ++al) {
        double acc = 0.0;
#pragma unroll
        for (int sa = 0; sa < 2; ++sa) {
          const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
          if (l < 0) continue;
          const double sgn = sa == 0 ? 1.0 : -1.0;
          const double* R = sa == 0 ? pr.rp[j] : pr.rc[j];
          const double dPa = al == 0 ? -R[1] : R[0];
          const double w = v[3 * l + 2];
          double term = P.minv_m[l] * dW[3 * l + al] + dPa * P.minv_I[l] * dW[3 * l + 2];
          if constexpr (HQ) {
            const double dth = SQ(3 * l + 2);
            term = -dth * R[al] * pr.vdot[3 * l + 2] + term - dth * dPa * w * w;
          }
          if constexpr (HV) term = term - 2.0 * R[al] * w * SV(3 * l + 2);
          acc += sgn * term;
        }
        zp[2 * a + al] = acc;
      }
    }
    M::tri_solve(pr.L, pr.Li, zp);  // generated straight-line sparse solves (gen_models.py)
    // dvdot = M^-1 (g + J^T dlam), dlam = -z (joint order)
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      const int j = M::jperm(a);
#pragma unroll
      for (int sa = 0; sa < 2; ++sa) {
        const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
        if (l < 0) continue;
        const double sgn = sa == 0 ? 1.0 : -1.0;
        const double* R = sa == 0 ? pr.rp[j] : pr.rc[j];
        const double l0 = -zp[2 * a], l1 = -zp[2 * a + 1];
        dW[3 * l] += sgn * l0;
        dW[3 * l + 1] += sgn * l1;
        dW[3 * l + 2] += sgn * ((-R[1]) * l0 + R[0] * l1);
      }
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      out[3 * l] = P.minv_m[l] * dW[3 * l];
      out[3 * l + 1] = P.minv_m[l] * dW[3 * l + 1];
      out[3 * l + 2] = P.minv_I[l] * dW[3 * l + 2];
    }
  }
  // d Omega (aux_rate, augmentation.py:134-153)
  double* dy = out + NQ;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int l = M::clink(i);
    const double ft = pr.u[NA + 2 * i], fn = pr.u[NA + 2 * i + 1], gam = pr.u[NA + 2 * NC + i];
    const double rx = pr.rr[i][0], rz = pr.rr[i][1];
    const double w = v[3 * l + 2];
    double dlamc = 0.0;
    if constexpr (HQ || HV) {
      double dJv0 = 0.0, dJv1 = 0.0, dvt = 0.0;
      if constexpr (HQ) {
        const double dth = SQ(3 * l + 2);
        dJv0 = -dth * rx * w;
        dJv1 = -dth * rz * w;
        if constexpr (M::IMPLICIT) dvt = (dn[i][1]) * pr.Jv[i][0] + (-dn[i][0]) * pr.Jv[i][1];
      }
      if constexpr (HV) {
        const double dw = SV(3 * l + 2);
        dJv0 += SV(3 * l) + (-rz) * dw;
        dJv1 += SV(3 * l + 1) + rx * dw;
      }
      dvt += pr.t[i][0] * dJv0 + pr.t[i][1] * dJv1;
      dlamc = dvt;
    }
    if constexpr (HU) {
      const double dft = SU(NA + 2 * i), dgam = SU(NA + 2 * NC + i);
      const double dsg = dft * pr.dsgf[i];
      dlamc += dgam * pr.sg[i] + gam * dsg;
    }
    dy[5 * i + 0] = HU ? SU(NA + 2 * i + 1) : 0.0;
    dy[5 * i + 1] = pr.dlam[i] * dlamc;
    dy[5 * i + 2] = HU ? SU(NA + 2 * NC + i) : 0.0;
    if constexpr (HU) {
      const double dft = SU(NA + 2 * i), dfn = SU(NA + 2 * i + 1);
      dy[5 * i + 3] = pr.dmu[i] * dfn - pr.sg[i] * dft;
    } else {
      dy[5 * i + 3] = 0.0;
    }
    dy[5 * i + 4] = HQ ? pr.dsrl[i] * dsd[i] : 0.0;
  }
  if constexpr (M::NGO > 0) {
    constexpr int NG = Prim<M>::NG;
    if constexpr (HQ) {
      double dg[Pos<NG>::v];
      int r = 0;
#pragma unroll
      for (int i = 0; i < NC; ++i) dg[r++] = -dsd[i];
#pragma unroll
      for (int k = 0; k < M::NJL; ++k) {
        const int jj = M::jl_joint(k);
        const int p = M::jparent(jj), c = M::jchild(jj);
        const double drel = SQ(3 * c + 2) - (p >= 0 ? SQ(3 * p + 2) : 0.0);
        dg[r++] = drel;
        dg[r++] = -drel;
      }
#pragma unroll
      for (int k = 0; k < M::NHB; ++k) {
        const double dpz = SQ(3 * M::hb_link(k) + 1);
        dg[r++] = -dpz;
        dg[r++] = dpz;
      }
#pragma unroll
      for (int jg = 0; jg < NG; ++jg) dg[jg] *= pr.dgp[jg];
#pragma unroll
      for (int o = 0; o < M::NGO; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int jg = 0; jg < NG; ++jg) acc += P.mix[o][jg] * dg[jg];
        dy[5 * NC + o] = acc;
      }
    } else {
#pragma unroll
      for (int o = 0; o < M::NGO; ++o) dy[5 * NC + o] = 0.0;
    }
  }
#undef SQ
#undef SV
#undef SU
}

// ---------------------------------------------------------------------------
template <class M>
struct Rec2 {
  Prim<M> pr;
  double xs[Dims<M>::NX];  // stage input (q, v)
  double r[Dims<M>::NR];   // unscaled rate rows: vdot (NQ), Omega (NY)
  double wq[3 * M::NL];    // sum_j h a_ij v_{s,j}: dS term of the q-row stage inputs
};

#ifndef CITO_JAC_ONE_WARP
// 2 (default): every rate-Jacobian direction (q, v and u: 32 for HalfCheetah) on ONE
// warp with the generic tangent code (kind 7), one warp fewer per CTA; 1: the same
// with the u-Jacobian warp kept idle (what was measured as "2" while this default
// stood after K2Dims: 0.108 vs 0.114 ms for 29 intervals against 0; the real 5-warp
// CTA: 0.087 vs 0.089 ms, same box); 0: q/v and u directions on two warps
// (specialised kinds 3 and 4).  Defined before K2Dims, which sizes the CTA from it.
#define CITO_JAC_ONE_WARP 2
#endif
template <class M>
struct K2Dims {
  using D = Dims<M>;
  static constexpr int NCW = (D::NCOL + 31) / 32;
  // warp roles, ordered so the heavy roles (primal, columns, rate Jacobian) sit on
  // distinct SM sub-partitions (warp w -> SMSP w % 4): 0 primal, 1..NCW columns, then
  // the rate Jacobian and the off-chain aux warp (+ the u-Jacobian warp in the
  // CITO_JAC_ONE_WARP=0/1 layouts)
#if CITO_JAC_ONE_WARP == 2
  static constexpr int W_COL0 = 1, W_JQV = 1 + NCW, W_AUX = 2 + NCW, W_JU = -1;
  static constexpr int NT = 32 * (3 + NCW);
#else
  static constexpr int W_COL0 = 1, W_JQV = 1 + NCW, W_AUX = 2 + NCW, W_JU = 3 + NCW;
  static constexpr int NT = 32 * (4 + NCW);
#endif
  static constexpr int NX = D::NX;
  static constexpr int PER = (NX + 31) / 32;  // state coordinates per lane of warp 0
};

// Per-thread state that lives across ticks, one union for all roles (each thread
// has exactly one role, so the roles share the same registers): warp 0 = state
// coordinates + stage slopes, aux = stage velocities + y accumulator/row,
// columns = substep-start tangents of the history coordinates.
template <class M>
struct RegState {
  static constexpr int PER = (Dims<M>::NX + 31) / 32;
  static constexpr int NH = Pos<M::NHIST>::v;
  static constexpr int NPU = Pos<M::NPUSH>::v, NYR = Pos<5 * M::NC + M::NGO>::v;
  static constexpr int a = 7 * PER, b = 8, c = 2 * NH + 2 * NPU + NYR;  // columns: history, push rows, y rows
  static constexpr int N = a > b ? (a > c ? a : c) : (b > c ? b : c);
};
#define RS_XR(p) rs[(p)]
#define RS_KR(j, p) rs[PER + (j) * PER + (p)]
#define RS_VS(j) rs[(j)]
#define RS_KY rs[6]
#define RS_YV rs[7]
#define RS_HQ(h) rs[(h)]
#define RS_HV(h) rs[RegState<M>::NH + (h)]
#ifndef CITO_COL_SMEM
#define CITO_COL_SMEM 0  // A/B: 1 = y-row accumulators in shared memory, 2 = + push rows
#endif
#if CITO_COL_SMEM >= 2
#define RS_PQ(p) sh.PQ[(p)][col]
#define RS_PV(p) sh.PV[(p)][col]
#else
#define RS_PQ(p) rs[2 * RegState<M>::NH + (p)]
#define RS_PV(p) rs[2 * RegState<M>::NH + RegState<M>::NPU + (p)]
#endif
#if CITO_COL_SMEM >= 1
#define RS_DY(k) sh.DY[(k)][col]
#else
#define RS_DY(k) rs[2 * RegState<M>::NH + 2 * RegState<M>::NPU + (k)]
#endif

template <class M>
struct AuxScratch {
  static constexpr int NG = Prim<M>::NG;
  double sgv[Pos<NG>::v];
};

template <class M>
struct Fused2Shared {
  using D = Dims<M>;
  Rec2<M> ring[4];
  SParams<M> sp;
  AuxScratch<M> ax;
  double At[2][D::NDIR][D::NRP];
  double KV[5][D::NH][D::NCOLP];
  double PQ[Pos<M::NPUSH>::v][D::NCOLP];
  double PV[Pos<M::NPUSH>::v][D::NCOLP];
  double DY[Pos<D::NY>::v][D::NCOLP];
  double x[D::NXT];
  double xn[D::NXT];  // the next interval's start state (defects), loaded with the inputs
  double vbs[2][D::NQ];
  double U[2 * D::NU + 1];
  double S;
  int bad;
};

// Accumulate into `a`, the first contribution assigned rather than added to 0.0
// (with every loop unrolled the `set` flags are compile-time constants, so the
// chain carries no "0.0 + x" additions; only the sign of an exact zero differs).
__device__ __forceinline__ void acc_add(double& a, bool& set, double x) {
  if (set) {
    a += x;
  } else {
    a = x;
    set = true;
  }
}

// Lane-0 critical chain of one rate evaluation: forces, Gram matrix, sparse
// Cholesky (generated straight-line code, M::chol_solve), joint reactions,
// vdot (cito/contact_dynamics.py:86-108, multibody.py:259-321).  Reads the
// stage input, cos/sin and FOH control of the record; writes the factor, the
// reactions and vdot (pr.vdot and the vdot rows of r).
template <class M>
__device__ __forceinline__ void crit_chain(const KParams& P, Rec2<M>& R, int t) {
  (void)t;
  using D = Dims<M>;
  constexpr int NL = M::NL, NJ = M::NJ, NC = M::NC, NA = M::NA, NQ = D::NQ;
  Prim<M>& pr = R.pr;
  const double* q = R.xs;
  const double* v = R.xs + NQ;
  double cl[NL], sl[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    cl[l] = pr.c[l];
    sl[l] = pr.s[l];
  }
  double W[NQ];
  bool Ws[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) {
    W[k] = 0.0;
    Ws[k] = false;
  }
#pragma unroll
  for (int l = 0; l < NL; ++l) acc_add(W[3 * l + 1], Ws[3 * l + 1], P.neg_mg[l]);
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p = M::jparent(j), c = M::jchild(j), a = M::jact(j);
    double mo = a >= 0 ? pr.u[a] : 0.0;
    if (P.jspring[j]) {
      const double th_p = p >= 0 ? q[3 * p + 2] : 0.0;
      const double om_p = p >= 0 ? v[3 * p + 2] : 0.0;
      const double rel = q[3 * c + 2] - th_p - P.jrest[j];
      mo = mo - P.jk[j] * rel - P.jd[j] * (v[3 * c + 2] - om_p);
    }
    acc_add(W[3 * c + 2], Ws[3 * c + 2], mo);
    if (p >= 0) acc_add(W[3 * p + 2], Ws[3 * p + 2], -mo);
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int l = M::clink(i);
    const double rx = cl[l] * P.cr[i][0] - sl[l] * P.cr[i][1];
    const double rz = sl[l] * P.cr[i][0] + cl[l] * P.cr[i][1];
    double n0, n1;
    if constexpr (M::IMPLICIT) {
      const T2 t2 = surface_t2(P, q[3 * l] + rx, q[3 * l + 1] + rz);
      const double gn = sqrt(t2.gx * t2.gx + t2.gz * t2.gz);
      n0 = t2.gx / gn;
      n1 = t2.gz / gn;
    } else {
      n0 = 0.0;
      n1 = 1.0;
    }
    const double t0 = n1, t1 = -n0;
    const double ft = pr.u[NA + 2 * i], fn = pr.u[NA + 2 * i + 1];
    const double F0 = t0 * ft + n0 * fn, F1 = t1 * ft + n1 * fn;
    acc_add(W[3 * l], Ws[3 * l], F0);
    acc_add(W[3 * l + 1], Ws[3 * l + 1], F1);
    acc_add(W[3 * l + 2], Ws[3 * l + 2], (-rz) * F0 + rx * F1);
  }
  double* vdot = R.r;
  if constexpr (NJ == 0) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      vdot[3 * l] = P.minv_m[l] * W[3 * l];
      vdot[3 * l + 1] = P.minv_m[l] * W[3 * l + 1];
      const double vd2 = P.minv_I[l] * W[3 * l + 2];
      vdot[3 * l + 2] = vd2;
      pr.vdot[3 * l + 2] = vd2;
    }
  } else {
    constexpr int NJ2 = 2 * NJ;
    double Rj[NJ][2][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int p = M::jparent(j), c = M::jchild(j);
      if (p >= 0) {
        Rj[j][0][0] = cl[p] * P.jrp[j][0] - sl[p] * P.jrp[j][1];
        Rj[j][0][1] = sl[p] * P.jrp[j][0] + cl[p] * P.jrp[j][1];
      } else {
        Rj[j][0][0] = Rj[j][0][1] = 0.0;
      }
      Rj[j][1][0] = cl[c] * P.jrc[j][0] - sl[c] * P.jrc[j][1];
      Rj[j][1][1] = sl[c] * P.jrc[j][0] + cl[c] * P.jrc[j][1];
    }
    CITO_MARK_P(t, 3);  // kinematics + forces done
    double Lr[NJ2 * (NJ2 + 1) / 2];
#pragma unroll
    for (int a = 0; a < NJ; ++a)
#pragma unroll
      for (int bp = 0; bp <= a; ++bp) {
        if (!M::lnzb(a, bp)) continue;
        const int j = M::jperm(a), k = M::jperm(bp);
        double g00 = 0.0, g01 = 0.0, g10 = 0.0, g11 = 0.0;
        bool gs = false, gs01 = false, gs10 = false, gs11 = false;
#pragma unroll
        for (int sa = 0; sa < 2; ++sa)
#pragma unroll
          for (int sb = 0; sb < 2; ++sb) {
            const int la = sa == 0 ? M::jparent(j) : M::jchild(j);
            const int lb = sb == 0 ? M::jparent(k) : M::jchild(k);
            if (la < 0 || la != lb) continue;
            const double sg = (sa == sb) ? 1.0 : -1.0;
            const double dA0 = -Rj[j][sa][1], dA1 = Rj[j][sa][0], dB0 = -Rj[k][sb][1], dB1 = Rj[k][sb][0];
            const double mI = P.minv_I[la], mm = P.minv_m[la];
            acc_add(g00, gs, sg * (dA0 * dB0 * mI + mm));
            acc_add(g01, gs01, sg * (dA0 * dB1 * mI));
            acc_add(g10, gs10, sg * (dA1 * dB0 * mI));
            acc_add(g11, gs11, sg * (dA1 * dB1 * mI + mm));
          }
        Lr[LI(2 * a, 2 * bp)] = g00;
        Lr[LI(2 * a + 1, 2 * bp)] = g10;
        Lr[LI(2 * a + 1, 2 * bp + 1)] = g11;
        if (a != bp) Lr[LI(2 * a, 2 * bp + 1)] = g01;
      }
    double y[NJ2];
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      const int j = M::jperm(a);
#pragma unroll
      for (int al = 0; al < 2; ++al) {
        double acc = 0.0;
        bool as = false;
#pragma unroll
        for (int sa = 0; sa < 2; ++sa) {
          const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
          if (l < 0) continue;
          const double sgn = sa == 0 ? 1.0 : -1.0;
          const double dP = al == 0 ? -Rj[j][sa][1] : Rj[j][sa][0];
          const double om = v[3 * l + 2];
          acc_add(acc, as,
                  sgn * (P.minv_m[l] * W[3 * l + al] + dP * P.minv_I[l] * W[3 * l + 2] - Rj[j][sa][al] * om * om));
        }
        y[2 * a + al] = acc;
      }
    }
    double Lir[NJ2];
    CITO_MARK_P(t, 4);  // Gram + rhs done
    M::chol_solve(Lr, y, Lir);
    CITO_MARK_P(t, 5);  // factor + solves done
#pragma unroll
    for (int r = 0; r < NJ2; ++r) {
      pr.Li[r] = Lir[r];
#pragma unroll
      for (int c = 0; c <= r; ++c)
        if (M::lnzb(r / 2, c / 2)) pr.L[LI(r, c)] = Lr[LI(r, c)];
    }
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      const int j = M::jperm(a);
      const double l0 = -y[2 * a], l1 = -y[2 * a + 1];
      pr.lam[2 * j] = l0;
      pr.lam[2 * j + 1] = l1;
#pragma unroll
      for (int sa = 0; sa < 2; ++sa) {
        const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
        if (l < 0) continue;
        const double sgn = sa == 0 ? 1.0 : -1.0;
        W[3 * l] += sgn * l0;
        W[3 * l + 1] += sgn * l1;
        W[3 * l + 2] += sgn * ((-Rj[j][sa][1]) * l0 + Rj[j][sa][0] * l1);
      }
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      vdot[3 * l] = P.minv_m[l] * W[3 * l];
      vdot[3 * l + 1] = P.minv_m[l] * W[3 * l + 1];
      const double vd2 = P.minv_I[l] * W[3 * l + 2];
      vdot[3 * l + 2] = vd2;
      pr.vdot[3 * l + 2] = vd2;
    }
  }
}

// Warp 1: everything of stage `a` that is off the critical chain.
template <class M>
__device__ __forceinline__ void aux_stage(const KParams& P, Fused2Shared<M>& sh, int a, int lane,
                                          double (&rs)[RegState<M>::N]) {
  using D = Dims<M>;
  constexpr int NL = M::NL, NJ = M::NJ, NC = M::NC, NA = M::NA, NQ = D::NQ, NY = D::NY;
  const int s = a / 6, i = a % 6;
  Rec2<M>& R = sh.ring[a & 3];
  Prim<M>& pr = R.pr;
  const SParams<M>& Q = sh.sp;
  const double* q = R.xs;
  const double* v = R.xs + NQ;
  const double S = sh.S, h = P.h;
  (void)NL;
  // 1: rotated joint anchors (per joint side), contact frames / forces / Omega (per contact)
  for (int e = lane; e < 2 * NJ + NC; e += 32) {
    if (e < 2 * NJ) {
      const int j = e >> 1, side = e & 1;
      const int l = side ? Q.jc[j] : Q.jp[j];
      if (l >= 0) {
        const double ax = side ? Q.jrc[j][0] : Q.jrp[j][0], az = side ? Q.jrc[j][1] : Q.jrp[j][1];
        const double c = pr.c[l], sn = pr.s[l];
        double* Rj = side ? pr.rc[j] : pr.rp[j];
        Rj[0] = c * ax - sn * az;
        Rj[1] = sn * ax + c * az;
      }
    } else {
      const int ci = e - 2 * NJ, l = Q.cl[ci];
      const double c = pr.c[l], sn = pr.s[l];
      const double rx = c * Q.cr[ci][0] - sn * Q.cr[ci][1];
      const double rz = sn * Q.cr[ci][0] + c * Q.cr[ci][1];
      pr.rr[ci][0] = rx;
      pr.rr[ci][1] = rz;
      const double Px = q[3 * l] + rx, Pz = q[3 * l + 1] + rz;
      double n0, n1, sd;
      if constexpr (M::IMPLICIT) {
        T2 t2 = surface_t2(P, Px, Pz);
        pr.hv[ci] = t2.v;
        pr.g[ci][0] = t2.gx;
        pr.g[ci][1] = t2.gz;
        pr.H[ci][0] = t2.hxx;
        pr.H[ci][1] = t2.hxz;
        pr.H[ci][2] = t2.hzz;
        const double gn = sqrt(t2.gx * t2.gx + t2.gz * t2.gz);
        pr.gn[ci] = gn;
        pr.ign3[ci] = 1.0 / (gn * gn * gn);
        n0 = t2.gx / gn;
        n1 = t2.gz / gn;
        sd = t2.v / gn;
      } else {
        n0 = 0.0;
        n1 = 1.0;
        sd = Pz - P.height;
      }
      pr.sd[ci] = sd;
      const double t0 = n1, t1 = -n0;
      pr.n[ci][0] = n0;
      pr.n[ci][1] = n1;
      pr.t[ci][0] = t0;
      pr.t[ci][1] = t1;
      const double ft = pr.u[NA + 2 * ci], fn = pr.u[NA + 2 * ci + 1], gam = pr.u[NA + 2 * NC + ci];
      pr.F[ci][0] = t0 * ft + n0 * fn;
      pr.F[ci][1] = t1 * ft + n1 * fn;
      const double om = v[3 * l + 2];
      const double Jv0 = v[3 * l] + (-rz) * om, Jv1 = v[3 * l + 1] + rx * om;
      pr.Jv[ci][0] = Jv0;
      pr.Jv[ci][1] = Jv1;
      const double q1 = ft * ft + 1.0, sq1 = sqrt(q1);
      const double sgt = ft / sq1;  // friction_stationarity (contact_dynamics.py:55-66)
      pr.sg[ci] = sgt;
      pr.dsgf[ci] = 1.0 / (q1 * sq1);
      const double lamc = t0 * Jv0 + t1 * Jv1 + gam * sgt;
      pr.lamc[ci] = lamc;
      pr.dlam[ci] = sabs_d(lamc);
      pr.dmu[ci] = sabs_d(Q.mu[ci] * fn) * Q.mu[ci];
      pr.dsrl[ci] = srelu_d(sd);
      double* yo = R.r + NQ + 5 * ci;  // aux_rate rows (augmentation.py:134-153)
      yo[0] = fn;
      yo[1] = sabs(lamc);
      yo[2] = gam;
      yo[3] = sabs(Q.mu[ci] * fn) - sabs(ft);
      yo[4] = srelu(sd);
    }
  }
  __syncwarp();
  if constexpr (M::NGO > 0) {  // path rows g(x, u) (augmentation.py:112-129) and their mixing
    constexpr int NG = Prim<M>::NG;
    if (lane == 0) {
      double gpl[Pos<NG>::v];
      int r = 0;
#pragma unroll
      for (int ci = 0; ci < NC; ++ci) gpl[r++] = -pr.sd[ci];
#pragma unroll
      for (int k = 0; k < M::NJL; ++k) {
        const int jj = M::jl_joint(k);
        const int p = M::jparent(jj), c = M::jchild(jj);
        const double rel = q[3 * c + 2] - (p >= 0 ? q[3 * p + 2] : 0.0);
        gpl[r++] = rel - P.jl_hi[k];
        gpl[r++] = P.jl_lo[k] - rel;
      }
#pragma unroll
      for (int k = 0; k < M::NHB; ++k) {
        const double pz = q[3 * M::hb_link(k) + 1];
        gpl[r++] = P.hb_lo[k] - pz;
        gpl[r++] = pz - P.hb_hi[k];
      }
      double sgv[Pos<NG>::v];
#pragma unroll
      for (int jg = 0; jg < NG; ++jg) {
        pr.gp[jg] = gpl[jg];
        pr.dgp[jg] = srelu_d(gpl[jg]);
        sgv[jg] = srelu(gpl[jg]);
      }
#pragma unroll
      for (int o = 0; o < M::NGO; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int jg = 0; jg < NG; ++jg) acc += P.mix[o][jg] * sgv[jg];
        R.r[NQ + 5 * NC + o] = acc;
      }
    }
    __syncwarp();
  }
  // 2: y accumulators (augmentation.py:206-209), dS terms of the q-row stage inputs
  if (lane < NY) {
    RS_KY = (i == 0 ? 0.0 : RS_KY) + P.b[i] * (S * R.r[NQ + lane]);
    if (i == 5) RS_YV = RS_YV + h * RS_KY;
  }
  if (lane < NQ) {
    const double vsk = v[lane];
    double ws = 0.0;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      if (j == i) RS_VS(j) = vsk;
      if (j < i) ws += P.ha[i][j] * RS_VS(j);
    }
    if (i == 5) RS_VS(5) = vsk;
    R.wq[lane] = ws;
    if (i == 5) {
      double w2 = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) w2 += P.b[j] * RS_VS(j);
      sh.vbs[s & 1][lane] = h * w2;
    }
  }
}

// One tangent column through RK stage I (record R, rate Jacobian At).
template <class M>
__device__ __forceinline__ void col_stage2(const KParams& P, Fused2Shared<M>& sh, const Rec2<M>& R,
                                           const double (*At)[Dims<M>::NRP], int s, const int I, int col, double S,
                                           double dS, bool isU, int um, bool uplus, double (&rs)[RegState<M>::N]) {
  using D = Dims<M>;
  constexpr int NQ = D::NQ, NR = D::NR, NDIRX = M::NDIRX;
  const double h = P.h;
  const double tau = h * (double)s + P.ch[I];
  const double hb = h * P.b[I];
  if (I == 0) {
#pragma unroll
    for (int p = 0; p < M::NPUSH; ++p) RS_PQ(p) += P.he1 * S * RS_PV(p);
  }
  // stage coefficients, once per tick (warp-uniform): S h^2 sum a a (q rows), h a (v rows)
  // stage-input tangents along the rate-Jacobian directions: base value, then the
  // history terms in stage order (a runtime loop of I steps over all directions:
  // no predicated dead terms, one small loop body)
  const double shc = S * P.hc1[I];
  double vals[Pos<NDIRX>::v];
#pragma unroll
  for (int kd = 0; kd < NDIRX; ++kd) {
    const int d = M::dir(kd);
    if (d < NQ) {
      const int hs = M::hslot(d);
      vals[kd] = RS_HQ(hs) + shc * RS_HV(hs) + dS * R.wq[d];
    } else {
      vals[kd] = RS_HV(M::hslot(d - NQ));
    }
  }
#pragma unroll 1
  for (int l = 0; l < I; ++l) {
    const double cq = S * P.cq[I][l], ca = P.ha[I][l];
#pragma unroll
    for (int kd = 0; kd < NDIRX; ++kd) {
      const int d = M::dir(kd);
      const int hs = M::hslot(d < NQ ? d : d - NQ);
      vals[kd] += (d < NQ ? cq : ca) * sh.KV[l][hs][col];
    }
  }
  const double coef = uplus ? tau : (1.0 - tau);
  // rate rows in chunks of RC so the accumulators of one chunk, the stage-input
  // tangents and the column state fit the register budget (3 CTAs/SM variant)
  constexpr int RC = CITO_COL_RC, NCH = (NR + RC - 1) / RC;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const int r0 = ch * RC;
    double accs[RC];
#pragma unroll
    for (int j = 0; j < RC; ++j) accs[j] = (isU && r0 + j < NR) ? At[NDIRX + um][r0 + j] * coef : 0.0;
#pragma unroll
    for (int kd = 0; kd < NDIRX; ++kd) {
      const double vk = vals[kd];
#pragma unroll
      for (int j = 0; j < RC; ++j)
        if (r0 + j < NR && M::adep(r0 + j, kd)) accs[j] += At[kd][r0 + j] * vk;
    }
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      const int rr = r0 + j;
      if (rr >= NR) break;
      const double dk = S * accs[j] + dS * R.r[rr];  // dS = 1 for the dilation column only
      if (rr < NQ) {
        const int hs = M::hslot(rr);
        if (hs >= 0) {
          if (I < 5) {
            sh.KV[I][hs][col] = dk;
          } else {
            double incv = P.b[5] * dk, incq = 0.0;
#pragma unroll
            for (int l = 0; l < 5; ++l) {
              const double kv = sh.KV[l][hs][col];
              incv += P.b[l] * kv;
              incq += P.e2[l] * kv;
            }
            RS_HQ(hs) = RS_HQ(hs) + P.he1 * S * RS_HV(hs) + S * incq + dS * sh.vbs[s & 1][rr];
            RS_HV(hs) = RS_HV(hs) + h * incv;
          }
        } else {
          const int p = M::pslot(rr);
          RS_PV(p) += hb * dk;
          RS_PQ(p) += S * P.e2[I] * dk + dS * hb * R.xs[NQ + rr];
        }
      } else {
        RS_DY(rr - NQ) += hb * dk;
      }
    }
  }
}

// JAC = false: the primal flow only (propagate for small batches): warps 0 and 1
// (critical chain + off-chain aux for the y rows), end states + finite flags.
template <class M, int MINB, bool JAC = true>
__global__ void __launch_bounds__(JAC ? K2Dims<M>::NT : 64, MINB) k_linearize2(const KParams P, int64_t B,
                                                                    const double* __restrict__ xt0s,
                                                                    const double* __restrict__ Us,
                                                                    const double* __restrict__ Ss,
                                                                    double* __restrict__ ends, double* __restrict__ jx,
                                                                    double* __restrict__ ju, double* __restrict__ js,
                                                                    int32_t* __restrict__ bad, const ZSrc zs) {
  using D = Dims<M>;
  using K = K2Dims<M>;
  constexpr int NQ = D::NQ, NX = D::NX, NU = D::NU, NY = D::NY, NXT = D::NXT, NCOL = D::NCOL;
  constexpr int NDIRX = M::NDIRX, NDIR = D::NDIR, PER = K::PER;
  static_assert(NQ <= 32 && NY <= 32, "aux warp owns one q coordinate and one y row per lane");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Fused2Shared<M>& sh = *reinterpret_cast<Fused2Shared<M>*>(smem_raw);
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  // programmatic dependent launch: a kernel enqueued after this one with the PDL attribute
  // (the CSC compaction) may start its independent prologue now; it waits for this grid's
  // completion and memory before reading any result (griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;");
#ifdef CITO_PROF
  if (g_cito_prof && blockIdx.x == 0 && threadIdx.x == 0) g_cito_prof[1664] = clock64();
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // model constants first: they do not depend on the producer of the inputs
  for (int j = tid; j < M::NJ; j += blockDim.x) {
    sh.sp.jrp[j][0] = P.jrp[j][0];
    sh.sp.jrp[j][1] = P.jrp[j][1];
    sh.sp.jrc[j][0] = P.jrc[j][0];
    sh.sp.jrc[j][1] = P.jrc[j][1];
    sh.sp.jp[j] = M::jparent(j);
    sh.sp.jc[j] = M::jchild(j);
  }
  for (int c = tid; c < M::NC; c += blockDim.x) {
    sh.sp.cr[c][0] = P.cr[c][0];
    sh.sp.cr[c][1] = P.cr[c][1];
    sh.sp.mu[c] = P.mu[c];
    sh.sp.cl[c] = M::clink(c);
  }
  // launched with programmatic dependent launch behind the kernel that uploads z (the
  // SCP-iteration graph): everything above overlapped it; the inputs are read only
  // after its completion (a no-op for a normal launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t zp = zs.z ? b / zs.n_int : 0, zk = zs.z ? b % zs.n_int : 0;
  const double* zb = zs.z ? zs.z + zp * zs.zstride : nullptr;
  const double* src_x = zs.z ? zb + (2 * zk + 1) * NXT : xt0s + b * NXT;
  const double* src_U = zs.z ? zb + zs.base_u + zk * (2 * NU + 1) : Us + b * 2 * NU;
  for (int k = tid; k < 2 * NU; k += blockDim.x) sh.U[k] = src_U[k];
  // z may live in page-locked host memory: every read of it is issued here, at once
  if (zs.defects)
    for (int k = tid; k < NXT; k += blockDim.x) sh.xn[k] = zb[(2 * zk + 2) * NXT + k];
  if (tid == 0) {
    sh.S = zs.z ? src_U[2 * NU] : Ss[b];
    sh.bad = 0;
  }
  // warp 0: state coordinates (lane + 32 p) and their stage slopes in registers
  double rs[RegState<M>::N];
#pragma unroll
  for (int k = 0; k < RegState<M>::N; ++k) rs[k] = 0.0;
  if (warp == 0) {
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int k = lane + 32 * p;
      RS_XR(p) = k < NX ? src_x[k] : 0.0;
    }
  }
  // warp 1: y row `lane` and the stage velocities of q coordinate `lane`
  constexpr int W_AUX = JAC ? K::W_AUX : 1;
  if (warp == W_AUX && lane < NY) RS_YV = src_x[NX + lane];
  // column threads
  const int col = tid - 32 * K::W_COL0;
  const bool colthr = JAC && warp >= K::W_COL0 && warp < K::W_COL0 + K::NCW && col < NCOL;
  const double dS = (col == NCOL - 1) ? 1.0 : 0.0;
  const int sc = (col >= 0 && col < M::NHCOL) ? M::hcol(col) : -1;
  const int uj = col - M::NHCOL;
  const bool isU = (uj >= 0) && (uj < 2 * NU);
  const int um = isU ? (uj % Pos<NU>::v) : 0;
  const bool uplus = isU && (uj >= NU);
  if (colthr) {
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const double e_q = (sc == c) ? 1.0 : 0.0, e_v = (sc == NQ + c) ? 1.0 : 0.0;
      if (M::hslot(c) >= 0) {
        RS_HQ(M::hslot(c)) = e_q;
        RS_HV(M::hslot(c)) = e_v;
      } else {
        RS_PQ(M::pslot(c)) = e_q;
        RS_PV(M::pslot(c)) = e_v;
      }
    }
#pragma unroll
    for (int k = 0; k < NY; ++k) RS_DY(k) = 0.0;
  }
  __syncthreads();
  const double S = sh.S, h = P.h;
  const int NST = 6 * P.substeps;
  for (int t = 0; t < NST + (JAC ? 3 : 1); ++t) {
    CITO_MARK((t * 8 + (warp < 8 ? warp : 7)) * 2);
    if (warp == 0) {
      if (t < NST) {
        const int s = t / 6, i = t % 6;
        Rec2<M>& R = sh.ring[t & 3];
        CITO_MARK_P(t, 0);
        // stage input (augmentation.py:200-205), coordinates owned by this lane
#pragma unroll
        for (int p = 0; p < PER; ++p) {
          const int k = lane + 32 * p;
          double a = RS_XR(p);
#pragma unroll
          for (int j = 0; j < 5; ++j)
            if (j < i) a = a + P.ha[i][j] * RS_KR(j, p);
          if (k < NX) R.xs[k] = a;
        }
        __syncwarp();
        CITO_MARK_P(t, 1);
        const double tau = h * (double)s + P.ch[i];
        for (int e = lane; e < M::NL + NU; e += 32) {
          if (e < M::NL) {
            double sv, cv;
            sincos(R.xs[3 * e + 2], &sv, &cv);
            R.pr.s[e] = sv;
            R.pr.c[e] = cv;
          } else {
            const int m = e - M::NL;
            R.pr.u[m] = (1.0 - tau) * sh.U[m] + tau * sh.U[NU + m];  // foh_eval :166-169
          }
        }
        __syncwarp();
        CITO_MARK_P(t, 2);
        if (lane == 0) crit_chain<M>(P, R, t);
        CITO_MARK_P(t, 6);
        __syncwarp();
        // stage slopes k_i = S * f (q rows: stage-input velocity, v rows: vdot)
#pragma unroll
        for (int p = 0; p < PER; ++p) {
          const int k = lane + 32 * p;
          double f = 0.0;
          if (k < NQ)
            f = R.xs[NQ + k];
          else if (k < NX)
            f = R.r[k - NQ];
          const double kk = S * f;
#pragma unroll
          for (int j = 0; j < 6; ++j)
            if (j == i) RS_KR(j, p) = kk;
          if (i == 5) {
            double inc = 0.0;
#pragma unroll
            for (int j = 0; j < 6; ++j) inc += P.b[j] * RS_KR(j, p);
            RS_XR(p) = RS_XR(p) + h * inc;
          }
        }
        CITO_MARK_P(t, 7);
      }
    } else if (warp == W_AUX) {
      if (t >= 1 && t <= NST) aux_stage<M>(P, sh, t - 1, lane, rs);
    } else if (JAC && (warp == K::W_JQV || warp == K::W_JU)) {
      if (t >= 2 && t <= NST + 1) {
        const int st = t - 2;
        const Rec2<M>& R = sh.ring[st & 3];
        const double* v = R.xs + NQ;
#if CITO_JAC_ONE_WARP  // every rate-Jacobian direction on one warp (generic kind 7)
        if (warp == K::W_JQV) {
          for (int kd = lane; kd < NDIR; kd += 32)
            tan_rate_k<M, 7>(P, R.pr, v, kd < NDIRX ? M::dir(kd) : NX + (kd - NDIRX), &sh.At[st & 1][kd][0]);
        }
#else
        if (warp == K::W_JQV) {  // q and v directions (kinds 1 | 2)
          for (int kd = lane; kd < NDIRX; kd += 32)
            tan_rate_k<M, 3>(P, R.pr, v, M::dir(kd), &sh.At[st & 1][kd][0]);
        } else {  // control directions (kind 4)
          for (int kd = NDIRX + lane; kd < NDIR; kd += 32)
            tan_rate_k<M, 4>(P, R.pr, v, NX + (kd - NDIRX), &sh.At[st & 1][kd][0]);
        }
#endif
      }
    } else if (JAC && colthr && t >= 3) {
      const int st = t - 3;
      col_stage2<M>(P, sh, sh.ring[st & 3], sh.At[st & 1], st / 6, st % 6, col, S, dS, isU, um, uplus, rs);
    }
    CITO_MARK((t * 8 + (warp < 8 ? warp : 7)) * 2 + 1);
    __syncthreads();
  }
  // ---- outputs
  if (warp == 0) {
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int k = lane + 32 * p;
      if (k < NX) sh.x[k] = RS_XR(p);
    }
  } else if (warp == W_AUX && lane < NY) {
    sh.x[NX + lane] = RS_YV;
  }
  if constexpr (JAC) {
  double* jxb = jx + b * NXT * NXT;
  double* jub = ju + b * NXT * 2 * NU;
  double* jsb = js + b * NXT;
  if (colthr) {
    double* dst;
    int stride;
    if (sc >= 0) {
      dst = jxb + sc;
      stride = NXT;
    } else if (isU) {
      dst = jub + uj;
      stride = 2 * NU;
    } else {
      dst = jsb;
      stride = 1;
    }
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const int hs = M::hslot(c);
      dst[c * stride] = hs >= 0 ? RS_HQ(hs) : RS_PQ(M::pslot(c));
      dst[(NQ + c) * stride] = hs >= 0 ? RS_HV(hs) : RS_PV(M::pslot(c));
    }
#pragma unroll
    for (int k = 0; k < NY; ++k) dst[(NX + k) * stride] = RS_DY(k);
  }
  if constexpr (M::NLCOL > 0) {  // closed-form columns (state directions no rate reads)
    double dqc = 0.0;
    for (int ss = 0; ss < P.substeps; ++ss) {
      double inc = 0.0;
#pragma unroll
      for (int ii = 0; ii < 6; ++ii) inc += P.b[ii] * S;
      dqc = dqc + h * inc;
    }
    for (int e = tid; e < M::NLCOL * NXT; e += blockDim.x) {
      const int lc = e / NXT, r = e % NXT;
      const int c = M::lcol(lc);
      double val = (r == c) ? 1.0 : 0.0;
      if (c >= NQ && r == c - NQ) val = dqc;
      jxb[r * NXT + c] = val;
    }
  }
  for (int e = tid; e < NXT * NY; e += blockDim.x) {
    const int r = e / Pos<NY>::v, c = NX + e % Pos<NY>::v;
    jxb[r * NXT + c] = (r == c) ? 1.0 : 0.0;
  }
  }  // JAC
  __syncthreads();
  for (int k = tid; k < NXT; k += blockDim.x) {
    const double e = sh.x[k];
    ends[b * NXT + k] = e;
    if (zs.defects) zs.defects[b * NXT + k] = sh.xn[k] - e;
    if (!isfinite(e)) sh.bad = 1;
  }
  __syncthreads();
  if (tid == 0 && bad) bad[b] = sh.bad;
#ifdef CITO_PROF
  if (g_cito_prof && blockIdx.x == 0 && threadIdx.x == 0) g_cito_prof[1665] = clock64();
#endif
}
