// cito_kernels.cuh — fp64 discretize+linearize kernels for sm_100a.
//
// Replaces cito.augmentation.Discretizer.{propagate_batch, linearize_batch}
// (/root/reference/pkg/src/cito/augmentation.py:180-242): a fixed-step
// Runge-Kutta-Fehlberg flow (5th-order weights, :46-56, :195-211) of the
// dilated augmented dynamics S*(f(x,u), Omega(x,u)) (:134-163) and the exact
// forward-mode derivatives of that discrete recursion w.r.t. (x~+, U, S).
//
// Formulation (differs from the reference's dense jacfwd on purpose):
//  * per RK stage the rate function is evaluated ONCE (primal, incl. the
//    Cholesky factor of the joint Gram matrix), then its Jacobian is formed
//    column by column (one thread per structurally relevant input direction)
//    with hand-derived forward-mode tangents that reuse the primal factor:
//       dlam = -G^{-1}(dJ vdot + J M^{-1}(dW + dJ^T lam) + dcurv)
//    (derivative of cito/contact_dynamics.py:86-95);
//  * the tangent columns of the interval map (one thread per column) are
//    advanced through the stage recursion with that Jacobian; only the
//    velocity-row stage increments are stored (q-row stage inputs follow
//    from q' = S v through precomputed tableau products).
// The topology (links/joints/contacts/path rows) is a compile-time template
// parameter (models_gen.cuh); numeric parameters are kernel arguments.
#pragma once

#include <cstdint>

// CITO_MODELS_GEN: a single-topology table generated at run time (the JIT build of
// paper_2604_09993_b200/build.py::build_topology); default: the bundled set
#ifdef CITO_MODELS_GEN
#include CITO_MODELS_GEN
#else
#include "models_gen.cuh"
#endif

#ifndef CITO_COL_RC
#define CITO_COL_RC 18  // rate rows per accumulator chunk of the column stage (register budget)
#endif

#define KMAX_L 16
#define KMAX_J 16
#define KMAX_C 8
#define KMAX_G 16
#define KMAX_GO 16
#define KMAX_E 96

// Numeric model parameters + tableau products, passed by value (constant bank).
struct KParams {
  double minv_m[KMAX_L], minv_I[KMAX_L], neg_mg[KMAX_L];
  double jrp[KMAX_J][2], jrc[KMAX_J][2];  // anchor - com (world parent: anchor itself)
  double jk[KMAX_J], jd[KMAX_J], jrest[KMAX_J];
  int32_t jspring[KMAX_J];
  double cr[KMAX_C][2], mu[KMAX_C], crest[KMAX_C];
  double height;
  double jl_lo[KMAX_G], jl_hi[KMAX_G], hb_lo[KMAX_G], hb_hi[KMAX_G];
  double mix[KMAX_GO][KMAX_G];
  // tableau (h = 1/substeps)
  int32_t substeps;
  double h;
  double ha[6][6];  // h * a_ij (the reference's `h * a` factor)
  double ch[6];     // c_i * h
  double b[6];      // b_i
  double hc1[6];    // h * sum_j a_ij
  double cq[6][6];  // h^2 * sum_j a_ij a_jl
  double e2[6];     // h^2 * sum_{i>l} b_i a_il
  double he1;       // h * sum_i b_i
  int32_t expr_len;
  int32_t expr_op[KMAX_E];
  double expr_arg[KMAX_E];
};

#define LI(r, c) ((r) * ((r) + 1) / 2 + (c))

// Optional per-role cycle instrumentation (tools/role_timing.py builds a separate
// library with -DCITO_PROF; the product build has none of it).
#ifdef CITO_PROF
__device__ long long* g_cito_prof = nullptr;
#define CITO_MARK(slot)                                                        \
  do {                                                                         \
    if (g_cito_prof && blockIdx.x == 0 && (threadIdx.x & 31) == 0) g_cito_prof[(slot)] = clock64(); \
  } while (0)
#define CITO_MARK_P(t, k)                                                                  \
  do {                                                                                     \
    if (g_cito_prof && blockIdx.x == 0 && threadIdx.x == 0) g_cito_prof[1024 + (t) * 16 + (k)] = clock64(); \
  } while (0)
#else
#define CITO_MARK_P(t, k) \
  do {                    \
  } while (0)
#define CITO_MARK(slot) \
  do {                  \
  } while (0)
#endif

// Decision-vector source of a linearize_all call: interval k reads x~+_k at
// z[(2k+1) n_xt], [U_k, S_k] at z[base_u + k (2 n_u + 1)] and writes the
// defect z[xm(k+1)] - end_k (cito/ocp.py:154-174, cito/scp.py:98-115).
struct ZSrc {
  const double* z;
  int64_t base_u;
  int64_t base_p;
  double* defects;
  int64_t zstride;  // distance between the decision vectors of consecutive problems (multi-start batches)
  int32_t n_int;    // intervals per problem (N - 1)
  int32_t n_node;   // nodes per problem (N)
  const double* de;  // optional device [delta, epsilon] (graph replays with changing delta)
};

template <int N>
struct Pos {
  static constexpr int v = N > 0 ? N : 1;
};

// ---------------------------------------------------------------------------
// implicit surface h(px, pz): value, gradient, Hessian (cito/multibody.py:144-172)
struct T2 {
  double v, gx, gz, hxx, hxz, hzz;
};

__device__ inline T2 surface_t2(const KParams& P, double px, double pz) {
  T2 st[16];
  int sp = 0;
  for (int k = 0; k < P.expr_len; ++k) {
    const int op = P.expr_op[k];
    const double arg = P.expr_arg[k];
    T2 r = {0, 0, 0, 0, 0, 0};
    if (op == 0) {
      r.v = arg;
    } else if (op == 1) {
      r.v = px;
      r.gx = 1.0;
    } else if (op == 2) {
      r.v = pz;
      r.gz = 1.0;
    } else if (op == 3 || op == 4) {
      T2 bb = st[--sp], a = st[--sp];
      if (op == 3) {
        r.v = a.v + bb.v;
        r.gx = a.gx + bb.gx;
        r.gz = a.gz + bb.gz;
        r.hxx = a.hxx + bb.hxx;
        r.hxz = a.hxz + bb.hxz;
        r.hzz = a.hzz + bb.hzz;
      } else {
        r.v = a.v * bb.v;
        r.gx = a.gx * bb.v + a.v * bb.gx;
        r.gz = a.gz * bb.v + a.v * bb.gz;
        r.hxx = a.hxx * bb.v + 2.0 * a.gx * bb.gx + a.v * bb.hxx;
        r.hxz = a.hxz * bb.v + a.gx * bb.gz + a.gz * bb.gx + a.v * bb.hxz;
        r.hzz = a.hzz * bb.v + 2.0 * a.gz * bb.gz + a.v * bb.hzz;
      }
    } else {
      T2 a = st[--sp];
      double f0, f1, f2;
      if (op == 5) {
        f0 = pow(a.v, arg);
        f1 = arg * pow(a.v, arg - 1.0);
        f2 = arg * (arg - 1.0) * pow(a.v, arg - 2.0);
      } else if (op == 6) {
        sincos(a.v, &f0, &f1);
        f2 = -f0;
      } else if (op == 7) {
        double s;
        sincos(a.v, &s, &f0);
        f1 = -s;
        f2 = -f0;
      } else if (op == 9) {  // log (variable exponent: a**b = exp(b log a))
        f0 = log(a.v);
        f1 = 1.0 / a.v;
        f2 = -f1 * f1;
      } else if (op == 10) {  // exp
        f0 = exp(a.v);
        f1 = f0;
        f2 = f0;
      } else {
        f0 = -a.v;
        f1 = -1.0;
        f2 = 0.0;
      }
      r.v = f0;
      r.gx = f1 * a.gx;
      r.gz = f1 * a.gz;
      r.hxx = f1 * a.hxx + f2 * a.gx * a.gx;
      r.hxz = f1 * a.hxz + f2 * a.gx * a.gz;
      r.hzz = f1 * a.hzz + f2 * a.gz * a.gz;
    }
    st[sp++] = r;
  }
  return st[0];
}

__device__ __forceinline__ double sabs(double x) { return sqrt(x * x + 1.0) - 1.0; }        // smoothmath.py:43-45
__device__ __forceinline__ double sabs_d(double x) { return x / sqrt(x * x + 1.0); }
__device__ __forceinline__ double srelu(double x) { return 0.5 * (x + sqrt(x * x + 1.0) - 1.0); }  // :60-63
__device__ __forceinline__ double srelu_d(double x) { return 0.5 * (1.0 + x / sqrt(x * x + 1.0)); }

// ---------------------------------------------------------------------------
// primal intermediates of one rate evaluation, consumed by the tangent threads
template <class M>
struct Prim {
  static constexpr int NL = M::NL, NJ2 = Pos<2 * M::NJ>::v, NC = Pos<M::NC>::v;
  static constexpr int NG = M::NC + 2 * M::NJL + 2 * M::NHB;
  double c[NL], s[NL];
  double rp[Pos<M::NJ>::v][2], rc[Pos<M::NJ>::v][2];  // R(theta) * (anchor - com)
  double L[NJ2 * (NJ2 + 1) / 2];                      // packed lower Cholesky factor of the Gram matrix
  double Li[NJ2];                                     // reciprocal pivots
  double lam[NJ2];                                    // joint reactions (phi_j)
  double vdot[3 * M::NL];
  double rr[NC][2], n[NC][2], t[NC][2], F[NC][2], Jv[NC][2];
  double hv[NC], g[NC][2], H[NC][3], gn[NC];  // implicit surface data
  double sd[NC], lamc[NC], sg[NC];
  double gp[Pos<NG>::v];
  // derivative factors of the smooth primitives, once per stage for all tangent
  // directions (filled by the off-chain warp of k_linearize2 only; tan_rate of
  // k_linearize computes them per lane): sabs'(lamc), sabs'(mu fn) mu, srelu'(sd),
  // 1 / (ft^2 + 1)^(3/2), 1 / |grad h|^3 (implicit terrain), srelu'(g)
  double dlam[NC], dmu[NC], dsrl[NC], dsgf[NC], ign3[NC];
  double dgp[Pos<NG>::v];
  double u[Pos<M::NA + 3 * M::NC>::v];
};

// rate function WITHOUT the dilation factor: out = [v; vdot; Omega] (n_xt)
//   forward_dynamics  cito/contact_dynamics.py:98-108 (+ :40-47, :76-95)
//   generalized_forces cito/multibody.py:285-321, kinematics :259-392
//   aux_rate           cito/augmentation.py:134-153, path g :112-129
template <class M>
__device__ void prim_rate(const KParams& P, const double* xs, const double* u, Prim<M>& pr, double* out) {
  // Every intermediate lives in registers; `pr` (shared memory) is only written,
  // so the dependent chain never waits on a shared-memory round trip.
  constexpr int NL = M::NL, NJ = M::NJ, NC = M::NC, NA = M::NA, NQ = 3 * NL;
  constexpr int NU = NA + 3 * NC;
  double q[NQ], v[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) {
    q[k] = xs[k];
    v[k] = xs[NQ + k];
  }
#pragma unroll
  for (int m = 0; m < NU; ++m) pr.u[m] = u[m];
  double cl[NL], sl[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    sincos(q[3 * l + 2], &sl[l], &cl[l]);
    pr.c[l] = cl[l];
    pr.s[l] = sl[l];
  }
  double W[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) W[k] = 0.0;
#pragma unroll
  for (int l = 0; l < NL; ++l) W[3 * l + 1] += P.neg_mg[l];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p = M::jparent(j), c = M::jchild(j), a = M::jact(j);
    double mo = 0.0;
    if (a >= 0) mo = mo + u[a];
    if (P.jspring[j]) {
      const double th_p = p >= 0 ? q[3 * p + 2] : 0.0;
      const double om_p = p >= 0 ? v[3 * p + 2] : 0.0;
      const double rel = q[3 * c + 2] - th_p - P.jrest[j];
      mo = mo - P.jk[j] * rel - P.jd[j] * (v[3 * c + 2] - om_p);
    }
    W[3 * c + 2] += mo;
    if (p >= 0) W[3 * p + 2] += -mo;
  }
  // contacts: frame, world force, wrench, Omega ingredients
  double sdl[Pos<NC>::v], Jvl[Pos<NC>::v][2], tl[Pos<NC>::v][2];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int l = M::clink(i);
    const double rx = cl[l] * P.cr[i][0] - sl[l] * P.cr[i][1];
    const double rz = sl[l] * P.cr[i][0] + cl[l] * P.cr[i][1];
    pr.rr[i][0] = rx;
    pr.rr[i][1] = rz;
    const double Px = q[3 * l] + rx, Pz = q[3 * l + 1] + rz;
    double n0, n1;
    if constexpr (M::IMPLICIT) {
      T2 t2 = surface_t2(P, Px, Pz);
      pr.hv[i] = t2.v;
      pr.g[i][0] = t2.gx;
      pr.g[i][1] = t2.gz;
      pr.H[i][0] = t2.hxx;
      pr.H[i][1] = t2.hxz;
      pr.H[i][2] = t2.hzz;
      const double gn = sqrt(t2.gx * t2.gx + t2.gz * t2.gz);
      pr.gn[i] = gn;
      n0 = t2.gx / gn;
      n1 = t2.gz / gn;
      sdl[i] = t2.v / gn;
    } else {
      n0 = 0.0;
      n1 = 1.0;
      sdl[i] = Pz - P.height;
    }
    pr.sd[i] = sdl[i];
    const double t0 = n1, t1 = -n0;
    tl[i][0] = t0;
    tl[i][1] = t1;
    pr.n[i][0] = n0;
    pr.n[i][1] = n1;
    pr.t[i][0] = t0;
    pr.t[i][1] = t1;
    const double ft = u[NA + 2 * i], fn = u[NA + 2 * i + 1];
    const double F0 = t0 * ft + n0 * fn, F1 = t1 * ft + n1 * fn;
    pr.F[i][0] = F0;
    pr.F[i][1] = F1;
    W[3 * l] += F0;
    W[3 * l + 1] += F1;
    W[3 * l + 2] += (-rz) * F0 + rx * F1;
    const double w = v[3 * l + 2];
    Jvl[i][0] = v[3 * l] + (-rz) * w;
    Jvl[i][1] = v[3 * l + 1] + rx * w;
    pr.Jv[i][0] = Jvl[i][0];
    pr.Jv[i][1] = Jvl[i][1];
  }
  double* vdot = out + NQ;
  if constexpr (NJ == 0) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      vdot[3 * l] = P.minv_m[l] * W[3 * l];
      vdot[3 * l + 1] = P.minv_m[l] * W[3 * l + 1];
      vdot[3 * l + 2] = P.minv_I[l] * W[3 * l + 2];
      pr.vdot[3 * l + 2] = vdot[3 * l + 2];
    }
  } else {
    constexpr int NJ2 = 2 * NJ;
    double R[NJ][2][2];  // [joint][side parent/child][x,z] = R(theta) (anchor - com)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int p = M::jparent(j), c = M::jchild(j);
      if (p >= 0) {
        R[j][0][0] = cl[p] * P.jrp[j][0] - sl[p] * P.jrp[j][1];
        R[j][0][1] = sl[p] * P.jrp[j][0] + cl[p] * P.jrp[j][1];
        pr.rp[j][0] = R[j][0][0];
        pr.rp[j][1] = R[j][0][1];
      } else {
        R[j][0][0] = R[j][0][1] = 0.0;
      }
      R[j][1][0] = cl[c] * P.jrc[j][0] - sl[c] * P.jrc[j][1];
      R[j][1][1] = sl[c] * P.jrc[j][0] + cl[c] * P.jrc[j][1];
      pr.rc[j][0] = R[j][1][0];
      pr.rc[j][1] = R[j][1][1];
    }
    // Gram matrix G = J M^-1 J^T in the no-fill elimination order M::jperm
    // (gen_models.py), packed lower, only the structurally nonzero blocks
    double Lr[NJ2 * (NJ2 + 1) / 2];
#pragma unroll
    for (int a = 0; a < NJ; ++a)
#pragma unroll
      for (int bp = 0; bp <= a; ++bp) {
        if (!M::lnzb(a, bp)) continue;
        const int j = M::jperm(a), k = M::jperm(bp);
#pragma unroll
        for (int al = 0; al < 2; ++al)
#pragma unroll
          for (int be = 0; be < 2; ++be)
            if (!(a == bp && be > al)) Lr[LI(2 * a + al, 2 * bp + be)] = 0.0;
#pragma unroll
        for (int sa = 0; sa < 2; ++sa)
#pragma unroll
          for (int sb = 0; sb < 2; ++sb) {
            const int la = sa == 0 ? M::jparent(j) : M::jchild(j);
            const int lb = sb == 0 ? M::jparent(k) : M::jchild(k);
            if (la < 0 || la != lb) continue;
            const double sg = (sa == sb) ? 1.0 : -1.0;
            const double dA[2] = {-R[j][sa][1], R[j][sa][0]}, dB[2] = {-R[k][sb][1], R[k][sb][0]};
#pragma unroll
            for (int al = 0; al < 2; ++al)
#pragma unroll
              for (int be = 0; be < 2; ++be) {
                if (a == bp && be > al) continue;
                double val = dA[al] * dB[be] * P.minv_I[la];
                if (al == be) val += P.minv_m[la];
                Lr[LI(2 * a + al, 2 * bp + be)] += sg * val;
              }
          }
      }
    // rhs = J (M^-1 W) + curv, in elimination order
    double y[NJ2];
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
          const double dP = al == 0 ? -R[j][sa][1] : R[j][sa][0];
          const double w = v[3 * l + 2];
          acc += sgn * (P.minv_m[l] * W[3 * l + al] + dP * P.minv_I[l] * W[3 * l + 2] - R[j][sa][al] * w * w);
        }
        y[2 * a + al] = acc;
      }
    }
    // sparse Cholesky G = L L^T (no fill outside M::lnzb), reciprocal pivots, both
    // solves: generated straight-line code (gen_models.py), every value in a register
    double Lir[NJ2];
    M::chol_solve(Lr, y, Lir);
    // publish the factor (elimination order) for the tangent threads
#pragma unroll
    for (int r = 0; r < NJ2; ++r) {
      pr.Li[r] = Lir[r];
#pragma unroll
      for (int c = 0; c <= r; ++c)
        if (M::lnzb(r / 2, c / 2)) pr.L[LI(r, c)] = Lr[LI(r, c)];
    }
    // lam (joint order) = -G^{-1} rhs ; vdot = M^-1 (W + J^T lam)
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
        W[3 * l + 2] += sgn * ((-R[j][sa][1]) * l0 + R[j][sa][0] * l1);
      }
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      vdot[3 * l] = P.minv_m[l] * W[3 * l];
      vdot[3 * l + 1] = P.minv_m[l] * W[3 * l + 1];
      vdot[3 * l + 2] = P.minv_I[l] * W[3 * l + 2];
      pr.vdot[3 * l + 2] = vdot[3 * l + 2];
    }
  }
#pragma unroll
  for (int k = 0; k < NQ; ++k) out[k] = v[k];
  // Omega (aux_rate)
  double* yo = out + 2 * NQ;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const double ft = u[NA + 2 * i], fn = u[NA + 2 * i + 1], gam = u[NA + 2 * NC + i];
    const double vt = tl[i][0] * Jvl[i][0] + tl[i][1] * Jvl[i][1];
    const double sgt = ft / sqrt(ft * ft + 1.0);
    pr.sg[i] = sgt;
    const double lamc = vt + gam * sgt;
    pr.lamc[i] = lamc;
    yo[5 * i + 0] = fn;
    yo[5 * i + 1] = sabs(lamc);
    yo[5 * i + 2] = gam;
    yo[5 * i + 3] = sabs(P.mu[i] * fn) - sabs(ft);
    yo[5 * i + 4] = srelu(sdl[i]);
  }
  if constexpr (M::NGO > 0) {
    constexpr int NG = Prim<M>::NG;
    double gpl[Pos<NG>::v];
    int r = 0;
#pragma unroll
    for (int i = 0; i < NC; ++i) gpl[r++] = -sdl[i];
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
      sgv[jg] = srelu(gpl[jg]);
    }
#pragma unroll
    for (int o = 0; o < M::NGO; ++o) {
      double acc = 0.0;
#pragma unroll
      for (int jg = 0; jg < NG; ++jg) acc += P.mix[o][jg] * sgv[jg];
      yo[5 * NC + o] = acc;
    }
  }
}

// Tangent of the unscaled rate along one input direction `dir` of (q, v, u):
//   dir in [0, NQ) -> q_dir, [NQ, 2NQ) -> v, [2NQ, 2NQ+NU) -> u.
// Writes out[0:NQ] = d vdot, out[NQ:NQ+NY] = d Omega.
template <class M>
__device__ void tan_rate(const KParams& P, const Prim<M>& pr, const double* v, int dir, double* out,
                         int ostride) {
  constexpr int NL = M::NL, NJ = M::NJ, NC = M::NC, NA = M::NA, NQ = 3 * NL, NX = 2 * NQ;
#define SQ(k) ((dir) == (k) ? 1.0 : 0.0)
#define SV(k) ((dir) == NQ + (k) ? 1.0 : 0.0)
#define SU(m) ((dir) == NX + (m) ? 1.0 : 0.0)
  double dW[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) dW[k] = 0.0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p = M::jparent(j), c = M::jchild(j), a = M::jact(j);
    double dm = a >= 0 ? SU(a) : 0.0;
    if (P.jspring[j]) {
      const double dth_p = p >= 0 ? SQ(3 * p + 2) : 0.0;
      const double dom_p = p >= 0 ? SV(3 * p + 2) : 0.0;
      dm = dm - P.jk[j] * (SQ(3 * c + 2) - dth_p) - P.jd[j] * (SV(3 * c + 2) - dom_p);
    }
    dW[3 * c + 2] += dm;
    if (p >= 0) dW[3 * p + 2] -= dm;
  }
  double dP[Pos<NC>::v][2], dn[Pos<NC>::v][2], dsd[Pos<NC>::v];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int l = M::clink(i);
    const double rx = pr.rr[i][0], rz = pr.rr[i][1];
    const double dth = SQ(3 * l + 2);
    dP[i][0] = SQ(3 * l) + dth * (-rz);
    dP[i][1] = SQ(3 * l + 1) + dth * rx;
    double dt0 = 0.0, dt1 = 0.0, dn0 = 0.0, dn1 = 0.0;
    if constexpr (M::IMPLICIT) {
      const double Hd0 = pr.H[i][0] * dP[i][0] + pr.H[i][1] * dP[i][1];
      const double Hd1 = pr.H[i][1] * dP[i][0] + pr.H[i][2] * dP[i][1];
      const double gn = pr.gn[i], g0 = pr.g[i][0], g1 = pr.g[i][1];
      const double gHd = g0 * Hd0 + g1 * Hd1;
      const double ign3 = 1.0 / (gn * gn * gn);
      dn0 = Hd0 / gn - g0 * gHd * ign3;
      dn1 = Hd1 / gn - g1 * gHd * ign3;
      dt0 = dn1;
      dt1 = -dn0;
      dsd[i] = (g0 * dP[i][0] + g1 * dP[i][1]) / gn - pr.hv[i] * gHd * ign3;
    } else {
      dsd[i] = dP[i][1];
    }
    dn[i][0] = dn0;
    dn[i][1] = dn1;
    const double ft = pr.u[NA + 2 * i], fn = pr.u[NA + 2 * i + 1];
    const double dft = SU(NA + 2 * i), dfn = SU(NA + 2 * i + 1);
    const double dF0 = dt0 * ft + pr.t[i][0] * dft + dn0 * fn + pr.n[i][0] * dfn;
    const double dF1 = dt1 * ft + pr.t[i][1] * dft + dn1 * fn + pr.n[i][1] * dfn;
    dW[3 * l] += dF0;
    dW[3 * l + 1] += dF1;
    dW[3 * l + 2] += -dth * (rx * pr.F[i][0] + rz * pr.F[i][1]) + (-rz) * dF0 + rx * dF1;
  }
  if constexpr (NJ == 0) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      out[(3 * l) * ostride] = P.minv_m[l] * dW[3 * l];
      out[(3 * l + 1) * ostride] = P.minv_m[l] * dW[3 * l + 1];
      out[(3 * l + 2) * ostride] = P.minv_I[l] * dW[3 * l + 2];
    }
  } else {
    constexpr int NJ2 = 2 * NJ;
    // g = dW + dJ^T lam (theta coordinates only)
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
    // rhs' = dJ vdot + J M^-1 g + dcurv
    double z[NJ2];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
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
          const double dth = SQ(3 * l + 2), w = v[3 * l + 2], dw = SV(3 * l + 2);
          const double term = -dth * R[al] * pr.vdot[3 * l + 2] + P.minv_m[l] * dW[3 * l + al] +
                              dPa * P.minv_I[l] * dW[3 * l + 2] - dth * dPa * w * w - 2.0 * R[al] * w * dw;
          acc += sgn * term;
        }
        z[2 * j + al] = acc;
      }
    // z <- G^{-1} z with the primal factor (elimination order M::jperm); dlam = -z
    double zp[NJ2];
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      zp[2 * a] = z[2 * M::jperm(a)];
      zp[2 * a + 1] = z[2 * M::jperm(a) + 1];
    }
    M::tri_solve(pr.L, pr.Li, zp);  // generated straight-line sparse solves (gen_models.py)
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      z[2 * M::jperm(a)] = zp[2 * a];
      z[2 * M::jperm(a) + 1] = zp[2 * a + 1];
    }
    // dvdot = M^-1 (g + J^T dlam)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int sa = 0; sa < 2; ++sa) {
        const int l = sa == 0 ? M::jparent(j) : M::jchild(j);
        if (l < 0) continue;
        const double sgn = sa == 0 ? 1.0 : -1.0;
        const double* R = sa == 0 ? pr.rp[j] : pr.rc[j];
        const double l0 = -z[2 * j], l1 = -z[2 * j + 1];
        dW[3 * l] += sgn * l0;
        dW[3 * l + 1] += sgn * l1;
        dW[3 * l + 2] += sgn * ((-R[1]) * l0 + R[0] * l1);
      }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      out[(3 * l) * ostride] = P.minv_m[l] * dW[3 * l];
      out[(3 * l + 1) * ostride] = P.minv_m[l] * dW[3 * l + 1];
      out[(3 * l + 2) * ostride] = P.minv_I[l] * dW[3 * l + 2];
    }
  }
  // d Omega
  double* dy = out + NQ * ostride;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int l = M::clink(i);
    const double ft = pr.u[NA + 2 * i], fn = pr.u[NA + 2 * i + 1], gam = pr.u[NA + 2 * NC + i];
    const double dft = SU(NA + 2 * i), dfn = SU(NA + 2 * i + 1), dgam = SU(NA + 2 * NC + i);
    const double rx = pr.rr[i][0], rz = pr.rr[i][1];
    const double dth = SQ(3 * l + 2), w = v[3 * l + 2], dw = SV(3 * l + 2);
    // d(J_i v) = dv_lin + d(dP/dth) w + dP/dth dw, d(dP/dth) = -dth * rr
    const double dJv0 = SV(3 * l) - dth * rx * w + (-rz) * dw;
    const double dJv1 = SV(3 * l + 1) - dth * rz * w + rx * dw;
    const double dvt = (dn[i][1]) * pr.Jv[i][0] + (-dn[i][0]) * pr.Jv[i][1] + pr.t[i][0] * dJv0 +
                       pr.t[i][1] * dJv1;
    const double q1 = ft * ft + 1.0;
    const double dsg = dft / (q1 * sqrt(q1));
    const double dlamc = dvt + dgam * pr.sg[i] + gam * dsg;
    dy[(5 * i + 0) * ostride] = dfn;
    dy[(5 * i + 1) * ostride] = sabs_d(pr.lamc[i]) * dlamc;
    dy[(5 * i + 2) * ostride] = dgam;
    dy[(5 * i + 3) * ostride] = sabs_d(P.mu[i] * fn) * P.mu[i] * dfn - pr.sg[i] * dft;
    dy[(5 * i + 4) * ostride] = srelu_d(pr.sd[i]) * dsd[i];
  }
  if constexpr (M::NGO > 0) {
    constexpr int NG = Prim<M>::NG;
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
    for (int jg = 0; jg < NG; ++jg) dg[jg] *= srelu_d(pr.gp[jg]);
#pragma unroll
    for (int o = 0; o < M::NGO; ++o) {
      double acc = 0.0;
#pragma unroll
      for (int jg = 0; jg < NG; ++jg) acc += P.mix[o][jg] * dg[jg];
      dy[(5 * NC + o) * ostride] = acc;
    }
  }
#undef SQ
#undef SV
#undef SU
}


template <class M>
struct Dims {
  static constexpr int NL = M::NL, NQ = 3 * NL, NX = 2 * NQ, NC = M::NC, NA = M::NA;
  static constexpr int NU = NA + 3 * NC, NY = 5 * NC + M::NGO, NXT = NX + NY;
  static constexpr int NCOL = M::NHCOL + 2 * NU + 1;  // advanced tangent columns: heavy x~+ columns, U-, U+, S
  static constexpr int NCOLX = NX + 2 * NU + 1;         // all non-y columns (incl. closed-form ones)
  static constexpr int NDIR = M::NDIRX + NU;    // rate-Jacobian input directions
  static constexpr int NR = NQ + NY;            // rate rows with a non-trivial Jacobian (vdot, Omega)
  static constexpr int NRP = (NR + 1) & ~1;     // padded to 16 B rows
  static constexpr int NCOLP = NCOL | 1;        // odd column stride (bank spread)
  static constexpr int NH = Pos<M::NHIST>::v;
  static constexpr int NT = ((NCOL > NDIR ? NCOL : NDIR) + 31) / 32 * 32;
};

// Per-stage record of the primal trajectory (a slot of K1's smem ring): everything
// the Jacobian and column warps need for that stage's rate Jacobian and dS terms,
// so they never recompute (or wait on) the primal chain.
template <class M>
struct Rec {
  Prim<M> pr;
  double vs[3 * M::NL];       // stage-input velocities
  double r[Dims<M>::NR];      // unscaled rate rows: vdot (NQ), Omega (NY)
  double wq[3 * M::NL];       // sum_j h a_ij v_{s,j}: dS term of the q-row stage inputs
};

// ---------------------------------------------------------------------------
// K2: primal RKF flow, one thread per interval (cito/augmentation.py:195-211);
// the throughput variant of propagate for batches larger than the SMs.
template <class M>
__global__ void __launch_bounds__(64) k_primal(const KParams P, int64_t B, const double* __restrict__ xt0s,
                                               const double* __restrict__ Us, const double* __restrict__ Ss,
                                               double* __restrict__ ends, int32_t* __restrict__ bad) {
  using D = Dims<M>;
  constexpr int NX = D::NX, NU = D::NU, NY = D::NY, NXT = D::NXT;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double x[NXT], xs[NX], r[NXT], K[6][NX], ky[Pos<NY>::v], U[2 * NU + 1];
  Prim<M> pr;
  for (int k = 0; k < NXT; ++k) x[k] = xt0s[b * NXT + k];
  for (int k = 0; k < 2 * NU; ++k) U[k] = Us[b * 2 * NU + k];
  const double S = Ss[b];
  const double h = P.h;
  for (int s = 0; s < P.substeps; ++s) {
    const double tau0 = h * (double)s;
#pragma unroll
    for (int k = 0; k < NY; ++k) ky[k] = 0.0;
    for (int i = 0; i < 6; ++i) {
      const double tau = tau0 + P.ch[i];
      for (int k = 0; k < NX; ++k) {
        double a = x[k];
        for (int j = 0; j < i; ++j) a = a + P.ha[i][j] * K[j][k];
        xs[k] = a;
      }
      double u[NU > 0 ? NU : 1];
#pragma unroll
      for (int m = 0; m < NU; ++m) u[m] = (1.0 - tau) * U[m] + tau * U[NU + m];  // foh_eval :166-169
      prim_rate<M>(P, xs, u, pr, r);
      for (int k = 0; k < NX; ++k) K[i][k] = S * r[k];
#pragma unroll
      for (int k = 0; k < NY; ++k) ky[k] += P.b[i] * (S * r[NX + k]);
    }
    for (int k = 0; k < NX; ++k) {
      double inc = 0.0;
      for (int j = 0; j < 6; ++j) inc += P.b[j] * K[j][k];
      x[k] = x[k] + h * inc;
    }
#pragma unroll
    for (int k = 0; k < NY; ++k) x[NX + k] = x[NX + k] + h * ky[k];
  }
  int nb = 0;
  for (int k = 0; k < NXT; ++k) {
    ends[b * NXT + k] = x[k];
    nb |= !isfinite(x[k]);
  }
  if (bad) bad[b] = nb;
}

// K5: pointwise audit of sampled states (verifier.replay_check, SURVEY.md §8(f)
// row 3; /root/reference/pkg/src/cito/verifier.py:257-272, 314-318): per sample
// (one thread) the contact signed distances (multibody.py:384-392), the joint
// anchor residuals joint_constraint_value (multibody.py:324-336) and the
// auxiliary rates Omega(x, u) (augmentation.py:134-153).
template <class M>
__global__ void __launch_bounds__(64) k_audit(const KParams P, int64_t B, const double* __restrict__ xs, int64_t xstride,
                                              const double* __restrict__ us, double* __restrict__ sds,
                                              double* __restrict__ cj, double* __restrict__ omega) {
  using D = Dims<M>;
  constexpr int NX = D::NX, NU = D::NU, NY = D::NY, NXT = D::NXT, NC = M::NC, NJ = M::NJ;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double x[NX], u[Pos<NU>::v], r[NXT];
  Prim<M> pr;
  for (int k = 0; k < NX; ++k) x[k] = xs[b * xstride + k];
  for (int m = 0; m < NU; ++m) u[m] = us[b * NU + m];
  prim_rate<M>(P, x, u, pr, r);
  for (int i = 0; i < NC; ++i) sds[b * NC + i] = pr.sd[i];
  for (int k = 0; k < NY; ++k) omega[b * NY + k] = r[NX + k];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int p = M::jparent(j), c = M::jchild(j);
    double px = P.jrp[j][0], pz = P.jrp[j][1];  // world parent: the anchor itself
    if (p >= 0) {
      px = x[3 * p] + pr.rp[j][0];
      pz = x[3 * p + 1] + pr.rp[j][1];
    }
    cj[b * 2 * NJ + 2 * j] = px - (x[3 * c] + pr.rc[j][0]);
    cj[b * 2 * NJ + 2 * j + 1] = pz - (x[3 * c + 1] + pr.rc[j][1]);
  }
}

// ===========================================================================
// K1 (fused, warp-specialized, software-pipelined) -- one CTA per interval.
//   warp 0      : primal producer.  Tick t computes RK stage t of the primal
//                 chain (lane 0 runs the rate function; the warp does the
//                 elementwise stage algebra) and publishes its record in
//                 ring[t % 3].
//   warp 1      : rate Jacobian of stage t-1 (one input direction per lane,
//                 tan_rate reusing the record's Cholesky factor) -> A[(t-1) % 2].
//   warps 2..   : one tangent column per thread, stage t-2.
// One __syncthreads per tick; the primal chain and the tangent work overlap,
// so a linearization takes ~max(primal, tangent) instead of their sum.
template <class M>
struct FusedDims {
  using D = Dims<M>;
  static constexpr int NCW = (D::NCOL + 31) / 32;
  static constexpr int NT = 64 + 32 * NCW;
};

template <class M>
struct SParams {
  static constexpr int NL = M::NL, NJ = Pos<M::NJ>::v, NC = Pos<M::NC>::v;
  double minv_m[NL], minv_I[NL], neg_mg[NL];
  double jrp[NJ][2], jrc[NJ][2], jk[NJ], jd[NJ], jrest[NJ];
  int jspring[NJ];
  double cr[NC][2], mu[NC];
  // topology tables for lane-indexed lookups (constexpr selects with a runtime
  // index compile to divergent jump tables)
  int jp[NJ], jc[NJ], ja[NJ], jperm[NJ], cl[NC];
  int ba[Pos<M::NBLK>::v], bb[Pos<M::NBLK>::v];
  int lc[Pos<M::NLCOL>::v];
};

template <class M>
struct PrimScratch {
  static constexpr int NJ2 = Pos<2 * M::NJ>::v;
  double W[3 * M::NL];
  double Lw[NJ2 * (NJ2 + 1) / 2];
  double y[NJ2];
  double mo[Pos<M::NJ>::v];
};

template <class M>
struct FusedShared {
  using D = Dims<M>;
  Rec<M> ring[3];
  PrimScratch<M> ps;
  SParams<M> sp;
  double At[2][D::NDIR][D::NRP];  // rate Jacobian, direction-major (row pairs load as LDS.128)
  double KV[5][D::NH][D::NCOLP];
  double PQ[Pos<M::NPUSH>::v][D::NCOLP];
  double PV[Pos<M::NPUSH>::v][D::NCOLP];
  double DY[Pos<D::NY>::v][D::NCOLP];
  double x[D::NXT];
  double xs[D::NX];
  double rf[D::NXT];
  double K[6][D::NX];
  double VS[6][D::NQ];
  double ky[Pos<D::NY>::v];
  double vbs[2][D::NQ];
  double U[2 * D::NU + 1];
  double xn[D::NXT];  // the next interval's start state (defects), loaded with the inputs
  double S;
  int bad;
};

// Warp-cooperative primal stage (the same arithmetic as prim_rate, spread over
// the 32 lanes of warp 0: links, joint sides, contacts, Gram blocks in
// parallel; only the sparse Cholesky + solves run on one lane).
template <class M>
__device__ __forceinline__ void fused_primal(const KParams& P, FusedShared<M>& sh, int t, int lane) {
  using D = Dims<M>;
  constexpr int NL = M::NL, NJ = M::NJ, NC = M::NC, NA = M::NA, NQ = D::NQ, NX = D::NX, NU = D::NU, NY = D::NY;
  constexpr int NR = D::NR, NJ2 = 2 * NJ;
  const int s = t / 6, i = t % 6;
  const double h = P.h, S = sh.S;
  const double tau = h * (double)s + P.ch[i];
  Rec<M>& R = sh.ring[t % 3];
  Prim<M>& pr = R.pr;
  PrimScratch<M>& w = sh.ps;
  const SParams<M>& Q = sh.sp;  // runtime-indexed parameters live in smem (divergent lanes)
  const double* q = sh.xs;
  const double* v = sh.xs + NQ;
  CITO_MARK_P(t, 0);
  // 0: stage input (cito/augmentation.py:200-205)
  for (int k = lane; k < NX; k += 32) {
    double a = sh.x[k];
    for (int j = 0; j < i; ++j) a = a + P.ha[i][j] * sh.K[j][k];
    sh.xs[k] = a;
  }
  __syncwarp();
  CITO_MARK_P(t, 1);
  // 1: cos/sin per link, FOH control (foh_eval :166-169)
  for (int e = lane; e < NL + NU; e += 32) {
    if (e < NL) {
      double sv, cv;
      sincos(q[3 * e + 2], &sv, &cv);
      pr.s[e] = sv;
      pr.c[e] = cv;
    } else {
      const int m = e - NL;
      pr.u[m] = (1.0 - tau) * sh.U[m] + tau * sh.U[NU + m];
    }
  }
  __syncwarp();
  CITO_MARK_P(t, 2);
  // 2: rotated joint anchors, contacts (frame, force, Omega ingredients), joint moments
  for (int e = lane; e < 2 * NJ + NC + NJ; e += 32) {
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
    } else if (e < 2 * NJ + NC) {
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
      const double sgt = ft / sqrt(ft * ft + 1.0);  // friction_stationarity (contact_dynamics.py:55-66)
      pr.sg[ci] = sgt;
      pr.lamc[ci] = t0 * Jv0 + t1 * Jv1 + gam * sgt;
    } else {
      const int j = e - 2 * NJ - NC;  // joint moment (multibody.py:303-320)
      const int p = Q.jp[j], c = Q.jc[j], a = Q.ja[j];
      double mo = 0.0;
      if (a >= 0) mo = mo + pr.u[a];
      if (Q.jspring[j]) {
        const double th_p = p >= 0 ? q[3 * p + 2] : 0.0;
        const double om_p = p >= 0 ? v[3 * p + 2] : 0.0;
        const double rel = q[3 * c + 2] - th_p - Q.jrest[j];
        mo = mo - Q.jk[j] * rel - Q.jd[j] * (v[3 * c + 2] - om_p);
      }
      w.mo[j] = mo;
    }
  }
  __syncwarp();
  CITO_MARK_P(t, 3);
  // 3: generalized forces per link; Gram blocks (elimination order, nonzero blocks only)
  for (int e = lane; e < NL + M::NBLK; e += 32) {
    if (e < NL) {
      const int l = e;
      double W0 = 0.0, W1 = Q.neg_mg[l], W2 = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if (M::jchild(j) == l) W2 += w.mo[j];
        if (M::jparent(j) == l) W2 += -w.mo[j];
      }
#pragma unroll
      for (int ci = 0; ci < NC; ++ci)
        if (M::clink(ci) == l) {
          const double F0 = pr.F[ci][0], F1 = pr.F[ci][1];
          W0 += F0;
          W1 += F1;
          W2 += (-pr.rr[ci][1]) * F0 + pr.rr[ci][0] * F1;
        }
      w.W[3 * l] = W0;
      w.W[3 * l + 1] = W1;
      w.W[3 * l + 2] = W2;
    } else if constexpr (NJ > 0) {
      const int kb = e - NL, a = Q.ba[kb], bp = Q.bb[kb];
      const int j = Q.jperm[a], k = Q.jperm[bp];
      double g00 = 0.0, g01 = 0.0, g10 = 0.0, g11 = 0.0;
#pragma unroll
      for (int sa = 0; sa < 2; ++sa)
#pragma unroll
        for (int sb = 0; sb < 2; ++sb) {
          const int la = sa == 0 ? Q.jp[j] : Q.jc[j];
          const int lb = sb == 0 ? Q.jp[k] : Q.jc[k];
          if (la < 0 || la != lb) continue;
          const double sg = (sa == sb) ? 1.0 : -1.0;
          const double* Ra = sa == 0 ? pr.rp[j] : pr.rc[j];
          const double* Rb = sb == 0 ? pr.rp[k] : pr.rc[k];
          const double dA0 = -Ra[1], dA1 = Ra[0], dB0 = -Rb[1], dB1 = Rb[0];
          const double mI = Q.minv_I[la], mm = Q.minv_m[la];
          g00 += sg * (dA0 * dB0 * mI + mm);
          g01 += sg * (dA0 * dB1 * mI);
          g10 += sg * (dA1 * dB0 * mI);
          g11 += sg * (dA1 * dB1 * mI + mm);
        }
      w.Lw[LI(2 * a, 2 * bp)] = g00;
      w.Lw[LI(2 * a + 1, 2 * bp)] = g10;
      w.Lw[LI(2 * a + 1, 2 * bp + 1)] = g11;
      if (a != bp) w.Lw[LI(2 * a, 2 * bp + 1)] = g01;
    }
  }
  __syncwarp();
  CITO_MARK_P(t, 4);
  if constexpr (NJ > 0) {
    // 4: rhs = J (M^-1 W) + curv, per joint (elimination order)
    for (int a = lane; a < NJ; a += 32) {
      const int j = Q.jperm[a];
#pragma unroll
      for (int al = 0; al < 2; ++al) {
        double acc = 0.0;
#pragma unroll
        for (int sa = 0; sa < 2; ++sa) {
          const int l = sa == 0 ? Q.jp[j] : Q.jc[j];
          if (l < 0) continue;
          const double sgn = sa == 0 ? 1.0 : -1.0;
          const double* Rj = sa == 0 ? pr.rp[j] : pr.rc[j];
          const double dP = al == 0 ? -Rj[1] : Rj[0];
          const double om = v[3 * l + 2];
          acc += sgn * (Q.minv_m[l] * w.W[3 * l + al] + dP * Q.minv_I[l] * w.W[3 * l + 2] - Rj[al] * om * om);
        }
        w.y[2 * a + al] = acc;
      }
    }
    __syncwarp();
  CITO_MARK_P(t, 5);
    // 5: sparse Cholesky + both triangular solves on one lane, in registers
    if (lane == 0) {
      double Lr[NJ2 * (NJ2 + 1) / 2], y[NJ2], Lir[NJ2];
#pragma unroll
      for (int r = 0; r < NJ2; ++r) {
        y[r] = w.y[r];
#pragma unroll
        for (int c = 0; c <= r; ++c) Lr[LI(r, c)] = M::lnzb(r / 2, c / 2) ? w.Lw[LI(r, c)] : 0.0;
      }
      M::chol_solve(Lr, y, Lir);  // generated straight-line sparse Cholesky + solves (gen_models.py)
#pragma unroll
      for (int r = 0; r < NJ2; ++r) {
        pr.Li[r] = Lir[r];
#pragma unroll
        for (int c = 0; c <= r; ++c)
          if (M::lnzb(r / 2, c / 2)) pr.L[LI(r, c)] = Lr[LI(r, c)];
      }
#pragma unroll
      for (int a = 0; a < NJ; ++a) {
        pr.lam[2 * M::jperm(a)] = -y[2 * a];
        pr.lam[2 * M::jperm(a) + 1] = -y[2 * a + 1];
      }
    }
    __syncwarp();
  CITO_MARK_P(t, 6);
  }
  // 6: vdot per link (M^-1 (W + J^T lam)), Omega per contact, mixed path rows
  double* rf = sh.rf;
  for (int e = lane; e < NL + NC + (M::NGO > 0 ? 1 : 0); e += 32) {
    if (e < NL) {
      const int l = e;
      double W0 = w.W[3 * l], W1 = w.W[3 * l + 1], W2 = w.W[3 * l + 2];
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int sa = 0; sa < 2; ++sa) {
          const int lj = sa == 0 ? M::jparent(j) : M::jchild(j);
          if (lj != l) continue;
          const double sgn = sa == 0 ? 1.0 : -1.0;
          const double* Rj = sa == 0 ? pr.rp[j] : pr.rc[j];
          const double l0 = pr.lam[2 * j], l1 = pr.lam[2 * j + 1];
          W0 += sgn * l0;
          W1 += sgn * l1;
          W2 += sgn * ((-Rj[1]) * l0 + Rj[0] * l1);
        }
      rf[NQ + 3 * l] = Q.minv_m[l] * W0;
      rf[NQ + 3 * l + 1] = Q.minv_m[l] * W1;
      const double vd2 = Q.minv_I[l] * W2;
      rf[NQ + 3 * l + 2] = vd2;
      pr.vdot[3 * l + 2] = vd2;
    } else if (e < NL + NC) {
      const int ci = e - NL;
      const double ft = pr.u[NA + 2 * ci], fn = pr.u[NA + 2 * ci + 1], gam = pr.u[NA + 2 * NC + ci];
      double* yo = rf + 2 * NQ + 5 * ci;
      yo[0] = fn;
      yo[1] = sabs(pr.lamc[ci]);
      yo[2] = gam;
      yo[3] = sabs(Q.mu[ci] * fn) - sabs(ft);
      yo[4] = srelu(pr.sd[ci]);
    } else if constexpr (M::NGO > 0) {
      constexpr int NG = Prim<M>::NG;
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
        sgv[jg] = srelu(gpl[jg]);
      }
#pragma unroll
      for (int o = 0; o < M::NGO; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int jg = 0; jg < NG; ++jg) acc += P.mix[o][jg] * sgv[jg];
        rf[2 * NQ + 5 * NC + o] = acc;
      }
    }
  }
  for (int k = lane; k < NQ; k += 32) rf[k] = v[k];
  __syncwarp();
  CITO_MARK_P(t, 7);
  // 7: stage bookkeeping
  for (int k = lane; k < NX; k += 32) sh.K[i][k] = S * rf[k];
  for (int k = lane; k < NY; k += 32) sh.ky[k] = (i == 0 ? 0.0 : sh.ky[k]) + P.b[i] * (S * rf[NX + k]);
  for (int k = lane; k < NQ; k += 32) {
    const double vsk = v[k];
    sh.VS[i][k] = vsk;
    R.vs[k] = vsk;
    double ws = 0.0;
    for (int j = 0; j < i; ++j) ws += P.ha[i][j] * sh.VS[j][k];
    R.wq[k] = ws;
  }
  for (int k = lane; k < NR; k += 32) R.r[k] = rf[NQ + k];
  __syncwarp();
  CITO_MARK_P(t, 8);
  if (i == 5) {  // end of substep: x <- x + h sum_i b_i k_i (:209)
    for (int k = lane; k < NQ; k += 32) {
      double ws = 0.0;
      for (int j = 0; j < 6; ++j) ws += P.b[j] * sh.VS[j][k];
      sh.vbs[s & 1][k] = h * ws;
    }
    for (int k = lane; k < NX; k += 32) {
      double inc = 0.0;
      for (int j = 0; j < 6; ++j) inc += P.b[j] * sh.K[j][k];
      sh.x[k] = sh.x[k] + h * inc;
    }
    for (int k = lane; k < NY; k += 32) sh.x[NX + k] = sh.x[NX + k] + h * sh.ky[k];
  }
}

// One tangent column through RK stage I (column warps of k_linearize).
// (one code copy for all six RK stages: the stage index I is runtime and the
// history loops are unrolled to 5 with predication -- keeps the kernel's code
// footprint inside the instruction caches)
template <class M>
__device__ __forceinline__ void col_stage(const KParams& P, FusedShared<M>& sh, int st, const int I, int col, double S,
                                          double dS,
                                          bool isU, int um, bool uplus, double (&hq)[Pos<M::NHIST>::v],
                                          double (&hv)[Pos<M::NHIST>::v]) {
  using D = Dims<M>;
  constexpr int NQ = D::NQ, NR = D::NR, NDIRX = M::NDIRX;
  const int s = st / 6;
  const Rec<M>& R = sh.ring[st % 3];
  const double(*At)[D::NRP] = sh.At[st & 1];
  const double h = P.h;
  const double tau = h * (double)s + P.ch[I];
  const double hb = h * P.b[I];
  if (I == 0) {  // push q rows: S h sum(b) * (substep-start dv)  (warp-uniform branch)
#pragma unroll
    for (int p = 0; p < M::NPUSH; ++p) sh.PQ[p][col] += P.he1 * S * sh.PV[p][col];
  }
  // stage-input tangents along the rate-Jacobian directions: base value, then the
  // history terms in stage order (a runtime loop of I steps over all directions:
  // no predicated dead terms, one small loop body)
  double vals[Pos<NDIRX>::v];
#pragma unroll
  for (int kd = 0; kd < NDIRX; ++kd) {
    const int d = M::dir(kd);
    if (d < NQ) {
      const int hs = M::hslot(d);
      vals[kd] = hq[hs] + S * P.hc1[I] * hv[hs] + dS * R.wq[d];
    } else {
      vals[kd] = hv[M::hslot(d - NQ)];
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
      const double dk = S * accs[j] + dS * R.r[rr];
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
            hq[hs] = hq[hs] + P.he1 * S * hv[hs] + S * incq + dS * sh.vbs[s & 1][rr];
            hv[hs] = hv[hs] + h * incv;
          }
        } else {
          const int p = M::pslot(rr);
          sh.PV[p][col] += hb * dk;
          sh.PQ[p][col] += S * P.e2[I] * dk + dS * hb * R.vs[rr];
        }
      } else {
        sh.DY[rr - NQ][col] += hb * dk;
      }
    }
  }
}

// IPC > 1: IPC intervals per CTA, one 4-warp group each, ticking in lockstep (one
// barrier per tick for all groups), so the groups' same-role warps share one SM
// sub-partition and fetch the same instructions at the same time.
template <class M, int MINB, int IPC = 1>
__global__ void __launch_bounds__(FusedDims<M>::NT * IPC, MINB) k_linearize(const KParams P, int64_t B,
                                                               const double* __restrict__ xt0s,
                                                               const double* __restrict__ Us,
                                                               const double* __restrict__ Ss,
                                                               double* __restrict__ ends, double* __restrict__ jx,
                                                               double* __restrict__ ju, double* __restrict__ js,
                                                               int32_t* __restrict__ bad, const ZSrc zs) {
  using D = Dims<M>;
  constexpr int NQ = D::NQ, NX = D::NX, NU = D::NU, NY = D::NY, NXT = D::NXT, NCOL = D::NCOL;
  constexpr int NDIRX = M::NDIRX, NDIR = D::NDIR, NHIST = M::NHIST;
  constexpr int NT1 = FusedDims<M>::NT;
  constexpr size_t SHB = (sizeof(FusedShared<M>) + 127) / 128 * 128;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int grp = IPC == 1 ? 0 : (int)(threadIdx.x / NT1);
  FusedShared<M>& sh = *reinterpret_cast<FusedShared<M>*>(smem_raw + grp * SHB);
  const int64_t b_raw = (int64_t)blockIdx.x * IPC + grp;
  if (IPC == 1 && b_raw >= B) return;
  const bool active = b_raw < B;  // a spare group recomputes interval B-1 and writes nothing
  const int64_t b = active ? b_raw : B - 1;
#ifndef CITO_BATCH_ROT
#define CITO_BATCH_ROT 1  // rotate the role -> warp slot map per interval group (4096: 1.766 -> 1.744 ms)
#endif
  // role-local thread index; CITO_BATCH_ROT=1 rotates the roles of group g by g warp slots,
  // so the same role of the lockstep groups lands on different SM sub-partitions
  const int slot = (int)((threadIdx.x % NT1) >> 5);
  const int tid = IPC == 1 ? (int)threadIdx.x
                           : (CITO_BATCH_ROT ? ((slot + grp) % (NT1 / 32)) * 32 + (int)(threadIdx.x & 31)
                                             : (int)(threadIdx.x % NT1)),
            warp = tid >> 5, lane = tid & 31;
  // inputs: either packed batches or gathered straight from the decision vector
  // z (cito/scp.py:98-100, layout cito/ocp.py:154-174)
  const int64_t zp = zs.z ? b / zs.n_int : 0, zk = zs.z ? b % zs.n_int : 0;  // problem, interval
  const double* zb = zs.z ? zs.z + zp * zs.zstride : nullptr;
  const double* src_x = zs.z ? zb + (2 * zk + 1) * NXT : xt0s + b * NXT;
  const double* src_U = zs.z ? zb + zs.base_u + zk * (2 * NU + 1) : Us + b * 2 * NU;
  for (int k = tid; k < NXT; k += NT1) sh.x[k] = src_x[k];
  for (int k = tid; k < 2 * NU; k += NT1) sh.U[k] = src_U[k];
  // z may live in page-locked host memory: every read of it is issued here, at once
  if (zs.defects)
    for (int k = tid; k < NXT; k += NT1) sh.xn[k] = zb[(2 * zk + 2) * NXT + k];
  if (tid == 0) {
    sh.S = zs.z ? src_U[2 * NU] : Ss[b];
    sh.bad = 0;
  }
  for (int l = tid; l < M::NL; l += NT1) {
    sh.sp.minv_m[l] = P.minv_m[l];
    sh.sp.minv_I[l] = P.minv_I[l];
    sh.sp.neg_mg[l] = P.neg_mg[l];
  }
  for (int j = tid; j < M::NJ; j += NT1) {
    sh.sp.jrp[j][0] = P.jrp[j][0];
    sh.sp.jrp[j][1] = P.jrp[j][1];
    sh.sp.jrc[j][0] = P.jrc[j][0];
    sh.sp.jrc[j][1] = P.jrc[j][1];
    sh.sp.jk[j] = P.jk[j];
    sh.sp.jd[j] = P.jd[j];
    sh.sp.jrest[j] = P.jrest[j];
    sh.sp.jspring[j] = P.jspring[j];
  }
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < M::NJ; ++j) {
      sh.sp.jp[j] = M::jparent(j);
      sh.sp.jc[j] = M::jchild(j);
      sh.sp.ja[j] = M::jact(j);
      sh.sp.jperm[j] = M::jperm(j);
    }
#pragma unroll
    for (int c = 0; c < M::NC; ++c) sh.sp.cl[c] = M::clink(c);
#pragma unroll
    for (int k = 0; k < M::NBLK; ++k) {
      sh.sp.ba[k] = M::blk_a(k);
      sh.sp.bb[k] = M::blk_b(k);
    }
#pragma unroll
    for (int k = 0; k < M::NLCOL; ++k) sh.sp.lc[k] = M::lcol(k);
  }
  for (int c = tid; c < M::NC; c += NT1) {
    sh.sp.cr[c][0] = P.cr[c][0];
    sh.sp.cr[c][1] = P.cr[c][1];
    sh.sp.mu[c] = P.mu[c];
  }
  // column state: seed = unit column of [x~+ | U- | U+ | S]
  const int col = tid - 64;
  const bool colthr = warp >= 2 && col < NCOL;
  const double dS = (col == NCOL - 1) ? 1.0 : 0.0;
  // state column seeded by this thread (heavy columns only; the closed-form ones
  // are written at the end)
  const int sc = (col >= 0 && col < M::NHCOL) ? M::hcol(col) : -1;
  const int uj = col - M::NHCOL;
  const bool isU = (uj >= 0) && (uj < 2 * NU);
  const int um = isU ? (uj % Pos<NU>::v) : 0;
  const bool uplus = isU && (uj >= NU);
  double hq[Pos<NHIST>::v], hv[Pos<NHIST>::v];  // history coordinates: substep-start values
  if (colthr) {
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const double e_q = (sc == c) ? 1.0 : 0.0, e_v = (sc == NQ + c) ? 1.0 : 0.0;
      if (M::hslot(c) >= 0) {
        hq[M::hslot(c)] = e_q;
        hv[M::hslot(c)] = e_v;
      } else {
        sh.PQ[M::pslot(c)][col] = e_q;
        sh.PV[M::pslot(c)][col] = e_v;
      }
    }
#pragma unroll
    for (int k = 0; k < NY; ++k) sh.DY[k][col] = 0.0;
  }
  __syncthreads();
  const double S = sh.S, h = P.h;
  const int NST = 6 * P.substeps;
  for (int t = 0; t < NST + 2; ++t) {
    CITO_MARK((t * 8 + warp) * 2);
    if (warp == 0) {
      if (t < NST) fused_primal<M>(P, sh, t, lane);
    } else if (warp == 1) {
      if (t >= 1 && t <= NST) {
        const int st = t - 1;
        const Rec<M>& R = sh.ring[st % 3];
        for (int kd = lane; kd < NDIR; kd += 32) {
          const int dir = kd < NDIRX ? M::dir(kd) : NX + (kd - NDIRX);
          tan_rate<M>(P, R.pr, R.vs, dir, &sh.At[st & 1][kd][0], 1);
        }
      }
    } else if (colthr && t >= 2) {
      const int st = t - 2;
      col_stage<M>(P, sh, st, st % 6, col, S, dS, isU, um, uplus, hq, hv);
    }
    CITO_MARK((t * 8 + warp) * 2 + 1);
    __syncthreads();
  }
  // ---- outputs
  double* jxb = jx + b * NXT * NXT;
  double* jub = ju + b * NXT * 2 * NU;
  double* jsb = js + b * NXT;
  if (colthr && active) {
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
      dst[c * stride] = hs >= 0 ? hq[hs] : sh.PQ[M::pslot(c)][col];
      dst[(NQ + c) * stride] = hs >= 0 ? hv[hs] : sh.PV[M::pslot(c)][col];
    }
#pragma unroll
    for (int k = 0; k < NY; ++k) dst[(NX + k) * stride] = sh.DY[k][col];
  }
  if constexpr (M::NLCOL > 0) {  // closed-form columns (state directions no rate reads)
    double dqc = 0.0;  // q-row of a v-column: per substep h * (sum_i b_i S), as the RK recursion computes it
    for (int ss = 0; ss < P.substeps; ++ss) {
      double inc = 0.0;
#pragma unroll
      for (int ii = 0; ii < 6; ++ii) inc += P.b[ii] * S;
      dqc = dqc + h * inc;
    }
    for (int e = active ? tid : M::NLCOL * NXT; e < M::NLCOL * NXT; e += NT1) {
      const int lc = e / NXT, r = e % NXT;
      const int c = sh.sp.lc[lc];
      double val = (r == c) ? 1.0 : 0.0;
      if (c >= NQ && r == c - NQ) val = dqc;
      jxb[r * NXT + c] = val;
    }
  }
  for (int e = active ? tid : NXT * NY; e < NXT * NY; e += NT1) {  // y0 columns of jx: identity (rates ignore y)
    const int r = e / Pos<NY>::v, c = NX + e % Pos<NY>::v;
    jxb[r * NXT + c] = (r == c) ? 1.0 : 0.0;
  }
  for (int k = active ? tid : NXT; k < NXT; k += NT1) {
    const double e = sh.x[k];
    ends[b * NXT + k] = e;
    if (zs.defects) zs.defects[b * NXT + k] = sh.xn[k] - e;  // scp.py:115
    if (!isfinite(e)) sh.bad = 1;
  }
  __syncthreads();
  if (tid == 0 && bad && active) bad[b] = sh.bad;
}
