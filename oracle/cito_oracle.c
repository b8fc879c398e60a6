/*
 * cito_oracle.c — CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * Plain-C restatement of the reference's discretize+linearize algorithm, used
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs, as the checker and the CPU baseline ("port").  It is
 * never linked into the product library.
 *
 * Derivatives are computed the way the reference computes them: dense
 * forward-mode AD (dual numbers carrying all D directions at once), i.e. what
 * jax.jacfwd does over the discrete RKF recursion
 *   (/root/reference/pkg/src/cito/augmentation.py:195-216),
 * including the solve through a dense LU with partial pivoting
 *   (jnp.linalg.solve, cito/contact_dynamics.py:94, :123).
 * The GPU kernel uses a different (explicit rate-Jacobian + tangent
 * recursion) formulation, so agreement between the two is a real check.
 *
 * Pinned against the reference itself: the tests/golden npz fixtures were produced by
 * running the UNMODIFIED reference source (tests/golden/make_golden.py, via
 * oracle/ref_runner.py) and tests/test_oracle_golden.py checks this file
 * against them.
 *
 * Each function cites the reference file:line it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

#include "../include/cito_b200.h"

/* ---------------- tiny pthread parallel-for (no OpenMP runtime in the image) */
typedef void (*pf_body)(void* ctx, int64_t i);
typedef struct {
  pf_body fn;
  void* ctx;
  int64_t n;
  int64_t next;
  pthread_mutex_t mu;
} pf_state;

static void* pf_worker(void* arg) {
  pf_state* st = (pf_state*)arg;
  for (;;) {
    pthread_mutex_lock(&st->mu);
    int64_t i = st->next++;
    pthread_mutex_unlock(&st->mu);
    if (i >= st->n) break;
    st->fn(st->ctx, i);
  }
  return NULL;
}

static int g_threads = 0;
int oracle_set_threads(int n) {
  g_threads = n;
  return n;
}
int oracle_get_threads(void) {
  if (g_threads > 0) return g_threads;
  const char* e = getenv("CITO_ORACLE_THREADS");
  if (e && atoi(e) > 0) return atoi(e);
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void parallel_for(int64_t n, pf_body fn, void* ctx) {
  int nt = oracle_get_threads();
  if (nt > n) nt = (int)n;
  if (n <= 0) return;
  if (nt < 1) nt = 1;
  /* always run on worker threads: with -O3 the inlined dual-number frames exceed
   * the 8 MB main-thread stack */
  pf_state st;
  st.fn = fn;
  st.ctx = ctx;
  st.n = n;
  st.next = 0;
  pthread_mutex_init(&st.mu, NULL);
  pthread_t th[256];
  if (nt > 256) nt = 256;
  pthread_attr_t attr;
  pthread_attr_init(&attr);
  pthread_attr_setstacksize(&attr, (size_t)256 << 20);
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], &attr, pf_worker, &st);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  pthread_attr_destroy(&attr);
  pthread_mutex_destroy(&st.mu);
}

#define MAXD 176

typedef struct {
  double v;
  double d[MAXD];
} dual;

static __thread int ND; /* active directions */

/* Algorithmic-flop counter: when enabled, every
 * dual op counts the flops a structurally sparse forward mode executes -- the
 * value flop(s) plus work only on tangent entries that are nonzero.  Counting
 * convention: + - * / sqrt sin cos = 1, FMA = 2. */
static __thread int COUNT;
static __thread double FLOPS;
static inline int nzd(const double* d, int i) { return d[i] != 0.0; }

static inline dual dc(double c) {
  dual r;
  r.v = c;
  memset(r.d, 0, sizeof(double) * ND);
  return r;
}
static inline dual dadd(dual a, dual b) {
  if (COUNT) {
    FLOPS += 1;
    for (int i = 0; i < ND; ++i) FLOPS += (nzd(a.d, i) && nzd(b.d, i));
  }
  for (int i = 0; i < ND; ++i) a.d[i] += b.d[i];
  a.v += b.v;
  return a;
}
static inline dual dsub(dual a, dual b) {
  if (COUNT) {
    FLOPS += 1;
    for (int i = 0; i < ND; ++i) FLOPS += (nzd(a.d, i) || nzd(b.d, i)) && nzd(b.d, i);
  }
  for (int i = 0; i < ND; ++i) a.d[i] -= b.d[i];
  a.v -= b.v;
  return a;
}
static inline dual dmul(dual a, dual b) {
  dual r;
  if (COUNT) {
    FLOPS += 1;
    for (int i = 0; i < ND; ++i) {
      const int na = nzd(a.d, i), nb = nzd(b.d, i);
      FLOPS += (na && nb) ? 3 : (na || nb);
    }
  }
  r.v = a.v * b.v;
  for (int i = 0; i < ND; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
  return r;
}
static inline dual dscale(dual a, double c) {
  if (COUNT) {
    FLOPS += 1;
    for (int i = 0; i < ND; ++i) FLOPS += nzd(a.d, i);
  }
  a.v *= c;
  for (int i = 0; i < ND; ++i) a.d[i] *= c;
  return a;
}
static inline dual ddiv(dual a, dual b) {
  dual r;
  if (COUNT) {
    FLOPS += 2;
    for (int i = 0; i < ND; ++i) {
      const int na = nzd(a.d, i), nb = nzd(b.d, i);
      FLOPS += nb ? 3 : na;
    }
  }
  r.v = a.v / b.v;
  double ib = 1.0 / b.v;
  for (int i = 0; i < ND; ++i) r.d[i] = (a.d[i] - r.v * b.d[i]) * ib;
  return r;
}
static inline dual dsqrt(dual a) {
  dual r;
  if (COUNT) {
    FLOPS += 2;
    for (int i = 0; i < ND; ++i) FLOPS += nzd(a.d, i);
  }
  r.v = sqrt(a.v);
  double f = 0.5 / r.v;
  for (int i = 0; i < ND; ++i) r.d[i] = a.d[i] * f;
  return r;
}
static inline dual dsin(dual a) {
  dual r;
  if (COUNT) {
    FLOPS += 2;
    for (int i = 0; i < ND; ++i) FLOPS += nzd(a.d, i);
  }
  r.v = sin(a.v);
  double c = cos(a.v);
  for (int i = 0; i < ND; ++i) r.d[i] = a.d[i] * c;
  return r;
}
static inline dual dcos(dual a) {
  dual r;
  if (COUNT) {
    FLOPS += 2;
    for (int i = 0; i < ND; ++i) FLOPS += nzd(a.d, i);
  }
  r.v = cos(a.v);
  double s = -sin(a.v);
  for (int i = 0; i < ND; ++i) r.d[i] = a.d[i] * s;
  return r;
}
static inline dual dneg(dual a) { return dscale(a, -1.0); }

/* ---------------- smooth primitives (cito/smoothmath.py:43-92) ---------- */
static dual smooth_abs(dual x) { /* :43-45 */
  return dsub(dsqrt(dadd(dmul(x, x), dc(1.0))), dc(1.0));
}
static dual smooth_relu(dual x) { /* :60-63 */
  return dscale(dsub(dadd(x, dsqrt(dadd(dmul(x, x), dc(1.0)))), dc(1.0)), 0.5);
}
static dual fb_value(dual a, dual b, double delta) { /* :90-92 */
  return dsub(dadd(a, b), dsqrt(dadd(dadd(dmul(a, a), dmul(b, b)), dc(delta))));
}
static dual snorm_grad_scalar(dual x) { /* cito/contact_dynamics.py:50-52 */
  return ddiv(x, dsqrt(dadd(dmul(x, x), dc(1.0))));
}

/* ---------------- implicit surface h(px,pz) (cito/multibody.py:144-172) -- */
typedef struct {
  double v, gx, gz, hxx, hxz, hzz;
} taylor2;

static taylor2 t2_eval(const cito_model_desc* m, double px, double pz) {
  taylor2 st[CITO_MAX_EXPR];
  int sp = 0;
  for (int k = 0; k < m->expr_len; ++k) {
    int op = m->expr_op[k];
    double arg = m->expr_arg[k];
    taylor2 r = {0, 0, 0, 0, 0, 0};
    if (op == CITO_OP_CONST) {
      r.v = arg;
      st[sp++] = r;
    } else if (op == CITO_OP_PX) {
      r.v = px;
      r.gx = 1.0;
      st[sp++] = r;
    } else if (op == CITO_OP_PZ) {
      r.v = pz;
      r.gz = 1.0;
      st[sp++] = r;
    } else if (op == CITO_OP_ADD) {
      taylor2 b = st[--sp], a = st[--sp];
      r.v = a.v + b.v;
      r.gx = a.gx + b.gx;
      r.gz = a.gz + b.gz;
      r.hxx = a.hxx + b.hxx;
      r.hxz = a.hxz + b.hxz;
      r.hzz = a.hzz + b.hzz;
      st[sp++] = r;
    } else if (op == CITO_OP_MUL) {
      taylor2 b = st[--sp], a = st[--sp];
      r.v = a.v * b.v;
      r.gx = a.gx * b.v + a.v * b.gx;
      r.gz = a.gz * b.v + a.v * b.gz;
      r.hxx = a.hxx * b.v + 2.0 * a.gx * b.gx + a.v * b.hxx;
      r.hxz = a.hxz * b.v + a.gx * b.gz + a.gz * b.gx + a.v * b.hxz;
      r.hzz = a.hzz * b.v + 2.0 * a.gz * b.gz + a.v * b.hzz;
      st[sp++] = r;
    } else if (op == CITO_OP_POW) {
      taylor2 a = st[--sp];
      double n = arg;
      double f0 = pow(a.v, n), f1 = n * pow(a.v, n - 1.0), f2 = n * (n - 1.0) * pow(a.v, n - 2.0);
      r.v = f0;
      r.gx = f1 * a.gx;
      r.gz = f1 * a.gz;
      r.hxx = f1 * a.hxx + f2 * a.gx * a.gx;
      r.hxz = f1 * a.hxz + f2 * a.gx * a.gz;
      r.hzz = f1 * a.hzz + f2 * a.gz * a.gz;
      st[sp++] = r;
    } else if (op == CITO_OP_SIN || op == CITO_OP_COS || op == CITO_OP_LOG || op == CITO_OP_EXP) {
      taylor2 a = st[--sp];
      double f0, f1, f2;
      if (op == CITO_OP_SIN) {
        f0 = sin(a.v);
        f1 = cos(a.v);
        f2 = -f0;
      } else if (op == CITO_OP_LOG) { /* a**b with symbolic b: exp(b log a) */
        f0 = log(a.v);
        f1 = 1.0 / a.v;
        f2 = -f1 * f1;
      } else if (op == CITO_OP_EXP) {
        f0 = exp(a.v);
        f1 = f0;
        f2 = f0;
      } else {
        f0 = cos(a.v);
        f1 = -sin(a.v);
        f2 = -f0;
      }
      r.v = f0;
      r.gx = f1 * a.gx;
      r.gz = f1 * a.gz;
      r.hxx = f1 * a.hxx + f2 * a.gx * a.gx;
      r.hxz = f1 * a.hxz + f2 * a.gx * a.gz;
      r.hzz = f1 * a.hzz + f2 * a.gz * a.gz;
      st[sp++] = r;
    } else if (op == CITO_OP_NEG) {
      taylor2 a = st[--sp];
      r.v = -a.v;
      r.gx = -a.gx;
      r.gz = -a.gz;
      r.hxx = -a.hxx;
      r.hxz = -a.hxz;
      r.hzz = -a.hzz;
      st[sp++] = r;
    }
  }
  return st[0];
}

/* h, grad h at a dual point P (chain rule through the 2nd-order Taylor data) */
static void surface_eval(const cito_model_desc* m, const dual* P, dual* h, dual* gx, dual* gz) {
  if (m->surface_kind == CITO_SURFACE_FLAT) { /* cito/multibody.py:107-121 */
    *h = dsub(P[1], dc(m->surface_height));
    *gx = dc(0.0);
    *gz = dc(1.0);
    return;
  }
  taylor2 t = t2_eval(m, P[0].v, P[1].v);
  h->v = t.v;
  gx->v = t.gx;
  gz->v = t.gz;
  for (int i = 0; i < ND; ++i) {
    h->d[i] = t.gx * P[0].d[i] + t.gz * P[1].d[i];
    gx->d[i] = t.hxx * P[0].d[i] + t.hxz * P[1].d[i];
    gz->d[i] = t.hxz * P[0].d[i] + t.hzz * P[1].d[i];
  }
}

static dual signed_distance_at(const cito_model_desc* m, const dual* P) {
  /* FlatSurface.signed_distance :120-121 ; ImplicitSurface.signed_distance :170-172 */
  dual h, gx, gz;
  surface_eval(m, P, &h, &gx, &gz);
  if (m->surface_kind == CITO_SURFACE_FLAT) return h;
  return ddiv(h, dsqrt(dadd(dmul(gx, gx), dmul(gz, gz))));
}

/* ---------------- kinematics (cito/multibody.py:259-411) ----------------- */
/* world point of a geometric-frame point on a link and its d/dtheta (:264-269) */
static void link_point_rr(const cito_model_desc* m, const dual* q, int link, const double* local, dual* P,
                          dual* dPdth, dual* Rr) {
  double rx = local[0] - m->link_com[link][0];
  double rz = local[1] - m->link_com[link][1];
  dual c = dcos(q[3 * link + 2]), s = dsin(q[3 * link + 2]);
  dual r0 = dsub(dscale(c, rx), dscale(s, rz));
  dual r1 = dadd(dscale(s, rx), dscale(c, rz));
  P[0] = dadd(q[3 * link], r0);
  P[1] = dadd(q[3 * link + 1], r1);
  if (dPdth) {
    dPdth[0] = dsub(dscale(dneg(s), rx), dscale(c, rz));
    dPdth[1] = dsub(dscale(c, rx), dscale(s, rz));
  }
  if (Rr) {
    Rr[0] = r0;
    Rr[1] = r1;
  }
}
static void link_point(const cito_model_desc* m, const dual* q, int link, const double* local, dual* P,
                       dual* dPdth) {
  link_point_rr(m, q, link, local, P, dPdth, NULL);
}

/* contact frame (:384-392): n = g/|g|, t = (n_z, -n_x) */
static void contact_frame(const cito_model_desc* m, const dual* P, dual* n, dual* t) {
  dual h, gx, gz;
  surface_eval(m, P, &h, &gx, &gz);
  dual nrm = dsqrt(dadd(dmul(gx, gx), dmul(gz, gz)));
  n[0] = ddiv(gx, nrm);
  n[1] = ddiv(gz, nrm);
  t[0] = n[1];
  t[1] = dneg(n[0]);
}

/* world contact force -> generalized force on the owning link (jac.T @ F) */
static void add_link_wrench(const cito_model_desc* m, dual* w, int link, const dual* dPdth, dual F0,
                            dual F1) {
  (void)m;
  w[3 * link] = dadd(w[3 * link], F0);
  w[3 * link + 1] = dadd(w[3 * link + 1], F1);
  w[3 * link + 2] = dadd(w[3 * link + 2], dadd(dmul(dPdth[0], F0), dmul(dPdth[1], F1)));
}

/* _contact_wrench (cito/contact_dynamics.py:76-83); forces (n_c, 2) = (phi_t, phi_n) */
static void contact_wrench(const cito_model_desc* m, const dual* q, const dual* forces, dual* w) {
  for (int i = 0; i < m->n_contacts; ++i) {
    int l = m->contact_link[i];
    dual P[2], dP[2], n[2], t[2];
    link_point(m, q, l, m->contact_offset[i], P, dP);
    contact_frame(m, P, n, t);
    /* rot @ f = t*f_t + n*f_n */
    dual F0 = dadd(dmul(t[0], forces[2 * i]), dmul(n[0], forces[2 * i + 1]));
    dual F1 = dadd(dmul(t[1], forces[2 * i]), dmul(n[1], forces[2 * i + 1]));
    add_link_wrench(m, w, l, dP, F0, F1);
  }
}

/* joint constraint Jacobian (dense n_j x n_q) and curvature (:324-358) */
static void joint_jacobian(const cito_model_desc* m, const dual* q, const dual* v, dual* J, dual* curv) {
  int nq = 3 * m->n_links;
  for (int r = 0; r < 2 * m->n_joints * nq; ++r) J[r] = dc(0.0);
  for (int j = 0; j < m->n_joints; ++j) {
    int p = m->joint_parent[j], c = m->joint_child[j];
    dual Pc[2], dPc[2], Rc[2];
    link_point_rr(m, q, c, m->joint_child_anchor[j], Pc, dPc, Rc);
    dual* Jx = J + (2 * j) * nq;
    dual* Jz = J + (2 * j + 1) * nq;
    /* c_j = P_parent - P_child */
    Jx[3 * c] = dc(-1.0);
    Jz[3 * c + 1] = dc(-1.0);
    Jx[3 * c + 2] = dneg(dPc[0]);
    Jz[3 * c + 2] = dneg(dPc[1]);
    /* curvature: -R(th_p) r_p w_p^2 + R(th_c) r_c w_c^2; R r = P - p */
    const int wc = curv != NULL;
    dual cx, cz;
    if (wc) {
      dual wc2 = dmul(v[3 * c + 2], v[3 * c + 2]);
      cx = dmul(Rc[0], wc2);
      cz = dmul(Rc[1], wc2);
    }
    if (p >= 0) {
      dual Pp[2], dPp[2], Rp[2];
      link_point_rr(m, q, p, m->joint_parent_anchor[j], Pp, dPp, Rp);
      Jx[3 * p] = dc(1.0);
      Jz[3 * p + 1] = dc(1.0);
      Jx[3 * p + 2] = dPp[0];
      Jz[3 * p + 2] = dPp[1];
      if (wc) {
        dual wp2 = dmul(v[3 * p + 2], v[3 * p + 2]);
        cx = dsub(cx, dmul(Rp[0], wp2));
        cz = dsub(cz, dmul(Rp[1], wp2));
      }
    }
    if (curv) {
      curv[2 * j] = cx;
      curv[2 * j + 1] = cz;
    }
  }
}

/* dense LU with partial pivoting, solve G x = rhs in place (jnp.linalg.solve) */
static void lu_solve(int n, dual* G, dual* rhs) {
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = fabs(G[k * n + k].v);
    for (int i = k + 1; i < n; ++i)
      if (fabs(G[i * n + k].v) > best) {
        best = fabs(G[i * n + k].v);
        piv = i;
      }
    if (piv != k) {
      for (int j = 0; j < n; ++j) {
        dual tmp = G[k * n + j];
        G[k * n + j] = G[piv * n + j];
        G[piv * n + j] = tmp;
      }
      dual tmp = rhs[k];
      rhs[k] = rhs[piv];
      rhs[piv] = tmp;
    }
    for (int i = k + 1; i < n; ++i) {
      dual f = ddiv(G[i * n + k], G[k * n + k]);
      for (int j = k + 1; j < n; ++j) G[i * n + j] = dsub(G[i * n + j], dmul(f, G[k * n + j]));
      rhs[i] = dsub(rhs[i], dmul(f, rhs[k]));
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    dual s = rhs[i];
    for (int j = i + 1; j < n; ++j) s = dsub(s, dmul(G[i * n + j], rhs[j]));
    rhs[i] = ddiv(s, G[i * n + i]);
  }
}

/* _eliminate_joint_forces (cito/contact_dynamics.py:86-95) / impact_map (:111-124):
 * out = base + minv*(w + J^T phi), phi = -G^{-1}(J (base_or_0 + minv*w) + curv) */
static void eliminate(const cito_model_desc* m, const dual* q, const dual* v, const dual* w, int impact,
                      const dual* vminus, dual* out) {
  int nq = 3 * m->n_links, nj = 2 * m->n_joints;
  double minv[3 * CITO_MAX_LINKS];
  for (int l = 0; l < m->n_links; ++l) {
    minv[3 * l] = 1.0 / m->link_mass[l];
    minv[3 * l + 1] = 1.0 / m->link_mass[l];
    minv[3 * l + 2] = 1.0 / m->link_inertia[l];
  }
  dual mw[3 * CITO_MAX_LINKS];
  for (int i = 0; i < nq; ++i) mw[i] = dscale(w[i], minv[i]);
  if (nj == 0) {
    for (int i = 0; i < nq; ++i) out[i] = impact ? dadd(vminus[i], mw[i]) : mw[i];
    return;
  }
  dual* J = (dual*)malloc(sizeof(dual) * nj * nq);
  dual* G = (dual*)malloc(sizeof(dual) * nj * nj);
  dual curv[2 * CITO_MAX_JOINTS], rhs[2 * CITO_MAX_JOINTS];
  joint_jacobian(m, q, v, J, impact ? NULL : curv);
  for (int a = 0; a < nj; ++a)
    for (int b = 0; b < nj; ++b) {
      dual s = dc(0.0);
      for (int k = 0; k < nq; ++k) s = dadd(s, dmul(J[a * nq + k], dscale(J[b * nq + k], minv[k])));
      G[a * nj + b] = s;
    }
  for (int a = 0; a < nj; ++a) {
    dual s = dc(0.0);
    for (int k = 0; k < nq; ++k) {
      dual term = impact ? dadd(vminus[k], mw[k]) : mw[k];
      s = dadd(s, dmul(J[a * nq + k], term));
    }
    rhs[a] = impact ? s : dadd(s, curv[a]);
  }
  lu_solve(nj, G, rhs);
  for (int k = 0; k < nq; ++k) {
    dual s = w[k];
    for (int a = 0; a < nj; ++a) s = dsub(s, dmul(J[a * nq + k], rhs[a])); /* phi = -x */
    dual acc = dscale(s, minv[k]);
    out[k] = impact ? dadd(vminus[k], acc) : acc;
  }
  free(J);
  free(G);
}

/* generalized_forces (cito/multibody.py:285-321) */
static void generalized_forces(const cito_model_desc* m, const dual* q, const dual* v, const dual* tau,
                               dual* w) {
  int nq = 3 * m->n_links;
  for (int i = 0; i < nq; ++i) w[i] = dc(0.0);
  for (int l = 0; l < m->n_links; ++l) w[3 * l + 1] = dadd(w[3 * l + 1], dc(-m->link_mass[l] * m->gravity));
  int act = 0;
  for (int j = 0; j < m->n_joints; ++j) {
    int p = m->joint_parent[j], c = m->joint_child[j];
    dual th_c = q[3 * c + 2], om_c = v[3 * c + 2];
    dual th_p = p >= 0 ? q[3 * p + 2] : dc(0.0);
    dual om_p = p >= 0 ? v[3 * p + 2] : dc(0.0);
    dual mo = dc(0.0);
    if (m->joint_actuated[j]) mo = dadd(mo, tau[act++]);
    if (m->joint_spring[j]) {
      dual rel = dsub(dsub(th_c, th_p), dc(m->joint_rest[j]));
      mo = dsub(dsub(mo, dscale(rel, m->joint_stiffness[j])), dscale(dsub(om_c, om_p), m->joint_damping[j]));
    }
    w[3 * c + 2] = dadd(w[3 * c + 2], mo);
    if (p >= 0) w[3 * p + 2] = dadd(w[3 * p + 2], dneg(mo));
  }
}

static int n_act(const cito_model_desc* m) {
  int a = 0;
  for (int j = 0; j < m->n_joints; ++j) a += m->joint_actuated[j] ? 1 : 0;
  return a;
}

static int n_path(const cito_model_desc* m) {
  return m->n_contacts + 2 * m->n_joint_limits + 2 * m->n_height_bounds;
}

/* augmented_rate (cito/augmentation.py:156-163) WITHOUT the factor S:
 * out = [v; vdot; Omega] (n_xt).  forward_dynamics cito/contact_dynamics.py:98-108,
 * aux_rate cito/augmentation.py:134-153, path g cito/augmentation.py:112-129. */
static void rate_unscaled(const cito_model_desc* m, const dual* x, const dual* u, dual* out) {
  int nq = 3 * m->n_links, nc = m->n_contacts, na = n_act(m);
  const dual* q = x;
  const dual* v = x + nq;
  const dual* tau = u;
  const dual* phi = u + na;
  const dual* gam = u + na + 2 * nc;
  dual w[3 * CITO_MAX_LINKS] = {{0}};
  generalized_forces(m, q, v, tau, w);
  if (nc) contact_wrench(m, q, phi, w);
  for (int i = 0; i < nq; ++i) out[i] = v[i];
  eliminate(m, q, v, w, 0, NULL, out + nq);
  dual* y = out + 2 * nq;
  dual sd[CITO_MAX_CONTACTS];
  for (int i = 0; i < nc; ++i) {
    int l = m->contact_link[i];
    dual P[2], dP[2], n[2], t[2];
    link_point(m, q, l, m->contact_offset[i], P, dP);
    contact_frame(m, P, n, t);
    /* friction_stationarity (cito/contact_dynamics.py:55-66) */
    dual Jv0 = dadd(v[3 * l], dmul(dP[0], v[3 * l + 2]));
    dual Jv1 = dadd(v[3 * l + 1], dmul(dP[1], v[3 * l + 2]));
    dual vt = dadd(dmul(t[0], Jv0), dmul(t[1], Jv1));
    dual lam = dadd(vt, dmul(gam[i], snorm_grad_scalar(phi[2 * i])));
    /* friction_cone_residual (:69-73) */
    dual rho = dsub(smooth_abs(dscale(phi[2 * i + 1], m->contact_mu[i])), smooth_abs(phi[2 * i]));
    sd[i] = signed_distance_at(m, P);
    y[5 * i + 0] = phi[2 * i + 1];
    y[5 * i + 1] = smooth_abs(lam);
    y[5 * i + 2] = gam[i];
    y[5 * i + 3] = rho;
    y[5 * i + 4] = smooth_relu(sd[i]);
  }
  if (m->n_g_out > 0) {
    int ng = n_path(m);
    dual g[CITO_MAX_PATH];
    int r = 0;
    for (int i = 0; i < nc; ++i) g[r++] = dneg(sd[i]);
    for (int k = 0; k < m->n_joint_limits; ++k) {
      int jj = m->jl_joint[k];
      int p = m->joint_parent[jj], c = m->joint_child[jj];
      dual rel = p >= 0 ? dsub(q[3 * c + 2], q[3 * p + 2]) : dsub(q[3 * c + 2], dc(0.0));
      g[r++] = dsub(rel, dc(m->jl_hi[k]));
      g[r++] = dsub(dc(m->jl_lo[k]), rel);
    }
    for (int k = 0; k < m->n_height_bounds; ++k) {
      dual pz = q[3 * m->hb_link[k] + 1];
      g[r++] = dsub(dc(m->hb_lo[k]), pz);
      g[r++] = dsub(pz, dc(m->hb_hi[k]));
    }
    dual sg[CITO_MAX_PATH];
    for (int j = 0; j < ng; ++j) sg[j] = smooth_relu(g[j]);
    for (int o = 0; o < m->n_g_out; ++o) {
      dual s = dc(0.0);
      for (int j = 0; j < ng; ++j) s = dadd(s, dscale(sg[j], m->mixing[o * CITO_MAX_PATH + j]));
      y[5 * nc + o] = s;
    }
  }
}

/* RKF tableau (cito/augmentation.py:46-56) */
static const double RKF_C[6] = {0.0, 1.0 / 4, 3.0 / 8, 12.0 / 13, 1.0, 1.0 / 2};
static const double RKF_A[6][5] = {{0},
                                   {1.0 / 4},
                                   {3.0 / 32, 9.0 / 32},
                                   {1932.0 / 2197, -7200.0 / 2197, 7296.0 / 2197},
                                   {439.0 / 216, -8.0, 3680.0 / 513, -845.0 / 4104},
                                   {-8.0 / 27, 2.0, -3544.0 / 2565, 1859.0 / 4104, -11.0 / 40}};
static const double RKF_B[6] = {16.0 / 135, 0.0, 6656.0 / 12825, 28561.0 / 56430, -9.0 / 50, 2.0 / 55};

/* flow (cito/augmentation.py:195-211) in dual arithmetic; seeds all D directions */
static void flow_interval(const cito_model_desc* m, int substeps, const double* xt0, const double* U,
                          double S, int with_tangents, double* end, double* jx, double* ju, double* js) {
  int nq = 3 * m->n_links, nc = m->n_contacts, na = n_act(m);
  int nu = na + 3 * nc;
  int ny = 5 * nc + m->n_g_out;
  int nxt = 2 * nq + ny;
  int D = with_tangents ? nxt + 2 * nu + 1 : 0;
  ND = D;
  dual* xt = (dual*)malloc(sizeof(dual) * nxt);
  dual* xs = (dual*)malloc(sizeof(dual) * nxt);
  dual* ks = (dual*)malloc(sizeof(dual) * 6 * nxt);
  dual* Ud = (dual*)malloc(sizeof(dual) * 2 * nu);
  dual* uu = (dual*)malloc(sizeof(dual) * nu);
  dual Sd = dc(S);
  for (int i = 0; i < nxt; ++i) {
    xt[i] = dc(xt0[i]);
    if (D) xt[i].d[i] = 1.0;
  }
  for (int i = 0; i < 2 * nu; ++i) {
    Ud[i] = dc(U[i]);
    if (D) Ud[i].d[nxt + i] = 1.0;
  }
  if (D) Sd.d[nxt + 2 * nu] = 1.0;
  double h = 1.0 / substeps;
  for (int s = 0; s < substeps; ++s) {
    double tau0 = h * (double)s;
    for (int st = 0; st < 6; ++st) {
      for (int i = 0; i < nxt; ++i) {
        dual acc = xt[i];
        for (int j = 0; j < st; ++j) acc = dadd(acc, dscale(ks[j * nxt + i], h * RKF_A[st][j]));
        xs[i] = acc;
      }
      double tau = tau0 + RKF_C[st] * h;
      for (int i = 0; i < nu; ++i) /* foh_eval (:166-169) */
        uu[i] = dadd(dscale(Ud[i], 1.0 - tau), dscale(Ud[nu + i], tau));
      rate_unscaled(m, xs, uu, ks + st * nxt);
      for (int i = 0; i < nxt; ++i) ks[st * nxt + i] = dmul(Sd, ks[st * nxt + i]);
    }
    for (int i = 0; i < nxt; ++i) {
      dual inc = dc(0.0);
      for (int st = 0; st < 6; ++st) inc = dadd(inc, dscale(ks[st * nxt + i], RKF_B[st]));
      xt[i] = dadd(xt[i], dscale(inc, h));
    }
  }
  for (int i = 0; i < nxt; ++i) {
    end[i] = xt[i].v;
    if (D) {
      for (int c = 0; c < nxt; ++c) jx[i * nxt + c] = xt[i].d[c];
      for (int c = 0; c < 2 * nu; ++c) ju[i * 2 * nu + c] = xt[i].d[nxt + c];
      js[i] = xt[i].d[nxt + 2 * nu];
    }
  }
  free(xt);
  free(xs);
  free(ks);
  free(Ud);
  free(uu);
}

static void dims(const cito_model_desc* m, int* nq, int* nu, int* ny, int* nxt) {
  *nq = 3 * m->n_links;
  *nu = n_act(m) + 3 * m->n_contacts;
  *ny = 5 * m->n_contacts + m->n_g_out;
  *nxt = 2 * *nq + *ny;
}

typedef struct {
  const cito_model_desc* m;
  int substeps, tangents, nxt, nu;
  const double *xt0s, *Us, *Ss;
  double *ends, *jx, *ju, *js;
  int32_t* bad;
} flow_ctx;

static void flow_body(void* vctx, int64_t b) {
  flow_ctx* c = (flow_ctx*)vctx;
  int nxt = c->nxt, nu = c->nu;
  flow_interval(c->m, c->substeps, c->xt0s + b * nxt, c->Us + b * 2 * nu, c->Ss[b], c->tangents,
                c->ends + b * nxt, c->tangents ? c->jx + b * nxt * nxt : NULL,
                c->tangents ? c->ju + b * nxt * 2 * nu : NULL, c->tangents ? c->js + b * nxt : NULL);
  int ok = 1;
  for (int i = 0; i < nxt; ++i) ok &= isfinite(c->ends[b * nxt + i]) ? 1 : 0;
  c->bad[b] = !ok;
}

static int run_flows(const cito_model_desc* m, int substeps, int tangents, int64_t B, const double* xt0s,
                     const double* Us, const double* Ss, double* ends, double* jx, double* ju, double* js,
                     int32_t* bad) {
  int nq, nu, ny, nxt;
  dims(m, &nq, &nu, &ny, &nxt);
  flow_ctx c = {m, substeps, tangents, nxt, nu, xt0s, Us, Ss, ends, jx, ju, js, bad};
  parallel_for(B, flow_body, &c);
  int nbad = 0;
  for (int64_t b = 0; b < B; ++b) nbad += bad[b];
  return nbad;
}

/* Discretizer.linearize_batch (cito/augmentation.py:236-242); returns #nonfinite ends */
int oracle_linearize(const cito_model_desc* m, int substeps, int64_t B, const double* xt0s, const double* Us,
                     const double* Ss, double* ends, double* jx, double* ju, double* js, int32_t* bad) {
  return run_flows(m, substeps, 1, B, xt0s, Us, Ss, ends, jx, ju, js, bad);
}

/* Discretizer.propagate_batch (cito/augmentation.py:226-234) */
int oracle_propagate(const cito_model_desc* m, int substeps, int64_t B, const double* xt0s, const double* Us,
                     const double* Ss, double* ends, int32_t* bad) {
  return run_flows(m, substeps, 0, B, xt0s, Us, Ss, ends, NULL, NULL, NULL, bad);
}

/* ---------------- node relations (cito/ocp.py:277-303) ------------------ */
/* psi_fn (:277-287) with its jacobian over the y pair */
static void psi_one(const cito_model_desc* m, const double* ypair, double delta, double eps, double* psi,
                    double* jac) {
  int nc = m->n_contacts, ny = 5 * nc + m->n_g_out;
  ND = 2 * ny;
  dual yp[2 * (5 * CITO_MAX_CONTACTS + CITO_MAX_GOUT)];
  for (int i = 0; i < 2 * ny; ++i) {
    yp[i] = dc(ypair[i]);
    yp[i].d[i] = 1.0;
  }
  int r = 0;
  dual rows[3 * CITO_MAX_CONTACTS + CITO_MAX_GOUT];
  for (int i = 0; i < nc; ++i) {
    dual d[5];
    for (int k = 0; k < 5; ++k) d[k] = dsub(yp[ny + 5 * i + k], yp[5 * i + k]);
    rows[r++] = fb_value(d[0], d[4], delta);
    rows[r++] = fb_value(d[0], d[1], delta);
    rows[r++] = fb_value(d[2], d[3], delta);
  }
  for (int i = 0; i < m->n_g_out; ++i) rows[r++] = dsub(dsub(yp[ny + 5 * nc + i], yp[5 * nc + i]), dc(eps));
  for (int a = 0; a < r; ++a) {
    psi[a] = rows[a].v;
    for (int c = 0; c < 2 * ny; ++c) jac[a * 2 * ny + c] = rows[a].d[c];
  }
}

/* theta_fn (:289-296) -> impact_residuals (cito/contact_dynamics.py:134-172) */
static void theta_one(const cito_model_desc* m, const double* vec, double delta, double* th, double* jac) {
  int nq = 3 * m->n_links, nc = m->n_contacts;
  int nv = 3 * nq + 3 * nc;
  ND = nv;
  dual x[3 * 3 * CITO_MAX_LINKS + 3 * CITO_MAX_CONTACTS];
  for (int i = 0; i < nv; ++i) {
    x[i] = dc(vec[i]);
    x[i].d[i] = 1.0;
  }
  const dual* q = x;
  const dual* vm = x + nq;
  const dual* vp = x + 2 * nq;
  const dual* Phi = x + 3 * nq;
  const dual* Gam = x + 3 * nq + 2 * nc;
  dual rows[6 * CITO_MAX_CONTACTS];
  for (int i = 0; i < nc; ++i) {
    int l = m->contact_link[i];
    dual P[2], dP[2], n[2], t[2];
    link_point(m, q, l, m->contact_offset[i], P, dP);
    contact_frame(m, P, n, t);
    dual sd = signed_distance_at(m, P);
    double e = m->contact_restitution[i];
    dual va[3], vb[3];
    for (int k = 0; k < 3; ++k) {
      va[k] = dadd(vp[3 * l + k], dscale(vm[3 * l + k], e));
      vb[k] = vp[3 * l + k];
    }
    dual Ja0 = dadd(va[0], dmul(dP[0], va[2])), Ja1 = dadd(va[1], dmul(dP[1], va[2]));
    dual Jb0 = dadd(vb[0], dmul(dP[0], vb[2])), Jb1 = dadd(vb[1], dmul(dP[1], vb[2]));
    dual vn_rest = dadd(dmul(n[0], Ja0), dmul(n[1], Ja1));
    dual vt_plus = dadd(dmul(t[0], Jb0), dmul(t[1], Jb1));
    dual Pt = Phi[2 * i], Pn = Phi[2 * i + 1];
    dual cone = dsub(smooth_abs(dscale(Pn, m->contact_mu[i])), smooth_abs(Pt));
    rows[2 * i] = dmul(Pn, vn_rest);
    rows[2 * i + 1] = dmul(Pn, dadd(vt_plus, dmul(Gam[i], snorm_grad_scalar(Pt))));
    rows[2 * nc + 4 * i + 0] = fb_value(Pn, sd, delta);
    rows[2 * nc + 4 * i + 1] = fb_value(Gam[i], cone, delta);
    rows[2 * nc + 4 * i + 2] = dneg(sd);
    rows[2 * nc + 4 * i + 3] = dneg(vn_rest);
  }
  for (int a = 0; a < 6 * nc; ++a) {
    th[a] = rows[a].v;
    for (int c = 0; c < nv; ++c) jac[a * nv + c] = rows[a].d[c];
  }
}

/* impulse_fn (:298-303) -> impact_map (cito/contact_dynamics.py:111-124) */
static void impulse_one(const cito_model_desc* m, const double* vec, double* imp, double* jac) {
  int nq = 3 * m->n_links, nc = m->n_contacts;
  int nv = 3 * nq + 2 * nc;
  ND = nv;
  dual x[3 * 3 * CITO_MAX_LINKS + 2 * CITO_MAX_CONTACTS];
  for (int i = 0; i < nv; ++i) {
    x[i] = dc(vec[i]);
    x[i].d[i] = 1.0;
  }
  const dual* q = x;
  const dual* vm = x + nq;
  const dual* vp = x + 2 * nq;
  const dual* Phi = x + 3 * nq;
  dual w[3 * CITO_MAX_LINKS] = {{0}}, vplus[3 * CITO_MAX_LINKS];
  if (nc) contact_wrench(m, q, Phi, w);
  eliminate(m, q, NULL, w, 1, vm, vplus);
  for (int a = 0; a < nq; ++a) {
    dual r = dsub(vp[a], vplus[a]);
    imp[a] = r.v;
    for (int c = 0; c < nv; ++c) jac[a * nv + c] = r.d[c];
  }
}

typedef struct {
  const cito_model_desc* m;
  int64_t Np;
  const double *y_pairs, *theta_vecs;
  double delta, eps;
  double *psi, *psi_jac, *theta, *theta_jac, *imp, *imp_jac;
} node_ctx;

static void node_body(void* vctx, int64_t k) {
  node_ctx* c = (node_ctx*)vctx;
  const cito_model_desc* m = c->m;
  int nq = 3 * m->n_links, nc = m->n_contacts, ny = 5 * nc + m->n_g_out;
  int npsi = 3 * nc + m->n_g_out;
  int nv = 3 * nq + 3 * nc, ni = 3 * nq + 2 * nc;
  if (k < c->Np) {
    psi_one(m, c->y_pairs + k * 2 * ny, c->delta, c->eps, c->psi + k * npsi, c->psi_jac + k * npsi * 2 * ny);
  } else {
    k -= c->Np;
    theta_one(m, c->theta_vecs + k * nv, c->delta, c->theta + k * 6 * nc, c->theta_jac + k * 6 * nc * nv);
    impulse_one(m, c->theta_vecs + k * nv, c->imp + k * nq, c->imp_jac + k * nq * ni);
  }
}

/* Transcription.node_constraints + node_jacobians, batched (cito/ocp.py:336-365) */
void oracle_node_linearize(const cito_model_desc* m, int64_t Np, int64_t Nn, const double* y_pairs,
                           const double* theta_vecs, double delta, double eps, double* psi, double* psi_jac,
                           double* theta, double* theta_jac, double* imp, double* imp_jac) {
  node_ctx c = {m, Np, y_pairs, theta_vecs, delta, eps, psi, psi_jac, theta, theta_jac, imp, imp_jac};
  parallel_for(Np + Nn, node_body, &c);
}

int oracle_max_directions(void) { return MAXD; }

typedef struct {
  const cito_model_desc* m;
  int substeps;
  const double *xt0, *U;
  double S, flops;
} count_ctx;

static double count_flops_impl(const cito_model_desc* m, int substeps, const double* xt0, const double* U,
                               double S);
static void count_body(void* v, int64_t i) {
  (void)i;
  count_ctx* c = (count_ctx*)v;
  c->flops = count_flops_impl(c->m, c->substeps, c->xt0, c->U, c->S);
}

/* structurally-sparse forward-mode flops of ONE interval linearization */
double oracle_count_flops(const cito_model_desc* m, int substeps, const double* xt0, const double* U, double S) {
  count_ctx c = {m, substeps, xt0, U, S, 0.0};
  parallel_for(1, count_body, &c); /* worker thread: large stack */
  return c.flops;
}

static double count_flops_impl(const cito_model_desc* m, int substeps, const double* xt0, const double* U,
                               double S) {
  int nq, nu, ny, nxt;
  dims(m, &nq, &nu, &ny, &nxt);
  double* end = (double*)malloc(sizeof(double) * nxt);
  double* jx = (double*)malloc(sizeof(double) * nxt * nxt);
  double* ju = (double*)malloc(sizeof(double) * nxt * 2 * nu + 8);
  double* js = (double*)malloc(sizeof(double) * nxt);
  COUNT = 1;
  FLOPS = 0.0;
  flow_interval(m, substeps, xt0, U, S, 1, end, jx, ju, js);
  COUNT = 0;
  free(end);
  free(jx);
  free(ju);
  free(js);
  return FLOPS;
}
