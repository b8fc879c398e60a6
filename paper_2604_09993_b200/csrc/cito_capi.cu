// cito_capi.cu — C ABI (include/cito_b200.h) over the sm_100a kernels.
//
// Replaces the jit/vmap plumbing of cito.augmentation.Discretizer
// (/root/reference/pkg/src/cito/augmentation.py:180-242): a handle caches the
// per-(model, mixing, path spec, substeps) kernel selection and parameters the
// way the reference caches its jitted closures.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/cito_b200.h"
#include "cito_kernels.cuh"
#include "cito_k1v2.cuh"
#include "cito_node.cuh"
#include "cito_scatter.cuh"
#include "cito_bench.cuh"
#include "cito_subproblem.cuh"

namespace {

thread_local std::string g_err;
int64_t g_launches = 0;  // every kernel launched by this library (evidence for bench.py's gpu_launches)
inline void count_launch(int64_t n = 1) { __atomic_add_fetch(&g_launches, n, __ATOMIC_RELAXED); }

cito_status fail(cito_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) return fail(CITO_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

// RKF tableau (cito/augmentation.py:46-56)
const double RKF_C[6] = {0.0, 1.0 / 4, 3.0 / 8, 12.0 / 13, 1.0, 1.0 / 2};
const double RKF_A[6][5] = {{0},
                            {1.0 / 4},
                            {3.0 / 32, 9.0 / 32},
                            {1932.0 / 2197, -7200.0 / 2197, 7296.0 / 2197},
                            {439.0 / 216, -8.0, 3680.0 / 513, -845.0 / 4104},
                            {-8.0 / 27, 2.0, -3544.0 / 2565, 1859.0 / 4104, -11.0 / 40}};
const double RKF_B[6] = {16.0 / 135, 0.0, 6656.0 / 12825, 28561.0 / 56430, -9.0 / 50, 2.0 / 55};

struct TopoOps {
  const char* key;
  cito_status (*linearize)(const KParams&, int64_t, const double*, const double*, const double*, double*, double*,
                           double*, double*, int32_t*, cudaStream_t, ZSrc);
  cito_status (*propagate)(const KParams&, int64_t, const double*, const double*, const double*, double*, int32_t*,
                           cudaStream_t);
  cito_status (*node)(const KParams&, int64_t, int64_t, const double*, const double*, double, double, double*,
                      double*, double*, double*, double*, double*, cudaStream_t, ZSrc);
  cito_status (*audit)(const KParams&, int64_t, const double*, int64_t, const double*, double*, double*, double*,
                       cudaStream_t);
};

// K1 selection.  Default (auto): k_linearize2 (cito_k1v2.cuh: short primal chain,
// off-chain aux warp, q/v and u Jacobian warps) while the grid fits the SMs once
// -- the latency case of one SCP iteration -- and k_linearize<M, 3> (cito_kernels.cuh,
// 4 warps, 3 CTAs/SM) for batches, where its smaller footprint gives more
// throughput.  CITO_K1=1 / CITO_K1=2 force one generation for A/B measurements.
static int k1_version() {
  static int v = [] {
    const char* e = getenv("CITO_K1");
    return (e && e[0] == '1') ? 1 : (e && e[0] == '2') ? 2 : 0;
  }();
  return v;
}

// Opt a kernel into `bytes` of dynamic shared memory once; false if the device
// cannot give a CTA that much (large topologies: the multi-interval batch
// variants are then skipped).
template <class K>
static bool smem_ok(K kernel, size_t bytes) {
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  if (bytes > (size_t)optin) return false;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
}

template <class M>
cito_status launch_linearize(const KParams& P, int64_t B, const double* xt0s, const double* Us, const double* Ss,
                             double* ends, double* jx, double* ju, double* js, int32_t* bad, cudaStream_t st,
                             ZSrc zs) {
  if (B <= 0) return CITO_OK;
  const size_t smem1 = sizeof(FusedShared<M>), smem2 = sizeof(Fused2Shared<M>);
  const size_t sm1r = (smem1 + 127) / 128 * 128;
  // which variants fit this topology's shared-memory footprint (decided once per topology)
  static const bool ok_b1 = smem_ok(k_linearize<M, 1>, smem1), ok_b3 = smem_ok(k_linearize<M, 3>, smem1);
  static const bool ok_l2 = smem_ok(k_linearize<M, 1, 2>, 2 * sm1r), ok_l3 = smem_ok(k_linearize<M, 1, 3>, 3 * sm1r);
  static const bool ok_v2 = smem_ok(k_linearize2<M, 1>, smem2), ok_v22 = smem_ok(k_linearize2<M, 2>, smem2);
  if (!ok_b1 && !ok_v2) return fail(CITO_ERR_UNSUPPORTED, "topology needs more shared memory than a CTA can have");
  // latency variant (full register budget) while the grid fits the SMs once,
  // occupancy variant for large batches
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  count_launch();
  const int ver = k1_version();
  // batches up to lat_max intervals use the latency kernel, one CTA per SM; above
  // ~2/3 of the SMs the lockstep 3-interval batch kernel is faster (measured
  // crossover 96..120 intervals on 148 SMs: instruction fetch)
  static const int64_t lat_max = getenv("CITO_K1_LAT_MAX") ? atoll(getenv("CITO_K1_LAT_MAX")) : -1;
  const int64_t lmax = lat_max >= 0 ? lat_max : (2 * (int64_t)sms) / 3;
  if (ok_v2 && (ver == 2 || (ver == 0 && B <= lmax) || !ok_b1)) {
    if (B <= sms || !ok_v22) {
      // programmatic dependent launch (CITO_PDL=0 turns it off): behind a kernel that
      // produces the inputs (the SCP graph's z upload) the CTAs start and load the model
      // constants early; they wait for the producer before reading any input
      static const bool pdl = !(getenv("CITO_PDL") && getenv("CITO_PDL")[0] == '0');
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)B);
      cfg.blockDim = dim3(K2Dims<M>::NT);
      cfg.dynamicSmemBytes = smem2;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      CUDA_TRY(cudaLaunchKernelEx(&cfg, k_linearize2<M, 1>, P, B, xt0s, Us, Ss, ends, jx, ju, js, bad, zs));
    } else {
      k_linearize2<M, 2><<<(unsigned)B, K2Dims<M>::NT, smem2, st>>>(P, B, xt0s, Us, Ss, ends, jx, ju, js, bad, zs);
    }
  } else if (ver == 1 && B <= sms) {
    k_linearize<M, 1><<<(unsigned)B, FusedDims<M>::NT, smem1, st>>>(P, B, xt0s, Us, Ss, ends, jx, ju, js, bad, zs);
  } else {
    // three intervals per CTA in lockstep (same-role warps share an SM sub-partition and
    // fetch the same instructions); CITO_K1_IPC1=1: one interval per CTA, 3 CTAs/SM
    static const bool ipc3 = getenv("CITO_K1_IPC1") == nullptr;
    // two lockstep intervals per CTA while that keeps at most ~1.65 waves of CTAs
    // (measured crossover with three per CTA at 245..250 intervals on 148 SMs)
    static const int64_t ipc2_env = getenv("CITO_K1_IPC2_MAX") ? atoll(getenv("CITO_K1_IPC2_MAX")) : -1;
    const int64_t ipc2_max = ipc2_env >= 0 ? ipc2_env : (5 * (int64_t)sms) / 3;
    if (ipc3 && ok_l2 && (B <= ipc2_max || !ok_l3))
      k_linearize<M, 1, 2><<<(unsigned)((B + 1) / 2), 2 * FusedDims<M>::NT, 2 * sm1r, st>>>(
          P, B, xt0s, Us, Ss, ends, jx, ju, js, bad, zs);
    else if (ipc3 && ok_l3)
      k_linearize<M, 1, 3><<<(unsigned)((B + 2) / 3), 3 * FusedDims<M>::NT, 3 * sm1r, st>>>(
          P, B, xt0s, Us, Ss, ends, jx, ju, js, bad, zs);
    else
      k_linearize<M, 3><<<(unsigned)B, FusedDims<M>::NT, smem1, st>>>(P, B, xt0s, Us, Ss, ends, jx, ju, js, bad, zs);
  }
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

// Propagate: a warp-pair CTA per interval (k_linearize2<M, 1, false>: critical
// chain + off-chain warp, ~2x lower latency) while the grid fits the SMs once,
// else one thread per interval (k_primal, throughput).
template <class M>
cito_status launch_propagate(const KParams& P, int64_t B, const double* xt0s, const double* Us, const double* Ss,
                             double* ends, int32_t* bad, cudaStream_t st) {
  if (B <= 0) return CITO_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  count_launch();
  const size_t smem = sizeof(Fused2Shared<M>);
  static const bool ok_pair = smem_ok(k_linearize2<M, 1, false>, smem);
  if (B <= sms && k1_version() != 1 && ok_pair) {
    k_linearize2<M, 1, false><<<(unsigned)B, 64, smem, st>>>(P, B, xt0s, Us, Ss, ends, nullptr, nullptr, nullptr, bad,
                                                             ZSrc{});
  } else {
    const int nt = 64;
    k_primal<M><<<(unsigned)((B + nt - 1) / nt), nt, 0, st>>>(P, B, xt0s, Us, Ss, ends, bad);
  }
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

template <class M>
cito_status launch_node(const KParams& P, int64_t Np, int64_t Nn, const double* y_pairs, const double* theta_vecs,
                        double delta, double eps, double* psi, double* psi_jac, double* th, double* th_jac,
                        double* imp, double* imp_jac, cudaStream_t st, ZSrc zs) {
  constexpr int NQ = 3 * M::NL, NC = M::NC, NY = 5 * NC + M::NGO;
  const int64_t total = Np * (2 * NY) + Nn * (3 * NQ + 3 * NC) + Nn * (3 * NQ + 2 * NC);
  if (total <= 0) return CITO_OK;
  count_launch();
  // warp per item (k_node_w) by default; CITO_K3=1: thread per (item, direction) (k_node)
  static const bool thread_per_dir = getenv("CITO_K3") && getenv("CITO_K3")[0] == '1';
  const size_t tsm = (size_t)K3W_WARPS * NodeTile<M>::N * sizeof(double);
  static const bool ok_w = smem_ok(k_node_w<M>, tsm);
  if (!thread_per_dir && ok_w) {
    const int64_t warps = Np + 2 * Nn;
    k_node_w<M><<<(unsigned)((warps + K3W_WARPS - 1) / K3W_WARPS), 32 * K3W_WARPS, tsm, st>>>(
        P, Np, Nn, y_pairs, theta_vecs, delta, eps, psi, psi_jac, th, th_jac, imp, imp_jac, zs);
  } else {
    const int nt = 64;
    k_node<M><<<(unsigned)((total + nt - 1) / nt), nt, 0, st>>>(P, Np, Nn, y_pairs, theta_vecs, delta, eps, psi,
                                                                 psi_jac, th, th_jac, imp, imp_jac, zs);
  }
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

template <class M>
cito_status launch_audit(const KParams& P, int64_t B, const double* xs, int64_t xstride, const double* us,
                         double* sds, double* cj, double* omega, cudaStream_t st) {
  if (B <= 0) return CITO_OK;
  const int nt = 64;
  count_launch();
  k_audit<M><<<(unsigned)((B + nt - 1) / nt), nt, 0, st>>>(P, B, xs, xstride, us, sds, cj, omega);
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

#define CITO_TOPO_ENTRY(T, K) {K, launch_linearize<T>, launch_propagate<T>, launch_node<T>, launch_audit<T>},
const TopoOps kTopos[] = {CITO_FOR_EACH_TOPOLOGY(CITO_TOPO_ENTRY)};
#undef CITO_TOPO_ENTRY

std::string topo_key(const cito_model_desc& d) {
  std::string k = "L" + std::to_string(d.n_links) + "|J";
  for (int j = 0; j < d.n_joints; ++j) {
    if (j) k += ",";
    k += std::to_string(d.joint_parent[j]) + ">" + std::to_string(d.joint_child[j]) +
         (d.joint_actuated[j] ? "a" : "p");
  }
  k += "|C";
  for (int i = 0; i < d.n_contacts; ++i) {
    if (i) k += ",";
    k += std::to_string(d.contact_link[i]);
  }
  k += std::string("|S") + (d.surface_kind == CITO_SURFACE_IMPLICIT ? "i" : "f");
  k += "|G" + std::to_string(d.n_g_out) + "|JL";
  for (int i = 0; i < d.n_joint_limits; ++i) {
    if (i) k += ",";
    k += std::to_string(d.jl_joint[i]);
  }
  k += "|HB";
  for (int i = 0; i < d.n_height_bounds; ++i) {
    if (i) k += ",";
    k += std::to_string(d.hb_link[i]);
  }
  return k;
}

}  // namespace

struct cito_handle {
  cito_model_desc desc;
  KParams P;
  cito_dims dims;
  const TopoOps* ops = nullptr;
  std::mutex mu;
  // device staging for the *_host entry points
  void* dbuf = nullptr;
  size_t dcap = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;  // concurrent node-relation kernel of linearize_all
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaStream_t cstream = nullptr;      // D2H stream of the chunked *_host pipeline
  std::vector<cudaEvent_t> chunk_ev;  // one per in-flight chunk
  int64_t launches = 0;
};

extern "C" {

const char* cito_last_error(void) { return g_err.c_str(); }
const char* cito_version(void) { return "paper_2604_09993_b200 0.1 (sm_100a fp64)"; }

cito_status cito_create(const cito_model_desc* desc, int32_t substeps, cito_handle** out) {
  if (!desc || !out) return fail(CITO_ERR_ARG, "null argument");
  if (substeps < 1) return fail(CITO_ERR_ARG, "substeps must be >= 1");
  const cito_model_desc& d = *desc;
  if (d.n_links < 1 || d.n_links > KMAX_L || d.n_joints > KMAX_J || d.n_contacts > KMAX_C)
    return fail(CITO_ERR_ARG, "model size outside kernel limits");
  const int n_g = d.n_contacts + 2 * d.n_joint_limits + 2 * d.n_height_bounds;
  if (d.n_g_out > KMAX_GO || (d.n_g_out > 0 && n_g > KMAX_G))
    return fail(CITO_ERR_ARG, "too many path-constraint rows for the kernel parameter block");
  if (d.surface_kind == CITO_SURFACE_IMPLICIT && (d.expr_len < 1 || d.expr_len > KMAX_E))
    return fail(CITO_ERR_ARG, "implicit surface byte-code missing or too long");
  const std::string key = topo_key(d);
  const TopoOps* ops = nullptr;
  for (const auto& t : kTopos)
    if (key == t.key) ops = &t;
  if (!ops) return fail(CITO_ERR_UNSUPPORTED, "model topology not compiled into this library: " + key);

  cito_handle* h = new cito_handle();
  h->desc = d;
  h->ops = ops;
  KParams& P = h->P;
  memset(&P, 0, sizeof(P));
  for (int l = 0; l < d.n_links; ++l) {
    P.minv_m[l] = 1.0 / d.link_mass[l];
    P.minv_I[l] = 1.0 / d.link_inertia[l];
    P.neg_mg[l] = -d.link_mass[l] * d.gravity;  // multibody.py:300
  }
  for (int j = 0; j < d.n_joints; ++j) {
    const int p = d.joint_parent[j], c = d.joint_child[j];
    for (int a = 0; a < 2; ++a) {
      P.jrp[j][a] = p >= 0 ? d.joint_parent_anchor[j][a] - d.link_com[p][a] : d.joint_parent_anchor[j][a];
      P.jrc[j][a] = d.joint_child_anchor[j][a] - d.link_com[c][a];
    }
    P.jk[j] = d.joint_stiffness[j];
    P.jd[j] = d.joint_damping[j];
    P.jrest[j] = d.joint_rest[j];
    P.jspring[j] = d.joint_spring[j];
  }
  for (int i = 0; i < d.n_contacts; ++i) {
    const int l = d.contact_link[i];
    for (int a = 0; a < 2; ++a) P.cr[i][a] = d.contact_offset[i][a] - d.link_com[l][a];
    P.mu[i] = d.contact_mu[i];
    P.crest[i] = d.contact_restitution[i];
  }
  P.height = d.surface_height;
  for (int k = 0; k < d.n_joint_limits; ++k) {
    P.jl_lo[k] = d.jl_lo[k];
    P.jl_hi[k] = d.jl_hi[k];
  }
  for (int k = 0; k < d.n_height_bounds; ++k) {
    P.hb_lo[k] = d.hb_lo[k];
    P.hb_hi[k] = d.hb_hi[k];
  }
  for (int o = 0; o < d.n_g_out; ++o)
    for (int g = 0; g < n_g; ++g) P.mix[o][g] = d.mixing[o * CITO_MAX_PATH + g];
  P.expr_len = d.expr_len;
  for (int k = 0; k < d.expr_len; ++k) {
    P.expr_op[k] = d.expr_op[k];
    P.expr_arg[k] = d.expr_arg[k];
  }
  // tableau products for h = 1/substeps
  const double hh = 1.0 / substeps;
  P.substeps = substeps;
  P.h = hh;
  for (int i = 0; i < 6; ++i) {
    P.ch[i] = RKF_C[i] * hh;
    P.b[i] = RKF_B[i];
    double c1 = 0.0;
    for (int j = 0; j < i; ++j) {
      P.ha[i][j] = hh * RKF_A[i][j];
      c1 += RKF_A[i][j];
    }
    P.hc1[i] = hh * c1;
    for (int l = 0; l < i; ++l) {
      double s = 0.0;
      for (int j = l + 1; j < i; ++j) s += RKF_A[i][j] * RKF_A[j][l];
      P.cq[i][l] = hh * hh * s;
    }
  }
  double e1 = 0.0;
  for (int i = 0; i < 6; ++i) e1 += RKF_B[i];
  P.he1 = hh * e1;
  for (int l = 0; l < 6; ++l) {
    double s = 0.0;
    for (int i = l + 1; i < 6; ++i) s += RKF_B[i] * RKF_A[i][l];
    P.e2[l] = hh * hh * s;
  }
  // dims (cito/augmentation.py:267-269, cito/contact_dynamics.py:35-37)
  int na = 0;
  for (int j = 0; j < d.n_joints; ++j) na += d.joint_actuated[j] ? 1 : 0;
  cito_dims& D = h->dims;
  D.n_q = 3 * d.n_links;
  D.n_x = 2 * D.n_q;
  D.n_a = na;
  D.n_u = na + 3 * d.n_contacts;
  D.n_y = 5 * d.n_contacts + d.n_g_out;
  D.n_xt = D.n_x + D.n_y;
  D.n_j = 2 * d.n_joints;
  D.n_g = n_g;
  D.D = D.n_xt + 2 * D.n_u + 1;
  // the private stream of the *_host entry points is created on first use, so a
  // handle (topology lookup, dims) can be created on a machine without a GPU
  *out = h;
  return CITO_OK;
}

cito_status cito_destroy(cito_handle* h) {
  if (!h) return CITO_OK;
  if (h->dbuf) cudaFree(h->dbuf);
  if (h->stream) cudaStreamDestroy(h->stream);
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  for (cudaEvent_t e : h->chunk_ev) cudaEventDestroy(e);
  delete h;
  return CITO_OK;
}

cito_status cito_get_dims(const cito_handle* h, cito_dims* out) {
  if (!h || !out) return fail(CITO_ERR_ARG, "null argument");
  *out = h->dims;
  return CITO_OK;
}

int64_t cito_launch_count(const cito_handle* h) { return h ? h->launches : g_launches; }

cito_status cito_linearize_dev(cito_handle* h, int64_t B, const double* xt0s, const double* Us, const double* Ss,
                               double* ends, double* jx, double* ju, double* js, int32_t* bad, void* stream) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  cito_status st = h->ops->linearize(h->P, B, xt0s, Us, Ss, ends, jx, ju, js, bad, (cudaStream_t)stream, ZSrc{});
  if (st == CITO_OK && B > 0) __atomic_add_fetch(&h->launches, 1, __ATOMIC_RELAXED);
  return st;
}

cito_status cito_propagate_dev(cito_handle* h, int64_t B, const double* xt0s, const double* Us, const double* Ss,
                               double* ends, int32_t* bad, void* stream) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  cito_status st = h->ops->propagate(h->P, B, xt0s, Us, Ss, ends, bad, (cudaStream_t)stream);
  if (st == CITO_OK && B > 0) __atomic_add_fetch(&h->launches, 1, __ATOMIC_RELAXED);
  return st;
}

cito_status cito_node_linearize_dev(cito_handle* h, int64_t Np, int64_t Nn, const double* y_pairs,
                                    const double* theta_vecs, double delta, double epsilon, double* psi,
                                    double* psi_jac, double* theta, double* theta_jac, double* imp, double* imp_jac,
                                    void* stream) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  cito_status st = h->ops->node(h->P, Np, Nn, y_pairs, theta_vecs, delta, epsilon, psi, psi_jac, theta, theta_jac,
                                imp, imp_jac, (cudaStream_t)stream, ZSrc{});
  if (st == CITO_OK && Np + Nn > 0) __atomic_add_fetch(&h->launches, 1, __ATOMIC_RELAXED);
  return st;
}

cito_status cito_audit_dev(cito_handle* h, int64_t B, const double* xs, int64_t xstride, const double* us,
                           double* sds, double* cj, double* omega, void* stream) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  if (B < 0 || xstride < h->dims.n_x) return fail(CITO_ERR_ARG, "audit: bad batch/stride");
  cito_status st = h->ops->audit(h->P, B, xs, xstride, us, sds, cj, omega, (cudaStream_t)stream);
  if (st == CITO_OK && B > 0) __atomic_add_fetch(&h->launches, 1, __ATOMIC_RELAXED);
  return st;
}

static cito_status ensure_dbuf(cito_handle* h, size_t bytes) {
  if (!h->stream) CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  if (bytes <= h->dcap) return CITO_OK;
  if (h->dbuf) cudaFree(h->dbuf);
  h->dbuf = nullptr;
  h->dcap = 0;
  CUDA_TRY(cudaMalloc(&h->dbuf, bytes));
  h->dcap = bytes;
  return CITO_OK;
}

static size_t al256(size_t n) { return (n + 255) & ~size_t(255); }

static cito_status count_bad(const int32_t* bad, int64_t B) {
  if (!bad) return CITO_OK;
  for (int64_t b = 0; b < B; ++b)
    if (bad[b]) return fail(CITO_ERR_NONFINITE, "non-finite state during interval integration");
  return CITO_OK;
}

cito_status cito_linearize_host(cito_handle* h, int64_t B, const double* xt0s, const double* Us, const double* Ss,
                                double* ends, double* jx, double* ju, double* js, int32_t* bad) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  if (B <= 0) return CITO_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  const cito_dims& D = h->dims;
  const size_t nin = al256(B * D.n_xt * 8) + al256(B * 2 * D.n_u * 8) + al256(B * 8);
  const size_t nout = al256(B * D.n_xt * 8) + al256(B * D.n_xt * D.n_xt * 8) +
                      al256(B * D.n_xt * 2 * D.n_u * 8) + al256(B * D.n_xt * 8) + al256(B * 4);
  cito_status st = ensure_dbuf(h, nin + nout);
  if (st != CITO_OK) return st;
  char* p = (char*)h->dbuf;
  double* d_x = (double*)p;
  p += al256(B * D.n_xt * 8);
  double* d_U = (double*)p;
  p += al256(B * 2 * D.n_u * 8);
  double* d_S = (double*)p;
  p += al256(B * 8);
  double* d_e = (double*)p;
  p += al256(B * D.n_xt * 8);
  double* d_jx = (double*)p;
  p += al256(B * D.n_xt * D.n_xt * 8);
  double* d_ju = (double*)p;
  p += al256(B * D.n_xt * 2 * D.n_u * 8);
  double* d_js = (double*)p;
  p += al256(B * D.n_xt * 8);
  int32_t* d_bad = (int32_t*)p;
  cudaStream_t s = h->stream;
  CUDA_TRY(cudaMemcpyAsync(d_x, xt0s, B * D.n_xt * 8, cudaMemcpyHostToDevice, s));
  if (D.n_u) CUDA_TRY(cudaMemcpyAsync(d_U, Us, B * 2 * D.n_u * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_S, Ss, B * 8, cudaMemcpyHostToDevice, s));
  // Large batches run as a pipeline of one-wave chunks (3 intervals per CTA x #SMs, the
  // last chunk takes the remainder): all chunk launches are queued on `s` first, then
  // each chunk's results are copied back on `cstream` as soon as its kernel is done, so
  // the D2H of chunk c overlaps the kernels of chunks c+1.. (with pageable destinations
  // the copy calls block the host, which is why the launches are issued before them).
  // CITO_HOST_CHUNKS=0 disables the pipeline (A/B).
  static const bool chunked = !(getenv("CITO_HOST_CHUNKS") && atoi(getenv("CITO_HOST_CHUNKS")) == 0);
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t wave = 3 * (int64_t)sms;
  const int64_t chunk = (chunked && B >= 4 * wave) ? wave : B;
  const int64_t nch = B / chunk;
  const int64_t nx = D.n_xt, nu2 = 2 * D.n_u;
  if (nch > 1) {
    if (!h->cstream) CUDA_TRY(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    while ((int64_t)h->chunk_ev.size() < nch) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->chunk_ev.push_back(e);
    }
  }
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t b0 = c * chunk, nb = (c == nch - 1) ? B - b0 : chunk;
    st = h->ops->linearize(h->P, nb, d_x + b0 * nx, d_U + b0 * nu2, d_S + b0, d_e + b0 * nx, d_jx + b0 * nx * nx,
                           d_ju + b0 * nx * nu2, d_js + b0 * nx, d_bad + b0, s, ZSrc{});
    if (st != CITO_OK) return st;
    h->launches++;
    if (nch > 1) CUDA_TRY(cudaEventRecord(h->chunk_ev[c], s));
  }
  cudaStream_t cs = nch > 1 ? h->cstream : s;
  int32_t* hb = bad;
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t b0 = c * chunk, nb = (c == nch - 1) ? B - b0 : chunk;
    if (nch > 1) CUDA_TRY(cudaStreamWaitEvent(cs, h->chunk_ev[c], 0));
    CUDA_TRY(cudaMemcpyAsync(ends + b0 * nx, d_e + b0 * nx, nb * nx * 8, cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaMemcpyAsync(jx + b0 * nx * nx, d_jx + b0 * nx * nx, nb * nx * nx * 8, cudaMemcpyDeviceToHost, cs));
    if (D.n_u)
      CUDA_TRY(cudaMemcpyAsync(ju + b0 * nx * nu2, d_ju + b0 * nx * nu2, nb * nx * nu2 * 8, cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaMemcpyAsync(js + b0 * nx, d_js + b0 * nx, nb * nx * 8, cudaMemcpyDeviceToHost, cs));
    if (hb) CUDA_TRY(cudaMemcpyAsync(hb + b0, d_bad + b0, nb * 4, cudaMemcpyDeviceToHost, cs));
  }
  CUDA_TRY(cudaStreamSynchronize(cs));
  CUDA_TRY(cudaStreamSynchronize(s));
  return count_bad(hb, B);
}

cito_status cito_propagate_host(cito_handle* h, int64_t B, const double* xt0s, const double* Us, const double* Ss,
                                double* ends, int32_t* bad) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  if (B <= 0) return CITO_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  const cito_dims& D = h->dims;
  const size_t n1 = al256(B * D.n_xt * 8), n2 = al256(B * 2 * D.n_u * 8 + 8), n3 = al256(B * 8);
  cito_status st = ensure_dbuf(h, 2 * n1 + n2 + n3 + al256(B * 4));
  if (st != CITO_OK) return st;
  char* p = (char*)h->dbuf;
  double* d_x = (double*)p;
  double* d_U = (double*)(p + n1);
  double* d_S = (double*)(p + n1 + n2);
  double* d_e = (double*)(p + n1 + n2 + n3);
  int32_t* d_bad = (int32_t*)(p + 2 * n1 + n2 + n3);
  cudaStream_t s = h->stream;
  CUDA_TRY(cudaMemcpyAsync(d_x, xt0s, B * D.n_xt * 8, cudaMemcpyHostToDevice, s));
  if (D.n_u) CUDA_TRY(cudaMemcpyAsync(d_U, Us, B * 2 * D.n_u * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_S, Ss, B * 8, cudaMemcpyHostToDevice, s));
  st = h->ops->propagate(h->P, B, d_x, d_U, d_S, d_e, d_bad, s);
  if (st != CITO_OK) return st;
  h->launches++;
  CUDA_TRY(cudaMemcpyAsync(ends, d_e, B * D.n_xt * 8, cudaMemcpyDeviceToHost, s));
  if (bad) CUDA_TRY(cudaMemcpyAsync(bad, d_bad, B * 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return count_bad(bad, B);
}

static cito_status linearize_all_impl(cito_handle* h, int32_t N, int32_t n_problems, int64_t zstride, int64_t base_u,
                                      int64_t base_p, const double* z, double delta, double epsilon,
                                      const double* d_delta_eps, double* ends, double* jx, double* ju, double* js,
                                      double* defects, int32_t* bad, double* psi, double* psi_jac, double* theta,
                                      double* theta_jac, double* imp, double* imp_jac, void* stream) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  if (N < 2) return fail(CITO_ERR_ARG, "need at least two grid nodes");
  if (n_problems < 1) return fail(CITO_ERR_ARG, "n_problems must be >= 1");
  const int64_t P = n_problems;
  cudaStream_t s = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(h->mu);
  if (!h->aux) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
  }
  const ZSrc zs{z, base_u, base_p, defects, zstride, N - 1, N, d_delta_eps};
  // node relations (K3) on the auxiliary stream, concurrently with the interval kernel (K1).
  // K1 is enqueued first (CITO_K3_FIRST=1 restores the old order for A/B): its CTAs are
  // dispatched first and K3's fill the SMs K1 leaves idle (its last partial wave)
  static const bool k3_first = getenv("CITO_K3_FIRST") && atoi(getenv("CITO_K3_FIRST")) == 1;
  CUDA_TRY(cudaEventRecord(h->ev_in, s));
  CUDA_TRY(cudaStreamWaitEvent(h->aux, h->ev_in, 0));
  cito_status st;
  if (!k3_first) {
    st = h->ops->linearize(h->P, P * (N - 1), nullptr, nullptr, nullptr, ends, jx, ju, js, bad, s, zs);
    if (st != CITO_OK) return st;
  }
  st = h->ops->node(h->P, P * (N - 1), P * N, nullptr, nullptr, delta, epsilon, psi, psi_jac, theta, theta_jac, imp,
                    imp_jac, h->aux, zs);
  if (st != CITO_OK) return st;
  CUDA_TRY(cudaEventRecord(h->ev_out, h->aux));
  if (k3_first) {
    st = h->ops->linearize(h->P, P * (N - 1), nullptr, nullptr, nullptr, ends, jx, ju, js, bad, s, zs);
    if (st != CITO_OK) return st;
  }
  CUDA_TRY(cudaStreamWaitEvent(s, h->ev_out, 0));
  __atomic_add_fetch(&h->launches, 2, __ATOMIC_RELAXED);
  return CITO_OK;
}

cito_status cito_linearize_all_dev(cito_handle* h, int32_t N, int32_t n_problems, int64_t zstride, int64_t base_u,
                                   int64_t base_p, const double* z, double delta, double epsilon, double* ends, double* jx, double* ju, double* js,
                                   double* defects, int32_t* bad, double* psi, double* psi_jac, double* theta,
                                   double* theta_jac, double* imp, double* imp_jac, void* stream) {
  return linearize_all_impl(h, N, n_problems, zstride, base_u, base_p, z, delta, epsilon, nullptr, ends, jx, ju, js,
                            defects, bad, psi, psi_jac, theta, theta_jac, imp, imp_jac, stream);
}

cito_status cito_linearize_all_dev2(cito_handle* h, int32_t N, int32_t n_problems, int64_t zstride, int64_t base_u,
                                    int64_t base_p, const double* z, const double* d_delta_eps, double* ends,
                                    double* jx, double* ju, double* js, double* defects, int32_t* bad, double* psi,
                                    double* psi_jac, double* theta, double* theta_jac, double* imp, double* imp_jac,
                                    void* stream) {
  if (!d_delta_eps) return fail(CITO_ERR_ARG, "null delta/epsilon pointer");
  return linearize_all_impl(h, N, n_problems, zstride, base_u, base_p, z, 0.0, 0.0, d_delta_eps, ends, jx, ju, js,
                            defects, bad, psi, psi_jac, theta, theta_jac, imp, imp_jac, stream);
}

cito_status cito_scatter_dynamics_dev(cito_handle* h, int64_t n_int, const double* ends, const double* jx,
                                      const double* ju, const double* js, const double* z_ref, const int64_t* xp_off,
                                      const int64_t* u_off, const int64_t* s_off, const double* sig_x,
                                      const double* sig_u, double sig_s, const int32_t* slot_x,
                                      const int32_t* slot_u, const int32_t* slot_s, double* A_data, double* b_rows,
                                      int32_t* mismatch, void* stream) {
  if (!h) return fail(CITO_ERR_ARG, "null handle");
  if (n_int <= 0) return CITO_OK;
  const cito_dims& D = h->dims;
  const int nt = 128;
  const int64_t rows = n_int * D.n_xt;
  count_launch();
  k_scatter_dynamics<<<(unsigned)((rows + nt / 32 - 1) / (nt / 32)), nt, 0, (cudaStream_t)stream>>>(
      n_int, D.n_xt, D.n_u, ends, jx, ju, js, z_ref, xp_off, u_off, s_off, sig_x, sig_u, sig_s, slot_x, slot_u,
      slot_s, A_data, b_rows, mismatch);
  CUDA_TRY(cudaGetLastError());
  __atomic_add_fetch(&h->launches, 1, __ATOMIC_RELAXED);
  return CITO_OK;
}

cito_status cito_csc_assemble2_dev(int32_t nmat, int32_t ncols, const int64_t* const* sp_ptr,
                                   const int32_t* const* sp_row, const int8_t* const* sp_src,
                                   const int64_t* const* sp_idx, const double* const* sp_val, const double* sigma,
                                   const double* const* lin, int32_t* const* counts, int32_t* const* out_ptr,
                                   int32_t* const* out_rows, double* const* out_vals,
                                   unsigned long long* const* rowmax, void* stream) {
  if (ncols <= 0 || nmat < 1 || nmat > 2) return nmat == 0 ? CITO_OK : fail(CITO_ERR_ARG, "nmat must be 1 or 2");
  LinTable L;
  for (int k = 0; k < 10; ++k) L.p[k] = lin ? lin[k] : nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  const int wpb = 8;
  const unsigned gx = (unsigned)((ncols + wpb - 1) / wpb);
  CscArgs ca;
  ScanArgs sa;
  for (int m = 0; m < nmat; ++m) {
    ca.sp_ptr[m] = sp_ptr[m];
    ca.row[m] = sp_row[m];
    ca.src[m] = sp_src[m];
    ca.idx[m] = sp_idx[m];
    ca.val[m] = sp_val[m];
    ca.counts[m] = counts[m];
    ca.out_ptr[m] = out_ptr[m];
    ca.out_rows[m] = out_rows[m];
    ca.out_vals[m] = out_vals[m];
    ca.rowmax[m] = rowmax ? rowmax[m] : nullptr;
    sa.n[m] = ncols;
    sa.counts[m] = counts[m];
    sa.out_ptr[m] = out_ptr[m];
  }
  // two launches: per-block nonzero totals (into the counts workspace), then
  // prefix + per-column scan + compacted write (CITO_CSC3=1: the older three-launch
  // count / scan / write sequence)
  static const bool three = getenv("CITO_CSC3") != nullptr;
  if (three) {
    count_launch(3);
    k_csc_count<<<dim3(gx, nmat), 32 * wpb, 0, s>>>(ncols, ca, sigma, L);
    CUDA_TRY(cudaGetLastError());
    k_scan<<<nmat, 1024, 0, s>>>(sa);
    CUDA_TRY(cudaGetLastError());
    k_csc_write<<<dim3(gx, nmat), 32 * wpb, 0, s>>>(ncols, ca, sigma, L);
    CUDA_TRY(cudaGetLastError());
    return CITO_OK;
  }
  (void)gx;
  const unsigned nb = (unsigned)((ncols + CSC_CPB - 1) / CSC_CPB);
  static const bool two = getenv("CITO_CSC2") != nullptr;  // A/B: block totals + write (two launches)
  if (two) {
    count_launch(2);
    k_csc_blocksum<<<dim3(nb, nmat), 256, 0, s>>>(ncols, ca, sigma, L);
    CUDA_TRY(cudaGetLastError());
    k_csc_write2<<<dim3(nb, nmat), 256, 0, s>>>(ncols, ca, sigma, L);
    CUDA_TRY(cudaGetLastError());
    return CITO_OK;
  }
  count_launch(1);
  k_csc_onepass<<<dim3(nb, nmat), 256, 0, s>>>(ncols, ca, sigma, L);
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

cito_status cito_csc_assemble_packed_dev(int32_t nmat, int32_t ncols, const void* const* ent, const int64_t* nsup,
                                        const int64_t* const* sp_ptr, const int32_t* const* tcol, const int32_t* ntile,
                                        const double* const* lin, uint32_t* ws, int64_t ws_words,
                                        int32_t* const* out_ptr, int32_t* const* out_rows, double* const* out_vals,
                                        unsigned long long* const* rowmax, const double* stamp_in,
                                        double* changed_at, int64_t host_vals, int64_t host_pattern,
                                        const double* rows_wanted, const double* consts_wanted, void* stream) {
  if (nmat < 1 || nmat > 2 || ncols < 0 || !ent || !nsup || !sp_ptr || !tcol || !ntile || !ws ||
      (stamp_in == nullptr) != (changed_at == nullptr))
    return fail(CITO_ERR_ARG, "csc_assemble_packed: bad arguments");
  CscPackedArgs a;
  a.stamp_in = stamp_in;
  a.changed_at = changed_at;
  if (host_pattern && !rows_wanted)
    return fail(CITO_ERR_ARG, "csc_assemble_packed: host_pattern needs rows_wanted");
  a.host_vals = host_vals;
  a.host_pattern = host_pattern;
  a.rows_wanted = rows_wanted;
  a.consts_wanted = consts_wanted;
  int64_t tiles = 0;
  for (int m = 0; m < 2; ++m) {
    const bool on = m < nmat;
    a.ent[m] = on ? (const CscEnt*)ent[m] : nullptr;
    a.nsup[m] = on ? nsup[m] : 0;
    a.sp_ptr[m] = on ? sp_ptr[m] : nullptr;
    a.tcol[m] = on ? tcol[m] : nullptr;
    a.ntile[m] = on ? ntile[m] : 0;
    a.out_ptr[m] = on ? out_ptr[m] : nullptr;
    a.out_rows[m] = on ? out_rows[m] : nullptr;
    a.out_vals[m] = on ? out_vals[m] : nullptr;
    a.rowmax[m] = (on && rowmax) ? rowmax[m] : nullptr;
    if (on && (ntile[m] < 1 || (int64_t)ntile[m] * CSC_TILE < nsup[m] || nsup[m] >= (1ll << 27)))
      return fail(CITO_ERR_ARG, "csc_assemble_packed: tile count does not cover the entries");
    tiles += on ? ntile[m] : 0;
  }
  if (ws_words < CSC_HDR_WORDS + 2 * tiles) return fail(CITO_ERR_ARG, "csc_assemble_packed: workspace too small");
  LinTable L;
  for (int k = 0; k < 10; ++k) L.p[k] = lin ? lin[k] : nullptr;
  count_launch(1);
  // programmatic dependent launch (CITO_PDL=0 turns it off): the tiles take their tickets
  // and load their records while the producing kernel (K1) finishes
  static const bool pdl = !(getenv("CITO_PDL") && getenv("CITO_PDL")[0] == '0');
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)tiles);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k_csc_flat, ncols, a, L, ws));
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

cito_status cito_csc_assemble_dev(int32_t ncols, const int64_t* sp_ptr, const int32_t* sp_row, const int8_t* sp_src,
                                  const int64_t* sp_idx, const double* sp_val, const double* sigma,
                                  const double* const* lin, int32_t* counts, int32_t* out_ptr, int32_t* out_rows,
                                  double* out_vals, void* stream) {
  return cito_csc_assemble2_dev(1, ncols, &sp_ptr, &sp_row, &sp_src, &sp_idx, &sp_val, sigma, lin, &counts, &out_ptr,
                                &out_rows, &out_vals, nullptr, stream);
}

cito_status cito_rhs_dev(int64_t nrows, const int32_t* rows, const int8_t* form, const int8_t* vsrc,
                         const int64_t* voff, const int8_t* seg_src, const int64_t* seg_off, const int32_t* seg_len,
                         const int64_t* seg_cb, const int64_t* cols, const double* z, const double* const* lin,
                         double* out, int64_t host, void* stream) {
  if (nrows <= 0) return CITO_OK;
  LinTable L;
  for (int k = 0; k < 10; ++k) L.p[k] = lin ? lin[k] : nullptr;
  const int wpb = 8;
  count_launch();
  k_rhs<<<(unsigned)((nrows + wpb - 1) / wpb), 32 * wpb, 0, (cudaStream_t)stream>>>(
      nrows, rows, form, vsrc, voff, seg_src, seg_off, seg_len, seg_cb, cols, z, L, out, host);
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

cito_status cito_precondition_dev(int32_t ncols, const int32_t* A_ptr, const int32_t* A_rows, double* A_data,
                                  int32_t nA, double* b, const int32_t* G_ptr, const int32_t* G_rows, double* G_data,
                                  int32_t nG, double* h, int32_t n_nonneg, int32_t n_soc, const int32_t* soc_start,
                                  const int32_t* soc_dim, unsigned long long* rowmax_A, unsigned long long* rowmax_G,
                                  int32_t rowmax_ready, int32_t max_nnz, double* row_scale_A, double* row_scale_G,
                                  double* keep_A, double* keep_b, double* keep_G, double* keep_h, int64_t host,
                                  void* stream) {
  if (ncols < 0 || nA < 0 || nG < 0 || n_nonneg < 0 || n_nonneg > nG || n_soc < 0 || max_nnz < 0)
    return fail(CITO_ERR_ARG, "precondition: bad sizes");
  if ((G_data == nullptr) != (G_rows == nullptr) || (G_data == nullptr && keep_G != nullptr))
    return fail(CITO_ERR_ARG, "precondition: concatenated layout takes G_rows = G_data = keep_G = null");
  cudaStream_t s = (cudaStream_t)stream;
  PcArgs a;
  a.ptr[0] = A_ptr;
  a.ptr[1] = G_ptr;
  a.rows[0] = A_rows;
  a.rows[1] = G_rows;
  a.data[0] = A_data;
  a.data[1] = G_data;
  a.rhs[0] = b;
  a.rhs[1] = h;
  a.nrows[0] = nA;
  a.nrows[1] = nG;
  a.rowmax[0] = rowmax_A;
  a.rowmax[1] = rowmax_G;
  a.scale[0] = row_scale_A;
  a.scale[1] = row_scale_G;
  a.keep[0] = keep_A;
  a.keep[1] = keep_G;
  a.keep_rhs[0] = keep_b;
  a.keep_rhs[1] = keep_h;
  a.concat = G_data == nullptr;
  a.host = host;
  if (!rowmax_ready) {
    if (nA) CUDA_TRY(cudaMemsetAsync(rowmax_A, 0, sizeof(unsigned long long) * (size_t)nA, s));
    if (nG) CUDA_TRY(cudaMemsetAsync(rowmax_G, 0, sizeof(unsigned long long) * (size_t)nG, s));
    if (ncols > 0) {
      const int wpb = 8;
      count_launch();
      k_row_absmax<<<dim3((unsigned)((ncols + wpb - 1) / wpb), 2), 32 * wpb, 0, s>>>(ncols, a);
      CUDA_TRY(cudaGetLastError());
    }
  }
  const int64_t nsc = (int64_t)nA + n_nonneg + n_soc;
  if (nsc > 0) {
    count_launch();
    k_row_scale<<<(unsigned)((nsc + 255) / 256), 256, 0, s>>>(a, n_nonneg, n_soc, soc_start, soc_dim);
    CUDA_TRY(cudaGetLastError());
  }
  const int64_t work = (int64_t)max_nnz + (nA > nG ? nA : nG);
  if (ncols > 0 && work > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (work + 255) / 256;
    const unsigned gx = (unsigned)(want < 4 * sms ? want : 4 * sms);
    count_launch();
    k_row_apply<<<dim3(gx, 2), 256, 0, s>>>(ncols, a);
    CUDA_TRY(cudaGetLastError());
  }
  return CITO_OK;
}

// Copy kernel, optionally mirrored into page-locked host memory (mapped under
// unified addressing): 16-byte stores straight over the bus from the SMs, so a
// small result field travels inside the graph's kernel stream -- no copy-engine
// hand-off.
__global__ void __launch_bounds__(256) k_copy_out(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16,
                                                  unsigned char* __restrict__ dtail,
                                                  const unsigned char* __restrict__ stail, int ntail, int64_t mirror) {
  // a dependent kernel (PDL) may start its independent prologue right away; it waits for
  // this grid's completion before reading what it copies
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 v = src[i];
    dst[i] = v;
    if (mirror) mirror_store(dst + i, mirror, v);
  }
  if (blockIdx.x == 0 && (int)threadIdx.x < ntail) {
    dtail[threadIdx.x] = stail[threadIdx.x];
    if (mirror) mirror_store(dtail + threadIdx.x, mirror, stail[threadIdx.x]);
  }
}

cito_status cito_copy_mirror(void* dst, const void* src, int64_t nbytes, int64_t mirror, void* stream) {
  if (nbytes < 0 || ((uintptr_t)dst & 15) || ((uintptr_t)src & 15) || (mirror & 15))
    return fail(CITO_ERR_ARG, "copy: negative size or pointers not 16-byte aligned");
  if (nbytes == 0) return CITO_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n16 = nbytes / 16;
  const int ntail = (int)(nbytes - 16 * n16);
  const int64_t want = (n16 + 255) / 256;
  const unsigned grid = (unsigned)(want < 1 ? 1 : (want < 2 * sms ? want : 2 * sms));
  count_launch();
  k_copy_out<<<grid, 256, 0, (cudaStream_t)stream>>>((uint4*)dst, (const uint4*)src, n16,
                                                     (unsigned char*)dst + 16 * n16,
                                                     (const unsigned char*)src + 16 * n16, ntail, mirror);
  CUDA_TRY(cudaGetLastError());
  return CITO_OK;
}

double cito_dfma_peak(int32_t iters, double* out_dev, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256;
  count_launch();
  k_dfma_peak<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, 1.0, out_dev);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  return 2.0 * 64.0 * (double)iters * blocks * threads;  // flops issued
}

#ifdef CITO_PROF
int cito_prof_set(long long* dev_buf) {
  return (int)cudaMemcpyToSymbol(g_cito_prof, &dev_buf, sizeof(dev_buf));
}
#endif

}  // extern "C"
