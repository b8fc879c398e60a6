/*
 * cito_b200.h — C ABI of the B200-native discretize+linearize path.
 *
 * Drop-in boundary for the reference's Python class
 *   cito.augmentation.Discretizer   (/root/reference/pkg/src/cito/augmentation.py:172-255)
 * and the value scatter of the multiple-shooting rows of
 *   cito.scp.build_subproblem      (/root/reference/pkg/src/cito/scp.py:226-236)
 *   cito.conic.canonicalize        (/root/reference/pkg/src/cito/conic.py:209-269).
 * The reference has no FFI of its own (pure Python + JAX); these entry points
 * are what a ctypes binding of that class binds (INTEGRATION.md shows it).
 *
 * Conventions: plain pointers + sizes, row-major float64 arrays, int32 CSC
 * indices, no torch types.  `*_host` entry points take HOST buffers and do
 * the host<->device copies inside the call; `*_dev` entry points take DEVICE
 * buffers and a cudaStream_t passed as void*.  Every call returns a
 * cito_status; cito_last_error() gives a message for the calling thread.
 * All entry points are reentrant (per-handle mutex around the staging
 * buffers), so the reference's ThreadPoolExecutor fan-out
 * (/root/reference/pkg/src/cito/scp.py:101-112) can call them concurrently.
 */
#ifndef CITO_B200_H
#define CITO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CITO_MAX_LINKS 16
#define CITO_MAX_JOINTS 16
#define CITO_MAX_CONTACTS 8
#define CITO_MAX_PATH 48 /* n_g = n_c + 2*joint_limits + 2*height_bounds */
#define CITO_MAX_GOUT 48 /* rows of the mixing matrix */
#define CITO_MAX_EXPR 256

/* surface kinds (cito/multibody.py:107-172) */
#define CITO_SURFACE_FLAT 0
#define CITO_SURFACE_IMPLICIT 1

/* postfix byte-code of an implicit surface h(px, pz) (cito/multibody.py:144-172);
 * the grammar of the reference: constants, +, *, **, sin, cos.  a**b with a
 * non-constant exponent b is emitted as  b a LOG MUL EXP  (= exp(b log a)). */
#define CITO_OP_CONST 0 /* push arg */
#define CITO_OP_PX 1
#define CITO_OP_PZ 2
#define CITO_OP_ADD 3
#define CITO_OP_MUL 4
#define CITO_OP_POW 5 /* a**arg (constant exponent) */
#define CITO_OP_SIN 6
#define CITO_OP_COS 7
#define CITO_OP_NEG 8
#define CITO_OP_LOG 9 /* natural log (variable-exponent powers) */
#define CITO_OP_EXP 10

typedef enum {
  CITO_OK = 0,
  CITO_ERR_ARG = 1,         /* bad argument / unsupported model (ValueError) */
  CITO_ERR_NONFINITE = 2,   /* non-finite end state (FloatingPointError)       */
  CITO_ERR_CUDA = 3,        /* CUDA runtime failure                            */
  CITO_ERR_UNSUPPORTED = 4  /* model topology outside the compiled set         */
} cito_status;

/*
 * Packed RobotModel + path-constraint spec + mixing matrix.
 *   links     cito/multibody.py:53-66     (mass, inertia, com_offset)
 *   joints    cito/multibody.py:68-89     (parent -1 = world)
 *   contacts  cito/multibody.py:92-104
 *   path g    cito/augmentation.py:100-131 (rows: -sd per contact, then
 *             (rel-hi, lo-rel) per joint limit, then (lo-pz, pz-hi) per height bound)
 *   mixing    n_g_out x n_g, row-major in mixing[] (cito/ocp.py:121-126); n_g_out = 0
 *             means the Discretizer was built with mixing=None (no path channels).
 */
typedef struct cito_model_desc {
  int32_t n_links, n_joints, n_contacts, surface_kind;
  double gravity;
  double surface_height;
  double link_mass[CITO_MAX_LINKS];
  double link_inertia[CITO_MAX_LINKS];
  double link_com[CITO_MAX_LINKS][2];
  int32_t joint_parent[CITO_MAX_JOINTS];
  int32_t joint_child[CITO_MAX_JOINTS];
  int32_t joint_actuated[CITO_MAX_JOINTS];
  int32_t joint_spring[CITO_MAX_JOINTS]; /* stiffness != 0 or damping != 0 */
  double joint_parent_anchor[CITO_MAX_JOINTS][2];
  double joint_child_anchor[CITO_MAX_JOINTS][2];
  double joint_stiffness[CITO_MAX_JOINTS];
  double joint_damping[CITO_MAX_JOINTS];
  double joint_rest[CITO_MAX_JOINTS];
  int32_t contact_link[CITO_MAX_CONTACTS];
  double contact_offset[CITO_MAX_CONTACTS][2];
  double contact_mu[CITO_MAX_CONTACTS];
  double contact_restitution[CITO_MAX_CONTACTS];
  int32_t n_joint_limits;
  int32_t jl_joint[CITO_MAX_PATH];
  double jl_lo[CITO_MAX_PATH], jl_hi[CITO_MAX_PATH];
  int32_t n_height_bounds;
  int32_t hb_link[CITO_MAX_PATH];
  double hb_lo[CITO_MAX_PATH], hb_hi[CITO_MAX_PATH];
  int32_t n_g_out;
  int32_t expr_len;
  double mixing[CITO_MAX_GOUT * CITO_MAX_PATH];
  int32_t expr_op[CITO_MAX_EXPR];
  double expr_arg[CITO_MAX_EXPR];
} cito_model_desc;

typedef struct cito_handle cito_handle;

/* sizes derived exactly as cito/augmentation.py:267-269, cito/contact_dynamics.py:35-37 */
typedef struct cito_dims {
  int32_t n_q, n_x, n_u, n_y, n_xt, n_j, n_a, n_g, D;
} cito_dims;

const char* cito_last_error(void);
const char* cito_version(void);

/* Discretizer.__init__ (cito/augmentation.py:180-216). substeps < 1 -> CITO_ERR_ARG. */
cito_status cito_create(const cito_model_desc* desc, int32_t substeps, cito_handle** out);
cito_status cito_destroy(cito_handle* h);
cito_status cito_get_dims(const cito_handle* h, cito_dims* out);

/* Discretizer.propagate_batch (cito/augmentation.py:226-234):
 *   xt0s (B, n_xt), Us (B, 2*n_u) = [U-, U+], Ss (B) -> ends (B, n_xt).
 * bad (B, optional) receives 1 for intervals whose end state is non-finite;
 * the call then returns CITO_ERR_NONFINITE (the Python layer raises
 * FloatingPointError listing them). */
cito_status cito_propagate_host(cito_handle* h, int64_t B, const double* xt0s, const double* Us,
                                const double* Ss, double* ends, int32_t* bad);
cito_status cito_propagate_dev(cito_handle* h, int64_t B, const double* xt0s, const double* Us,
                               const double* Ss, double* ends, int32_t* bad, void* stream);

/* Discretizer.linearize_batch (cito/augmentation.py:236-242):
 *   -> ends (B, n_xt), jx (B, n_xt, n_xt), ju (B, n_xt, 2*n_u), js (B, n_xt).
 * Exact forward-mode derivatives of the discrete RKF recursion. */
cito_status cito_linearize_host(cito_handle* h, int64_t B, const double* xt0s, const double* Us,
                                const double* Ss, double* ends, double* jx, double* ju, double* js,
                                int32_t* bad);
cito_status cito_linearize_dev(cito_handle* h, int64_t B, const double* xt0s, const double* Us,
                               const double* Ss, double* ends, double* jx, double* ju, double* js,
                               int32_t* bad, void* stream);

/* Node relations of cito.ocp.Transcription (cito/ocp.py:277-303, 336-365):
 *   psi  (Np, n_psi) and psi_jac (Np, n_psi, 2 n_y) from y_pairs (Np, 2 n_y)
 *   theta (Nn, 6 n_c) and theta_jac (Nn, 6 n_c, 3 n_q + 3 n_c) from theta_vecs
 *   imp  (Nn, n_q)  and imp_jac (Nn, n_q, 3 n_q + 2 n_c) from the first
 *        3 n_q + 2 n_c entries of theta_vecs.  Device buffers. */
cito_status cito_node_linearize_dev(cito_handle* h, int64_t Np, int64_t Nn, const double* y_pairs,
                                    const double* theta_vecs, double delta, double epsilon,
                                    double* psi, double* psi_jac, double* theta, double* theta_jac,
                                    double* imp, double* imp_jac, void* stream);

/* Pointwise audit of sampled states for verifier.replay_check
 * (cito/verifier.py:257-272, 314-318): for each of B samples, x = the first n_x
 * entries of row b of xs (row stride xstride >= n_x), u = us (B, n_u):
 *   sds   (B, n_c)        contact signed distances (multibody.py:384-392)
 *   cj    (B, 2 n_joints) joint anchor residuals   (multibody.py:324-336)
 *   omega (B, n_y)        auxiliary rates Omega(x, u) (augmentation.py:134-153).
 * Device buffers. */
cito_status cito_audit_dev(cito_handle* h, int64_t B, const double* xs, int64_t xstride, const double* us,
                           double* sds, double* cj, double* omega, void* stream);

/* linearize_all (cito/scp.py:87-135) on a device-resident decision vector z
 * (layout cito/ocp.py:154-174: node states [xm_k, xp_k] at 2k n_xt / (2k+1) n_xt,
 * interval blocks [U_k, S_k] at base_u + k (2 n_u + 1), node impulses
 * [Phi_k, Gamma_k] at base_p + 3 n_c k; base_u = 2 N n_xt,
 * base_p = base_u + (N-1)(2 n_u + 1)).  Interval kernel and node-relation
 * kernel read z directly (no host/device gathers), run concurrently (the node
 * kernel on an internal stream joined back into `stream`), and the defects
 * z[xm(k+1)] - ends[k] are written by the interval kernel.  n_problems > 1
 * linearizes a multi-start batch of independent decision vectors stored
 * zstride doubles apart in one launch (outputs stacked problem-major). */
cito_status cito_linearize_all_dev(cito_handle* h, int32_t N, int32_t n_problems, int64_t zstride, int64_t base_u,
                                   int64_t base_p, const double* z, double delta, double epsilon, double* ends, double* jx, double* ju, double* js,
                                   double* defects, int32_t* bad, double* psi, double* psi_jac, double* theta,
                                   double* theta_jac, double* imp, double* imp_jac, void* stream);

/* Same as cito_linearize_all_dev with the relaxation parameters read from
 * device memory (d_delta_eps = {delta, epsilon}), so one captured CUDA graph of
 * an SCP iteration replays for every delta of the homotopy (scp.py:354-380). */
cito_status cito_linearize_all_dev2(cito_handle* h, int32_t N, int32_t n_problems, int64_t zstride, int64_t base_u,
                                    int64_t base_p, const double* z, const double* d_delta_eps, double* ends,
                                    double* jx, double* ju, double* js, double* defects, int32_t* bad, double* psi,
                                    double* psi_jac, double* theta, double* theta_jac, double* imp, double* imp_jac,
                                    void* stream);

/* Multiple-shooting rows of the SCP subproblem, written straight into CSC value
 * slots (cito/scp.py:226-236 + cito/conic.py:209-269).  The slot map is built
 * once per sparsity pattern by the host (paper_2604_09993_b200/scatter.py):
 *   slot_x (n_int, n_xt, n_xt), slot_u (n_int, n_xt, 2 n_u), slot_s (n_int, n_xt)
 *   give the position in A_data of -jx[k,r,j]*sigma etc., or -1 where the
 *   reference pattern has no entry (the value must then be exactly zero).
 * b_rows (n_int*n_xt) receives b = ends - (jx.z_xp + ju.z_u + js.z_s).
 * mismatch (device int32, 1 element) counts entries whose value is nonzero
 * but has no slot (or zero with a slot) -> caller must rebuild the pattern. */
cito_status cito_scatter_dynamics_dev(cito_handle* h, int64_t n_int, const double* ends,
                                      const double* jx, const double* ju, const double* js,
                                      const double* z_ref, const int64_t* xp_off,
                                      const int64_t* u_off, const int64_t* s_off,
                                      const double* sig_x, const double* sig_u, double sig_s,
                                      const int32_t* slot_x, const int32_t* slot_u,
                                      const int32_t* slot_s, double* A_data, double* b_rows,
                                      int32_t* mismatch, void* stream);

/* Whole-subproblem CSC assembly (cito/scp.py:160-351 +
 * cito/conic.py:99-125, 209-269).  A superset CSC (sp_ptr[ncols+1], sp_row)
 * carries one value recipe per entry: sp_src < 0 -> constant sp_val, else
 * (sp_val * lin[sp_src][sp_idx]) * sigma[col].  Exact zeros are dropped and the
 * rest compacted: out_ptr[ncols+1] (int32), out_rows/out_vals[<= superset nnz].
 * lin: HOST array of 10 device pointers {jx, ju, js, imp_jac, theta_jac,
 * psi_jac, ends, imp_v, theta, psi}; counts: device int32 workspace
 * [ncols + 64] per matrix.  The one-pass compaction keeps a fixed header
 * [ticket, finished CTAs, pad, pad] at the start of counts[0] followed by one
 * uint64 flag per column block; it returns them to zero at the end of every
 * launch, so the rules are: ZERO the workspace before its first use, keep it
 * between calls (any ncols up to the size it was allocated for), and zero it
 * again after a call that returned CITO_ERR_CUDA (a launch that did not
 * complete leaves its tickets behind).  One workspace per stream: two
 * concurrent launches must not share it. */
cito_status cito_csc_assemble_dev(int32_t ncols, const int64_t* sp_ptr, const int32_t* sp_row, const int8_t* sp_src,
                                  const int64_t* sp_idx, const double* sp_val, const double* sigma,
                                  const double* const* lin, int32_t* counts, int32_t* out_ptr, int32_t* out_rows,
                                  double* out_vals, void* stream);

/* Same as cito_csc_assemble_dev for nmat (1 or 2, e.g. A and G) matrices with
 * the same column count in one set of launches; every pointer argument except
 * sigma and lin is a HOST array of nmat device pointers.  rowmax (optional,
 * NULL = off): per matrix a ZEROED device uint64[nrows] that receives the row
 * inf-norms (bit patterns of max |value|) for cito_precondition_dev. */
cito_status cito_csc_assemble2_dev(int32_t nmat, int32_t ncols, const int64_t* const* sp_ptr,
                                   const int32_t* const* sp_row, const int8_t* const* sp_src,
                                   const int64_t* const* sp_idx, const double* const* sp_val, const double* sigma,
                                   const double* const* lin, int32_t* const* counts, int32_t* const* out_ptr,
                                   int32_t* const* out_rows, double* const* out_vals,
                                   unsigned long long* const* rowmax, void* stream);

/* Packed form of cito_csc_assemble2_dev (the default of the Python layer): one
 * 16-byte record per superset entry, {double w; uint32 key; int32 row}, sorted by
 * (column, row): key = (src + 1) << 27 | idx (idx < 2^27); src < 0 -> constant
 * value w, else value = lin[src][idx] * w with w = sign * sigma[col] (sign = +-1,
 * which makes it bit-identical to (sign * lin) * sigma).  Entries are processed in
 * flat tiles of 2048 (one CTA each): ntile[m] >= max(1, ceil(nsup[m] / 2048))
 * tiles, tcol[m] (device int32[ntile + 1]) = first column whose first superset
 * entry lies in tile t (searchsorted(sp_ptr, 2048 t)), ncols + 1 at the end.
 * ws: device uint32 workspace of ws_words >= 4 + 2 * (sum of ntile) words,
 * zero before the first call; the kernel leaves it zero (zero it again after a
 * call that returned CITO_ERR_CUDA).  Pointer arguments except ws, lin (host
 * array of 10 device pointers) and the host arrays nsup/ntile are host arrays of
 * nmat device pointers.  stamp_in / changed_at (device doubles, both null or both
 * set): when any row index or column pointer written differs from what out_rows /
 * out_ptr held before the call, *changed_at = *stamp_in -- the caller learns that
 * the sparsity pattern moved since the previous call over the same outputs.
 * nmat = 2 with out_rows[1] = out_vals[1] = NULL: concatenated output -- the second
 * matrix's entries follow the first's nonzeros in out_rows[0] / out_vals[0], its
 * column pointers (out_ptr[1]) relative to its own first entry.
 * host_vals / host_pattern (0 = off): byte offsets from the device outputs to a
 * page-locked host mirror laid out the same way; the kernel also stores every
 * value (host_vals), the stamp and, while *rows_wanted (device double) != 0,
 * every column pointer and row index (host_pattern) there, so the result
 * crosses the bus during the compaction.  consts_wanted (device double, NULL =
 * always): while it is 0 the mirror already holds this pattern's constant
 * entries and 16-byte chunks of constants only are not stored again. */
cito_status cito_csc_assemble_packed_dev(int32_t nmat, int32_t ncols, const void* const* ent, const int64_t* nsup,
                                        const int64_t* const* sp_ptr, const int32_t* const* tcol, const int32_t* ntile,
                                        const double* const* lin, uint32_t* ws, int64_t ws_words,
                                        int32_t* const* out_ptr, int32_t* const* out_rows, double* const* out_vals,
                                        unsigned long long* const* rowmax, const double* stamp_in,
                                        double* changed_at, int64_t host_vals, int64_t host_pattern,
                                        const double* rows_wanted, const double* consts_wanted, void* stream);

/* b / h of the linearized rows: out[rows[i]] = form ? J.z[cols] - v : v - J.z[cols]
 * with J split in up to 3 segments (seg_src < 0 = unused), v = lin[vsrc[i]][voff[i]];
 * host != 0: each row also stored at out + host bytes (a page-locked host mirror). */
cito_status cito_rhs_dev(int64_t nrows, const int32_t* rows, const int8_t* form, const int8_t* vsrc,
                         const int64_t* voff, const int8_t* seg_src, const int64_t* seg_off, const int32_t* seg_len,
                         const int64_t* seg_cb, const int64_t* cols, const double* z, const double* const* lin,
                         double* out, int64_t host, void* stream);

/* cito.conic.precondition (cito/conic.py:290-338) of a device-resident program
 * (CSC A: nA rows, G: nG rows, int32 indptr/indices, ncols columns), in place:
 *   row_scale_A[i] = 1 / inf-norm of row i (1 for an all-zero row);
 *   row_scale_G    = the same for the n_nonneg orthant rows; each SOC block
 *                    k (rows soc_start[k] .. + soc_dim[k], device int32 arrays)
 *                    shares 1 / max over its rows (1 if that max is 0);
 *   A.data, b, G.data, h multiplied by their row's scale (values bit-identical
 *   to scipy's Da @ A).
 * rowmax_A/G: device uint64 workspaces [nA]/[nG]; rowmax_ready != 0 means they
 * already hold the norms (fused into the compaction), else this call computes
 * them; the call leaves them zero (ready for the next fused compaction).
 * max_nnz: upper bound of the stored entries of A and G.
 * keep_A/keep_b/keep_G/keep_h (optional, NULL = off): device arrays that receive
 * the values before scaling.  G_rows = G_data = keep_G = NULL selects the
 * concatenated layout of cito_csc_assemble_packed_dev: G's entries follow A's
 * A_ptr[ncols] nonzeros in A_rows / A_data / keep_A, G_ptr relative to them.
 * host (0 = off): byte offset from every output (data, b/h, row scales) to a
 * page-locked host mirror that also receives it.
 * The cost scaling (c / omega, P / omega) is a host-side scalar (Python layer). */
cito_status cito_precondition_dev(int32_t ncols, const int32_t* A_ptr, const int32_t* A_rows, double* A_data,
                                  int32_t nA, double* b, const int32_t* G_ptr, const int32_t* G_rows, double* G_data,
                                  int32_t nG, double* h, int32_t n_nonneg, int32_t n_soc, const int32_t* soc_start,
                                  const int32_t* soc_dim, unsigned long long* rowmax_A, unsigned long long* rowmax_G,
                                  int32_t rowmax_ready, int32_t max_nnz, double* row_scale_A, double* row_scale_G,
                                  double* keep_A, double* keep_b, double* keep_G, double* keep_h, int64_t host,
                                  void* stream);

/* Copy nbytes src -> dst with a kernel (device or page-locked host memory; SM stores,
 * no copy-engine transfer); mirror != 0: also to dst + mirror bytes (a page-locked
 * host mirror of dst).  dst, src and mirror 16-byte aligned.  Used inside an SCP
 * iteration's graph for the small result fields (flags, constant rhs rows). */
cito_status cito_copy_mirror(void* dst, const void* src, int64_t nbytes, int64_t mirror, void* stream);

/* FP64 DFMA throughput probe (roofline denominator; not part of the reference
 * interface).  Launches one kernel on `stream`; returns the flops it issues
 * (time it with events on the same stream), or -1 on launch failure. */
double cito_dfma_peak(int32_t iters, double* out_dev, void* stream);

/* Number of kernel launches issued by this handle since creation, or by the
 * whole library when h is NULL (evidence for bench.py's gpu_launches). */
int64_t cito_launch_count(const cito_handle* h);

#ifdef __cplusplus
}
#endif

#endif /* CITO_B200_H */
