// cito_scatter.cuh — multiple-shooting rows of the SCP subproblem straight into
// CSC value slots (K4).
//
// Replaces the dynamics-row loop of cito.scp.build_subproblem
// (/root/reference/pkg/src/cito/scp.py:226-236, eq() at :186-201) followed by
// cito.conic.canonicalize/_to_csc (/root/reference/pkg/src/cito/conic.py:120-125,
// 209-269).  Row (k, r) of A (k-th interval, r-th state row) holds
//   -jx[k,r,j]*sigma_x[j] at column xp(k)+j, -ju[k,r,j]*sigma_u[j mod n_u] at u(k)+j,
//   -js[k,r]*sigma_S at s(k)         (plus the constant +sigma / slack entries)
// and b = ends[k,r] - (jx[k,r].z[xp(k)] + ju[k,r].z[u(k)] + js[k,r]*z[s(k)]).
// One warp per row; the value is multiplied exactly as the reference does
// (vals = -jrow; svals = vals * sigma), so values differ from the reference
// only through the Jacobians themselves.  Exact zeros are never stored
// (conic.py:116-125): an entry whose value is zero must have no slot, a nonzero
// value must have one; violations are counted in *mismatch so the host can
// rebuild the pattern.
#pragma once

#include <cstdint>

__global__ void __launch_bounds__(128) k_scatter_dynamics(
    int64_t n_int, int n_xt, int n_u, const double* __restrict__ ends, const double* __restrict__ jx,
    const double* __restrict__ ju, const double* __restrict__ js, const double* __restrict__ z_ref,
    const int64_t* __restrict__ xp_off, const int64_t* __restrict__ u_off, const int64_t* __restrict__ s_off,
    const double* __restrict__ sig_x, const double* __restrict__ sig_u, double sig_s,
    const int32_t* __restrict__ slot_x, const int32_t* __restrict__ slot_u, const int32_t* __restrict__ slot_s,
    double* __restrict__ A_data, double* __restrict__ b_rows, int32_t* __restrict__ mismatch) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_int * n_xt) return;
  const int64_t k = row / n_xt;
  const int nu2 = 2 * n_u;
  const double* jxr = jx + row * n_xt;
  const double* jur = ju + row * nu2;
  const double* zx = z_ref + xp_off[k];
  const double* zu = z_ref + u_off[k];
  const int32_t* sx = slot_x + row * n_xt;
  const int32_t* su = slot_u + row * nu2;
  double dot = 0.0;
  int bad = 0;
  for (int j = lane; j < n_xt; j += 32) {
    const double v = jxr[j];
    dot += v * zx[j];
    const double sv = (-v) * sig_x[j];
    const int32_t sl = sx[j];
    if (sl >= 0) {
      A_data[sl] = sv;
      bad += (sv == 0.0);
    } else {
      bad += (sv != 0.0);
    }
  }
  for (int j = lane; j < nu2; j += 32) {
    const double v = jur[j];
    dot += v * zu[j];
    const double sv = (-v) * sig_u[j % n_u];
    const int32_t sl = su[j];
    if (sl >= 0) {
      A_data[sl] = sv;
      bad += (sv == 0.0);
    } else {
      bad += (sv != 0.0);
    }
  }
  if (lane == 0) {
    const double v = js[row];
    dot += v * z_ref[s_off[k]];
    const double sv = (-v) * sig_s;
    const int32_t sl = slot_s[row];
    if (sl >= 0) {
      A_data[sl] = sv;
      bad += (sv == 0.0);
    } else {
      bad += (sv != 0.0);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dot += __shfl_xor_sync(0xffffffffu, dot, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane == 0) {
    b_rows[row] = ends[row] - dot;
    if (bad && mismatch) atomicAdd(mismatch, bad);
  }
}
