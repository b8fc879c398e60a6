// cito_subproblem.cuh — device assembly of the SCP subproblem's CSC matrices
// (SURVEY.md §8(f) row 1): replaces cito.scp.build_subproblem's row loops and
// cito.conic.canonicalize/_to_csc (/root/reference/pkg/src/cito/scp.py:160-351,
// conic.py:99-125, 209-269).
//
// The host lays out a superset CSC (every entry that can be nonzero, rows
// sorted inside each column) with a recipe per entry: a constant, or
// (sign * LIN[src][idx]) * sigma[col] for the linearized rows.  Per iteration:
//   k_csc_count   warp per column: evaluate, count exact nonzeros
//   k_scan        single CTA: exclusive scan of the counts -> indptr (int32)
//   k_csc_write   warp per column: evaluate again, ballot-compact the nonzeros
// which is the reference's `keep = vals != 0` + eliminate_zeros + sort_indices.
// k_rhs forms b / h of the linearized rows (warp per row, up to 3 segments).
#pragma once

#include <cstdint>

struct LinTable {
  const double* p[10];  // jx, ju, js, imp_jac, theta_jac, psi_jac, ends, imp_v, theta, psi
};

// L.p[s] without indexing the parameter array dynamically (which would copy the
// table to local memory): selects between the 10 kernel-parameter pointers
__device__ __forceinline__ const double* lin_ptr(const LinTable& L, int s) {
  const double* p = L.p[0];
#pragma unroll
  for (int k = 1; k < 10; ++k)
    if (s == k) p = L.p[k];
  return p;
}

__device__ __forceinline__ double sp_value(int64_t e, double sig, const int8_t* __restrict__ src,
                                           const int64_t* __restrict__ idx, const double* __restrict__ val,
                                           const LinTable& L) {
  const int s = src[e];
  return s < 0 ? val[e] : (val[e] * L.p[s][idx[e]]) * sig;
}

// up to two matrices (A, G) per launch: blockIdx.y selects the matrix
struct CscArgs {
  const int64_t* sp_ptr[2];
  const int32_t* row[2];
  const int8_t* src[2];
  const int64_t* idx[2];
  const double* val[2];
  int32_t* counts[2];
  int32_t* out_ptr[2];
  int32_t* out_rows[2];
  double* out_vals[2];
  unsigned long long* rowmax[2];  // optional (nullptr): row inf-norms for the preconditioner, as |v| bits
};

__global__ void __launch_bounds__(256) k_csc_count(int32_t ncols, const CscArgs a, const double* __restrict__ sigma,
                                                   const LinTable L) {
  const int m = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const int64_t* __restrict__ sp_ptr = a.sp_ptr[m];
  const double sig = sigma[c];
  int n = 0;
  for (int64_t e = sp_ptr[c] + lane; e < sp_ptr[c + 1]; e += 32)
    n += sp_value(e, sig, a.src[m], a.idx[m], a.val[m], L) != 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if (lane == 0) a.counts[m][c] = n;
}

// Exclusive scan of the per-column counts -> indptr (int32), one CTA per matrix
// (blockIdx.x selects the matrix).  Each thread scans a contiguous run in
// registers, warps combine with shuffles, one pass over the data.
struct ScanArgs {
  int32_t n[2];
  const int32_t* counts[2];
  int32_t* out_ptr[2];
};

__global__ void __launch_bounds__(1024) k_scan(const ScanArgs a) {
  const int m = blockIdx.x;
  const int32_t n = a.n[m];
  const int32_t* __restrict__ counts = a.counts[m];
  int32_t* __restrict__ out_ptr = a.out_ptr[m];
  __shared__ int32_t warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int32_t per = (n + 1023) / 1024;
  const int32_t lo = min(n, tid * per), hi = min(n, lo + per);
  int32_t local = 0;
  for (int32_t i = lo; i < hi; ++i) local += counts[i];
  int32_t incl = local;  // inclusive warp scan of the per-thread totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int32_t w = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    warp_tot[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int32_t run = (wid > 0 ? warp_tot[wid - 1] : 0) + incl - local;  // exclusive prefix of this thread's run
  for (int32_t i = lo; i < hi; ++i) {
    out_ptr[i] = run;
    run += counts[i];
  }
  if (tid == 1023) out_ptr[n] = warp_tot[31];
}

__global__ void __launch_bounds__(256) k_csc_write(int32_t ncols, const CscArgs a, const double* __restrict__ sigma,
                                                   const LinTable L) {
  const int m = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const int64_t* __restrict__ sp_ptr = a.sp_ptr[m];
  const double sig = sigma[c];
  int32_t base = a.out_ptr[m][c];
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t e0 = sp_ptr[c]; e0 < sp_ptr[c + 1]; e0 += 32) {
    const int64_t e = e0 + lane;
    const bool in = e < sp_ptr[c + 1];
    const double v = in ? sp_value(e, sig, a.src[m], a.idx[m], a.val[m], L) : 0.0;
    const bool nz = in && v != 0.0;
    const unsigned msk = __ballot_sync(0xffffffffu, nz);
    if (nz) {
      const int32_t pos = base + __popc(msk & lt);
      const int32_t r = a.row[m][e];
      a.out_rows[m][pos] = r;
      a.out_vals[m][pos] = v;
      // fused row inf-norm (cito/conic.py:281-287): non-negative doubles order like their bits
      if (a.rowmax[m]) atomicMax(&a.rowmax[m][r], (unsigned long long)__double_as_longlong(fabs(v)));
    }
    base += __popc(msk);
  }
}


// ---------------------------------------------------------------------------
// Two-launch compaction (replaces count + scan + write): columns are processed
// in blocks of CSC_CPB columns (one CTA, 8 warps).
//   k_csc_blocksum  number of exact nonzeros of every column block -> bsum[block]
//   k_csc_write2    prefix = sum of bsum over the preceding blocks (CTA reduce),
//                   per-column counts + warp scan -> indptr of the block's
//                   columns, then the ballot-compacted write (+ row inf-norms)
#define CSC_CPB 32

__global__ void __launch_bounds__(256) k_csc_blocksum(int32_t ncols, const CscArgs a, const double* __restrict__ sigma,
                                                      const LinTable L) {
  const int m = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t* __restrict__ sp_ptr = a.sp_ptr[m];
  __shared__ int32_t wsum[8];
  int n = 0;
  for (int k = warp; k < CSC_CPB; k += 8) {
    const int64_t c = (int64_t)blockIdx.x * CSC_CPB + k;
    if (c >= ncols) break;
    const double sig = sigma[c];
    for (int64_t e = sp_ptr[c] + lane; e < sp_ptr[c + 1]; e += 32)
      n += sp_value(e, sig, a.src[m], a.idx[m], a.val[m], L) != 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if (lane == 0) wsum[warp] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += wsum[w];
    a.counts[m][blockIdx.x] = t;  // the counts workspace holds the block totals
  }
}

__global__ void __launch_bounds__(256) k_csc_write2(int32_t ncols, const CscArgs a, const double* __restrict__ sigma,
                                                    const LinTable L) {
  const int m = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t* __restrict__ sp_ptr = a.sp_ptr[m];
  const int64_t c0 = (int64_t)blockIdx.x * CSC_CPB;
  __shared__ int32_t red[8];
  __shared__ int32_t ccount[CSC_CPB];
  __shared__ int32_t cbase[CSC_CPB];
  // prefix over the preceding column blocks
  int pre = 0;
  for (int j = tid; j < (int)blockIdx.x; j += blockDim.x) pre += a.counts[m][j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 0) red[warp] = pre;
  // per-column nonzero counts of this block
  for (int k = warp; k < CSC_CPB; k += 8) {
    const int64_t c = c0 + k;
    int n = 0;
    if (c < ncols) {
      const double sig = sigma[c];
      for (int64_t e = sp_ptr[c] + lane; e < sp_ptr[c + 1]; e += 32)
        n += sp_value(e, sig, a.src[m], a.idx[m], a.val[m], L) != 0.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) ccount[k] = n;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the block's column counts (CSC_CPB == 32: one per lane)
    int blockpre = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) blockpre += red[w];
    const int v = ccount[lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int base = blockpre + incl - v;
    cbase[lane] = base;
    const int64_t c = c0 + lane;
    if (c < ncols) a.out_ptr[m][c] = base;
    if (c == ncols - 1) a.out_ptr[m][ncols] = base + v;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int k = warp; k < CSC_CPB; k += 8) {
    const int64_t c = c0 + k;
    if (c >= ncols) break;
    const double sig = sigma[c];
    int32_t base = cbase[k];
    for (int64_t e0 = sp_ptr[c]; e0 < sp_ptr[c + 1]; e0 += 32) {
      const int64_t e = e0 + lane;
      const bool in = e < sp_ptr[c + 1];
      const double v = in ? sp_value(e, sig, a.src[m], a.idx[m], a.val[m], L) : 0.0;
      const bool nz = in && v != 0.0;
      const unsigned msk = __ballot_sync(0xffffffffu, nz);
      if (nz) {
        const int32_t pos = base + __popc(msk & lt);
        const int32_t r = a.row[m][e];
        a.out_rows[m][pos] = r;
        a.out_vals[m][pos] = v;
        if (a.rowmax[m]) atomicMax(&a.rowmax[m][r], (unsigned long long)__double_as_longlong(fabs(v)));
      }
      base += __popc(msk);
    }
  }
}

// One-pass CSC compaction (default): each column block counts its exact nonzeros,
// publishes its total, then sums the totals of the preceding blocks (decoupled
// look-back), scans its columns and writes.  Deadlock freedom does not rely on
// the hardware dispatching CTAs in blockIdx order: every CTA takes its tile from
// an atomic ticket, so a tile only ever waits on tiles whose CTAs started before
// it (already resident or finished), whatever else shares the SMs (the rhs kernel
// on the side stream, a CUDA graph's neighbours).  Tiles are numbered over both
// matrices (A's blocks first), gridDim = (column blocks, nmat).
// Workspace (the caller's counts[0], int32[ncols + 64]): a fixed header
//   [0] ticket  [1] finished CTAs  [2..3] padding
// then one uint64 flag per tile: (1 << 32) | block total once published.  The
// last CTA of a launch returns header and flags to zero, so every launch --
// e.g. every replay of a captured CUDA graph -- starts from a clean workspace;
// the workspace must be zero before the first launch (and again after a launch
// that did not complete, see include/cito_b200.h).
#define CSC_HDR_WORDS 4

__global__ void __launch_bounds__(256) k_csc_onepass(int32_t ncols, const CscArgs a, const double* __restrict__ sigma,
                                                     const LinTable L) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = gridDim.x, ntiles = gridDim.x * gridDim.y;
  unsigned* hdr = reinterpret_cast<unsigned*>(a.counts[0]);
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(a.counts[0] + CSC_HDR_WORDS);
  __shared__ int32_t red[8];
  __shared__ int32_t ccount[CSC_CPB];
  __shared__ int32_t cbase[CSC_CPB];
  __shared__ int tile_s, last_s;
  if (tid == 0) tile_s = (int)atomicAdd(&hdr[0], 1u);
  __syncthreads();
  const int tile = tile_s;
  const int m = tile / nb, bx = tile - m * nb;
  const int64_t* __restrict__ sp_ptr = a.sp_ptr[m];
  const int64_t c0 = (int64_t)bx * CSC_CPB;
  // per-column nonzero counts of this block
  for (int k = warp; k < CSC_CPB; k += 8) {
    const int64_t c = c0 + k;
    int n = 0;
    if (c < ncols) {
      const double sig = sigma[c];
      for (int64_t e = sp_ptr[c] + lane; e < sp_ptr[c + 1]; e += 32)
        n += sp_value(e, sig, a.src[m], a.idx[m], a.val[m], L) != 0.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) ccount[k] = n;
  }
  __syncthreads();
  if (warp == 0) {  // publish this block's total
    int t = ccount[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) atomicExch(&flags[tile], (1ull << 32) | (unsigned)t);
  }
  // prefix over the preceding column blocks of the same matrix (tiles m*nb .. tile-1,
  // all taken by CTAs that started before this one)
  int pre = 0;
  for (int j = m * nb + tid; j < tile; j += blockDim.x) {
    unsigned long long f;
    do {
      f = *((volatile unsigned long long*)&flags[j]);
    } while ((f >> 32) == 0ull);
    pre += (int)(unsigned)(f & 0xffffffffull);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 0) red[warp] = pre;
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the block's column counts (CSC_CPB == 32: one per lane)
    int blockpre = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) blockpre += red[w];
    const int v = ccount[lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int base = blockpre + incl - v;
    cbase[lane] = base;
    const int64_t c = c0 + lane;
    if (c < ncols) a.out_ptr[m][c] = base;
    if (c == ncols - 1) a.out_ptr[m][ncols] = base + v;
  }
  // every read of the flags by this CTA is done: count it as finished
  if (tid == 0) {
    __threadfence();
    last_s = atomicAdd(&hdr[1], 1u) == (unsigned)ntiles - 1u;
  }
  __syncthreads();
  if (last_s) {  // all other CTAs are past their look-back: clean the workspace for the next launch
    for (int j = tid; j < ntiles; j += blockDim.x) flags[j] = 0ull;
    if (tid == 0) {
      hdr[0] = 0u;
      hdr[1] = 0u;
    }
    __threadfence();
  }
  const unsigned lt = (1u << lane) - 1u;
  for (int k = warp; k < CSC_CPB; k += 8) {
    const int64_t c = c0 + k;
    if (c >= ncols) break;
    const double sig = sigma[c];
    int32_t base = cbase[k];
    for (int64_t e0 = sp_ptr[c]; e0 < sp_ptr[c + 1]; e0 += 32) {
      const int64_t e = e0 + lane;
      const bool in = e < sp_ptr[c + 1];
      const double v = in ? sp_value(e, sig, a.src[m], a.idx[m], a.val[m], L) : 0.0;
      const bool nz = in && v != 0.0;
      const unsigned msk = __ballot_sync(0xffffffffu, nz);
      if (nz) {
        const int32_t pos = base + __popc(msk & lt);
        const int32_t r = a.row[m][e];
        a.out_rows[m][pos] = r;
        a.out_vals[m][pos] = v;
        if (a.rowmax[m]) atomicMax(&a.rowmax[m][r], (unsigned long long)__double_as_longlong(fabs(v)));
      }
      base += __popc(msk);
    }
  }
}

// ---------------------------------------------------------------------------
// Entry-parallel compaction (default since round 2): the superset entries of A and
// G are processed as flat tiles of CSC_TILE = 256 x CSC_TJ entries, one CTA per tile,
// instead of a warp per column (A has ~20 superset entries per column, G ~3, so a
// warp per column idles most lanes and serialises dependent loads).
//   record  CscEnt {w, key, row} (16 B, one vector load): key = (src + 1) << 27 | idx;
//           src < 0: constant value w; else value = lin[src][idx] * w with
//           w = val * sigma[col] folded on the host (val = +-1 for every linearized
//           entry, so lin * (val sigma) == (val lin) sigma bit for bit)
//   flags   one ballot per (stage j, warp) -> 64 masks in smem; one warp scans the
//           64 popcounts: offsets of every entry inside the tile; the tile total is
//           published and summed by the following tiles (decoupled look-back over
//           ticket-ordered tiles, as in k_csc_onepass)
//   indptr  the columns whose first superset entry lies in the tile (tcol[t] ..
//           tcol[t+1]) read their offset from the masks: no per-column pass at all
// Workspace ws: [ticket, finished CTAs, pad, pad] + one uint64 flag per tile, zero
// before the first launch; the last CTA returns it to zero.
// Concatenated output (out_rows[1] = out_vals[1] = null): matrix 1's entries follow
// matrix 0's nonzeros in out_rows[0] / out_vals[0] (its tiles look back over matrix
// 0's tiles too), its column pointers stay relative to its own first entry -- both
// matrices' values then sit in one array that comes back in one copy.
#define CSC_TJ 8
#define CSC_TILE (256 * CSC_TJ)

struct __align__(16) CscEnt {
  double w;
  uint32_t key;
  int32_t row;
};

struct CscPackedArgs {
  const CscEnt* ent[2];
  int64_t nsup[2];
  const int64_t* sp_ptr[2];
  const int32_t* tcol[2];  // ntile + 1 entries: first column owned by each tile, ncols + 1 at the end
  int32_t ntile[2];
  int32_t* out_ptr[2];
  int32_t* out_rows[2];
  double* out_vals[2];
  unsigned long long* rowmax[2];
  // pattern-change stamp (both null = off): a CTA that writes a row index or a
  // column pointer different from what the output held before stores *stamp_in
  // into *changed_at, so the host learns whether the CSC pattern moved since the
  // previous launch over the same outputs (and skips re-copying the indices)
  const double* stamp_in;
  double* changed_at;
  // host mirror (0 = off): the values (host_vals) / the pattern (host_pattern: the stamp,
  // and the column pointers and row indices while *rows_wanted != 0) are also stored
  // at that byte offset from their device address -- into page-locked host memory
  // laid out like the device outputs, so the result crosses the bus while the
  // compaction runs instead of in a copy after it
  int64_t host_vals, host_pattern;
  const double* rows_wanted;
  // optional (null = always): while *consts_wanted == 0 the host mirror already holds
  // this pattern's constant entries (src < 0: value w, the same every call), so 16-byte
  // chunks of constants only are not stored again
  const double* consts_wanted;
};

template <class T>
__device__ __forceinline__ void mirror_store(T* dev_addr, int64_t delta, T v) {
  *reinterpret_cast<T*>(reinterpret_cast<char*>(dev_addr) + delta) = v;
}

__global__ void __launch_bounds__(256) k_csc_flat(int32_t ncols, const CscPackedArgs a, const LinTable L,
                                                  unsigned* __restrict__ ws) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = a.ntile[0] + a.ntile[1];
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(ws + CSC_HDR_WORDS);
  __shared__ int tile_s, last_s, tbase_s, ttot_s, obase_s;
  __shared__ unsigned masks[CSC_TJ][8];
  __shared__ int base[CSC_TJ][8];
  __shared__ int red[8], red_b[8];
  // the tile's output staged for the host mirror: written back as whole 16-byte
  // chunks of its contiguous output range (full bus lines instead of scattered words)
  __shared__ __align__(16) double stage_v[CSC_TILE];
  __shared__ __align__(16) int32_t stage_r[CSC_TILE];
  __shared__ uint8_t stage_c[CSC_TILE];
  if (tid == 0) tile_s = (int)atomicAdd(&ws[0], 1u);
  __syncthreads();
  const int tile = tile_s;
  const int m = tile < a.ntile[0] ? 0 : 1;
  const int t0 = m ? a.ntile[0] : 0, lt = tile - t0;
  const bool concat = a.out_vals[1] == nullptr;
  const int64_t e0 = (int64_t)lt * CSC_TILE, nsup = a.nsup[m];
  const CscEnt* __restrict__ ent = a.ent[m];
  // evaluate the tile's entries: record loads first (all in flight), then the lin loads
  uint32_t key[CSC_TJ];
  int32_t row[CSC_TJ];
  double v[CSC_TJ];
#pragma unroll
  for (int j = 0; j < CSC_TJ; ++j) {
    const int64_t e = e0 + j * 256 + tid;
    if (e < nsup) {
      const CscEnt r = ent[e];
      v[j] = r.w;
      key[j] = r.key;
      row[j] = r.row;
    } else {
      v[j] = 0.0;
      key[j] = 0u;
      row[j] = 0;
    }
  }
  // launched with programmatic dependent launch behind the linearization: everything
  // above (ticket, record loads) overlapped the producer's tail; its results are read
  // only after this point (a no-op for a normal launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int j = 0; j < CSC_TJ; ++j) {
    const int s = (int)(key[j] >> 27) - 1;
    if (s >= 0) v[j] = lin_ptr(L, s)[key[j] & 0x7ffffffu] * v[j];
  }
#pragma unroll
  for (int j = 0; j < CSC_TJ; ++j) {
    const unsigned mk = __ballot_sync(0xffffffffu, v[j] != 0.0);
    if (lane == 0) masks[j][warp] = mk;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 64 (j, warp) popcounts in entry order
    const int i0 = 2 * lane, i1 = 2 * lane + 1;
    const int c0 = __popc(masks[i0 >> 3][i0 & 7]), c1 = __popc(masks[i1 >> 3][i1 & 7]);
    int incl = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int ex = incl - c0 - c1;
    base[i0 >> 3][i0 & 7] = ex;
    base[i1 >> 3][i1 & 7] = ex + c0;
    if (lane == 31) {
      ttot_s = incl;
      atomicExch(&flags[tile], (1ull << 32) | (unsigned)incl);  // publish the tile total
    }
  }
  // look-back: totals of the preceding tiles of this matrix (ticket order: all started
  // earlier); concatenated output: of matrix 0's tiles too (`before`: its nonzeros)
  int pre = 0, before = 0;
  for (int j = (concat ? 0 : t0) + tid; j < tile; j += blockDim.x) {
    unsigned long long f;
    do {
      f = *((volatile unsigned long long*)&flags[j]);
    } while ((f >> 32) == 0ull);
    const int cnt = (int)(unsigned)(f & 0xffffffffull);
    if (j >= t0)
      pre += cnt;
    else
      before += cnt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pre += __shfl_xor_sync(0xffffffffu, pre, o);
    before += __shfl_xor_sync(0xffffffffu, before, o);
  }
  if (lane == 0) {
    red[warp] = pre;
    red_b[warp] = before;
  }
  __syncthreads();
  if (tid == 0) {
    int t = 0, tb0 = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      t += red[w];
      tb0 += red_b[w];
    }
    tbase_s = t;
    obase_s = tb0;
    __threadfence();
    last_s = atomicAdd(&ws[1], 1u) == (unsigned)ntiles - 1u;
  }
  __syncthreads();
  if (last_s) {  // every CTA is past its look-back: clean the workspace for the next launch
    for (int j = tid; j < ntiles; j += blockDim.x) flags[j] = 0ull;
    if (tid == 0) {
      ws[0] = 0u;
      ws[1] = 0u;
    }
    __threadfence();
  }
  const int tb = tbase_s;
  const unsigned ltm = (1u << lane) - 1u;
  int32_t* __restrict__ orow = concat ? a.out_rows[0] + obase_s : a.out_rows[m];
  double* __restrict__ oval = concat ? a.out_vals[0] + obase_s : a.out_vals[m];
  unsigned long long* rmax = a.rowmax[m];
  const bool stamp = a.changed_at != nullptr;
  const int64_t hv = a.host_vals, hp = a.host_pattern, hr = (hp && *a.rows_wanted != 0.0) ? hp : 0;
  bool moved = false;
  // the previous launch's row indices at this tile's positions, all loads in flight
  // before the first store (one memory round trip for the stamp, not one per entry)
  int32_t old_row[CSC_TJ];
  if (stamp) {
#pragma unroll
    for (int j = 0; j < CSC_TJ; ++j)
      old_row[j] = v[j] != 0.0 ? orow[tb + base[j][warp] + __popc(masks[j][warp] & ltm)] : 0;
  }
#pragma unroll
  for (int j = 0; j < CSC_TJ; ++j) {
    if (v[j] != 0.0) {
      const int pos = tb + base[j][warp] + __popc(masks[j][warp] & ltm);
      if (stamp) moved |= old_row[j] != row[j];
      orow[pos] = row[j];
      oval[pos] = v[j];
      if (hv) {
        stage_v[pos - tb] = v[j];
        stage_c[pos - tb] = (key[j] >> 27) == 0u;  // a constant entry
      }
      if (hr) stage_r[pos - tb] = row[j];
      // fused row inf-norm (cito/conic.py:281-287): non-negative doubles order like their bits
      if (rmax) atomicMax(&rmax[row[j]], (unsigned long long)__double_as_longlong(fabs(v[j])));
    }
  }
  // indptr of the columns whose first superset entry lies in this tile
  const int64_t* __restrict__ sp = a.sp_ptr[m];
  const int c_lo = a.tcol[m][lt], c_hi = a.tcol[m][lt + 1];
  const int64_t nin = nsup - e0 < CSC_TILE ? nsup - e0 : CSC_TILE;
  for (int c = c_lo + tid; c < c_hi && c <= ncols; c += blockDim.x) {
    const int64_t l = sp[c] - e0;
    int cnt;
    if (l >= nin) {
      cnt = ttot_s;
    } else {
      const int j = (int)(l >> 8), r = (int)(l & 255), w = r >> 5, ln = r & 31;
      cnt = base[j][w] + __popc(masks[j][w] & ((1u << ln) - 1u));
    }
    if (stamp) moved |= a.out_ptr[m][c] != tb + cnt;
    a.out_ptr[m][c] = tb + cnt;
    if (hr) mirror_store(a.out_ptr[m] + c, hr, tb + cnt);  // the pattern: only into a buffer that wants it
  }
  if (stamp && __syncthreads_or(moved) && tid == 0) {
    *a.changed_at = *a.stamp_in;
    if (hp) mirror_store(a.changed_at, hp, *a.stamp_in);
  }
  if (hv || hr) {  // the staged range [tb, tb + ttot) -> host, 16-byte stores
    __syncthreads();
    const int n = ttot_s;
    if (hv) {
      double* hd = reinterpret_cast<double*>(reinterpret_cast<char*>(oval + tb) + hv);
      const int head = (reinterpret_cast<uintptr_t>(hd) & 15) ? 1 : 0;
      const int np = (n - head) >> 1;
      double2* d2 = reinterpret_cast<double2*>(hd + head);
      const bool cw = a.consts_wanted == nullptr || *a.consts_wanted != 0.0;
      for (int k = tid; k < np; k += blockDim.x) {
        const int e = head + 2 * k;
        if (cw || !(stage_c[e] && stage_c[e + 1])) d2[k] = make_double2(stage_v[e], stage_v[e + 1]);
      }
      if (tid == 0 && head && n > 0 && (cw || !stage_c[0])) hd[0] = stage_v[0];
      if (tid == 1 && n > head && ((n - head) & 1) && (cw || !stage_c[n - 1])) hd[n - 1] = stage_v[n - 1];
    }
    if (hr) {
      int32_t* hd = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(orow + tb) + hr);
      const int head = (int)((16 - (reinterpret_cast<uintptr_t>(hd) & 15)) & 15) / 4;
      const int h0 = head < n ? head : n;
      const int nq = (n - h0) >> 2;
      int4* d4 = reinterpret_cast<int4*>(hd + h0);
      for (int k = tid; k < nq; k += blockDim.x) {
        const int e = h0 + 4 * k;
        d4[k] = make_int4(stage_r[e], stage_r[e + 1], stage_r[e + 2], stage_r[e + 3]);
      }
      if (tid < h0) hd[tid] = stage_r[tid];
      const int t0e = h0 + 4 * nq;
      if (tid < n - t0e) hd[t0e + tid] = stage_r[t0e + tid];
    }
  }
}

__global__ void __launch_bounds__(256) k_rhs(int64_t nrows, const int32_t* __restrict__ rows,
                                             const int8_t* __restrict__ form, const int8_t* __restrict__ vsrc,
                                             const int64_t* __restrict__ voff, const int8_t* __restrict__ seg_src,
                                             const int64_t* __restrict__ seg_off, const int32_t* __restrict__ seg_len,
                                             const int64_t* __restrict__ seg_cb, const int64_t* __restrict__ cols,
                                             const double* __restrict__ z, const LinTable L,
                                             double* __restrict__ out, int64_t host) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= nrows) return;
  double dot = 0.0;
#pragma unroll
  for (int sgi = 0; sgi < 3; ++sgi) {
    const int s = seg_src[3 * i + sgi];
    if (s < 0) continue;
    const double* J = L.p[s] + seg_off[3 * i + sgi];
    const int64_t* cz = cols + seg_cb[3 * i + sgi];
    const int len = seg_len[3 * i + sgi];
    for (int j = lane; j < len; j += 32) dot += J[j] * z[cz[j]];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane == 0) {
    const double v = L.p[vsrc[i]][voff[i]];
    const double r = form[i] == 0 ? v - dot : dot - v;  // dynamics: ends - J.ref ; others: J.ref - value
    out[rows[i]] = r;
    if (host) mirror_store(out + rows[i], host, r);  // page-locked host mirror (0 = off)
  }
}

// ---------------------------------------------------------------------------
// Preconditioning of the assembled program on the device:
// cito.conic.precondition (/root/reference/pkg/src/cito/conic.py:290-338).
//   row inf-norms  (conic.py:281-287)  fused into k_csc_write, or k_row_absmax
//                                      for a program that was uploaded as is
//   row scales     (conic.py:294-309)  A and the orthant rows of G: 1/norm (1 for
//                                      an all-zero row); each SOC block of G
//                                      shares 1/max over its rows (1 if the max is 0)
//   scaling        (conic.py:321-331)  data[e] *= scale[row[e]], b *= sA, h *= sG
//                                      (Da @ A is one product per entry in scipy too,
//                                      so the scaled values are bit-identical)
struct PcArgs {
  const int32_t* ptr[2];
  const int32_t* rows[2];
  double* data[2];
  double* rhs[2];
  int32_t nrows[2];
  unsigned long long* rowmax[2];
  double* scale[2];
  double* keep[2];      // optional: the unscaled values are stored here before scaling
  double* keep_rhs[2];  // optional: the unscaled b / h
  int32_t concat;       // G's entries follow A's nonzeros in rows[0] / data[0] / keep[0]
  int64_t host;         // host mirror of every output (byte offset from the device address; 0 = off)
};

// entry arrays of matrix m (concatenated layout: G starts after A's nonzeros)
__device__ __forceinline__ int32_t pc_off(const PcArgs& a, int m, int32_t ncols) {
  return (a.concat && m == 1) ? a.ptr[0][ncols] : 0;
}

__global__ void __launch_bounds__(256) k_row_absmax(int32_t ncols, const PcArgs a) {
  const int m = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const int mm = a.concat ? 0 : m;
  const int32_t off = pc_off(a, m, ncols);
  for (int32_t e = a.ptr[m][c] + lane; e < a.ptr[m][c + 1]; e += 32) {
    const double v = a.data[mm][off + e];
    if (v != 0.0) atomicMax(&a.rowmax[m][a.rows[mm][off + e]], (unsigned long long)__double_as_longlong(fabs(v)));
  }
}

// one thread per A row, per orthant row of G, and per SOC block of G; every row
// max is read by exactly one thread, which returns it to zero for the next call
// (the fused norms of the next compaction accumulate into a zeroed workspace)
__global__ void __launch_bounds__(256) k_row_scale(const PcArgs a, int32_t n_nonneg, int32_t n_soc,
                                                   const int32_t* __restrict__ soc_start,
                                                   const int32_t* __restrict__ soc_dim) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nA = a.nrows[0];
  if (i < nA) {
    const double r = __longlong_as_double((long long)a.rowmax[0][i]);
    a.rowmax[0][i] = 0ull;
    a.scale[0][i] = 1.0 / (r == 0.0 ? 1.0 : r);  // ra[ra == 0] = 1; da = 1 / ra
    if (a.host) mirror_store(a.scale[0] + i, a.host, a.scale[0][i]);
    return;
  }
  const int64_t j = i - nA;
  if (j < n_nonneg) {
    const double r = __longlong_as_double((long long)a.rowmax[1][j]);
    a.rowmax[1][j] = 0ull;
    a.scale[1][j] = r != 0.0 ? 1.0 / r : 1.0;
    if (a.host) mirror_store(a.scale[1] + j, a.host, a.scale[1][j]);
    return;
  }
  const int64_t k = j - n_nonneg;
  if (k < n_soc) {
    const int32_t s0 = soc_start[k], d = soc_dim[k];
    double mx = 0.0;
    for (int32_t r = 0; r < d; ++r) {
      mx = fmax(mx, __longlong_as_double((long long)a.rowmax[1][s0 + r]));
      a.rowmax[1][s0 + r] = 0ull;
    }
    const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
    for (int32_t r = 0; r < d; ++r) {
      a.scale[1][s0 + r] = sc;
      if (a.host) mirror_store(a.scale[1] + s0 + r, a.host, sc);
    }
  }
}

// grid-stride over the stored entries (valid prefix = ptr[ncols]) and the rhs rows;
// the unscaled values go to keep / keep_rhs first when given
__global__ void __launch_bounds__(256) k_row_apply(int32_t ncols, const PcArgs a) {
  const int m = blockIdx.y, mm = a.concat ? 0 : m;
  const int32_t nnz = a.ptr[m][ncols], off = pc_off(a, m, ncols);
  const int64_t total = (int64_t)nnz + a.nrows[m];
  const double* __restrict__ sc = a.scale[m];
  double* __restrict__ data = a.data[mm] + off;
  const int32_t* __restrict__ rows = a.rows[mm] + off;
  double* __restrict__ keep = a.keep[mm] ? a.keep[mm] + off : nullptr;
  double* __restrict__ keep_rhs = a.keep_rhs[m];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nnz) {
      const double v = data[i];
      if (keep) keep[i] = v;
      const double w = sc[rows[i]] * v;
      data[i] = w;
      if (a.host) mirror_store(data + i, a.host, w);
    } else {
      const int64_t r = i - nnz;
      const double v = a.rhs[m][r];
      if (keep_rhs) keep_rhs[r] = v;
      a.rhs[m][r] = sc[r] * v;
      if (a.host) mirror_store(a.rhs[m] + r, a.host, sc[r] * v);
    }
  }
}
