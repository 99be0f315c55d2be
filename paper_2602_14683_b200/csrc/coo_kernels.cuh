// K7: sparse COO count tensors at beta = 1 (new; the reference has no sparse
// path -- read_coo io.cpp:87-142 densifies, SURVEY.md 8(c) "Sparse path").
//
// At beta = 1, P = X / max(Xhat, eps) vanishes where X = 0 and Q == 1, so
//   Num^(n)(i_n, r) = sum_{nnz} p * prod_{m != n} A_m(i_m, r)        (cp.cpp:117)
//   Den^(n)(r)      = prod_{m != n} colsum(A_m)(r)                    (cp.cpp:119-120)
//   D_1(X | Xhat)   = sum_{nnz} [x log(x / y) - x] + sum_{all} y      (divergence.cpp:20)
// and sum_all y = sum_r prod_m colsum(A_m)(r) is closed form too.  The dense
// engine's factor-side machinery (MU finalize, J-CoMM N1 inner loop, BMMe,
// fit loop) is reused unchanged; only the X passes are replaced.
//
// Determinism: no float atomics.  Each mode has its own copy of the nonzeros
// sorted by i_n (stable, duplicates merged in input order at ingestion); the
// copy is cut into "pieces" of <= kCooPiece nonzeros that never straddle two
// keys.  coo_piece_kernel sums one piece per warp in nonzero order,
// coo_key_reduce_kernel sums the pieces of one key in a fixed strided tree.
#pragma once
#include <cstdint>

#include "cp_kernels.cuh"
#include "device_math.cuh"

namespace ntfg {

constexpr int kCooPiece = 256;

struct CooPieceParams {
  int order, n, R;
  const int32_t* idx[kMaxOrder];  // SoA indices of this mode's sorted copy
  const double* val;
  const int64_t* piece_start;     // [npieces + 1]
  int64_t npieces;
  const double* fac[kMaxOrder];   // model factors [I_m][R]
  double eps;
  double* partial;                // [npieces][R] (nullable: objective only)
  double* obj;                    // [npieces] nnz part of D_1 (nullable)
  unsigned* flags;
};

// one warp per piece; lane l holds ranks l, l + 32, ... (RW per lane)
template <int RW>
static __global__ void __launch_bounds__(256) coo_piece_kernel(const CooPieceParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned bad = 0;
  for (int64_t pc = warp0; pc < p.npieces; pc += nwarps) {
    const int64_t j0 = p.piece_start[pc], j1 = p.piece_start[pc + 1];
    double acc[RW];
#pragma unroll
    for (int w = 0; w < RW; ++w) acc[w] = 0.0;
    double obj = 0.0;
    for (int64_t jb = j0; jb < j1; jb += 32) {
      const int cnt = int(j1 - jb < 32 ? j1 - jb : 32);
      // lane l stages nonzero jb + l; broadcast below
      int32_t my[kMaxOrder];
#pragma unroll
      for (int m = 0; m < kMaxOrder; ++m) my[m] = (m < p.order && lane < cnt) ? p.idx[m][jb + lane] : 0;
      const double myx = lane < cnt ? p.val[jb + lane] : 0.0;
#pragma unroll 2
      for (int t = 0; t < cnt; ++t) {
        double a[kMaxOrder][RW];
#pragma unroll
        for (int m = 0; m < kMaxOrder; ++m) {
          if (m >= p.order) break;
          const int64_t im = __shfl_sync(0xffffffffu, my[m], t);
#pragma unroll
          for (int w = 0; w < RW; ++w) {
            const int r = lane + 32 * w;
            a[m][w] = r < p.R ? __ldg(p.fac[m] + im * p.R + r) : 0.0;
          }
        }
        const double x = __shfl_sync(0xffffffffu, myx, t);
        // Xhat = sum_r prod_m A_m(i_m, r)   (cp.cpp:26-76, ascending m)
        double part = 0.0, off[RW];
#pragma unroll
        for (int w = 0; w < RW; ++w) {
          double all = 1.0, o = 1.0;
#pragma unroll
          for (int m = 0; m < kMaxOrder; ++m) {
            if (m >= p.order) break;
            all *= a[m][w];
            if (m != p.n) o *= a[m][w];
          }
          part += all;
          off[w] = o;
        }
        const double y = warp_sum(part);
        const double c = y < p.eps ? p.eps : y;  // std::max(xhat, eps)
        const double pw = x / c;                 // weight_entries beta = 1 (kernels.hpp)
#pragma unroll
        for (int w = 0; w < RW; ++w) acc[w] = fma(pw, off[w], acc[w]);
        if (p.obj && lane == 0) {
          if (!(y > 0.0)) bad |= 1u;
          if (x < 0.0) bad |= 2u;
          if (x > 0.0 && y > 0.0) obj += x * log(x / y) - x;  // + y: closed form
        }
      }
    }
    if (p.partial) {
#pragma unroll
      for (int w = 0; w < RW; ++w) {
        const int r = lane + 32 * w;
        if (r < p.R) p.partial[pc * p.R + r] = acc[w];
      }
    }
    if (p.obj && lane == 0) p.obj[pc] = obj;
  }
  if (bad && p.flags) atomicOr(p.flags, bad);
}

// Lane-per-nonzero version (round 2).  ncu of the kernel above at C4: 73% issue
// utilisation, 235 warp instructions per nonzero -- every nonzero costs the
// whole warp two index shuffles per mode, a 10-shuffle fp64 warp sum and a
// 20-of-32-lane gather.  Here a warp takes 32 nonzeros of its piece at once:
//   phase 1 (lane = nonzero): Xhat = sum_r prod_m A_m(i_m, r) sequentially in r
//           (each lane streams its own N factor rows: 16-byte loads, the
//           second visit hits L1), p = x / max(Xhat, eps), and the off-mode
//           products prod_{m != n} A_m(i_m, r) go to shared memory [32][R|1];
//   phase 2 (lane = rank): acc(r) = fma(p_j, off_j(r), acc(r)) over the batch in
//           nonzero order -- the same fma chain per rank as before.
// No shuffles, no atomics; the summation order per (piece, rank) is unchanged,
// Xhat is now a sequential sum over r (was a butterfly over lanes).
constexpr int kCooWarps = 4;  // warps per CTA (shared memory: 32 x (R|1) doubles each)
inline size_t coo_piece2_smem(int R) { return size_t(kCooWarps) * (size_t(32) * (R | 1) + 64) * sizeof(double); }

static __global__ void __launch_bounds__(kCooWarps * 32) coo_piece2_kernel(const CooPieceParams p) {
  extern __shared__ __align__(16) double coo_sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int R = p.R, RS = R | 1;
  double* off = coo_sm + size_t(w) * (size_t(32) * RS + 64);
  double* pj = off + size_t(32) * RS;
  double* tj = pj + 32;
  const int64_t warp0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const bool vec = (R & 1) == 0;  // rows of R doubles start 16-byte aligned
  unsigned bad = 0;
  for (int64_t pc = warp0; pc < p.npieces; pc += nwarps) {
    const int64_t j0 = p.piece_start[pc], j1 = p.piece_start[pc + 1];
    double acc0 = 0.0, acc1 = 0.0, obj = 0.0;
    for (int64_t jb = j0; jb < j1; jb += 32) {
      const int cnt = int(j1 - jb < 32 ? j1 - jb : 32);
      if (lane < cnt) {
        const double* row[kMaxOrder];
#pragma unroll
        for (int m = 0; m < kMaxOrder; ++m)
          row[m] = m < p.order ? p.fac[m] + int64_t(p.idx[m][jb + lane]) * R : nullptr;
        const double x = p.val[jb + lane];
        double y = 0.0;
        if (vec) {
#pragma unroll 5
          for (int r = 0; r < R; r += 2) {
            double2 a = __ldg(reinterpret_cast<const double2*>(row[0] + r));
#pragma unroll
            for (int m = 1; m < kMaxOrder; ++m) {
              if (m >= p.order) break;
              const double2 b = __ldg(reinterpret_cast<const double2*>(row[m] + r));
              a.x *= b.x;
              a.y *= b.y;
            }
            y += a.x;
            y += a.y;
          }
        } else {
          for (int r = 0; r < R; ++r) {
            double a = __ldg(row[0] + r);
#pragma unroll
            for (int m = 1; m < kMaxOrder; ++m) {
              if (m >= p.order) break;
              a *= __ldg(row[m] + r);
            }
            y += a;
          }
        }
        const double c = y < p.eps ? p.eps : y;  // std::max(xhat, eps)
        pj[lane] = x / c;                        // weight_entries beta = 1 (kernels.hpp)
        if (p.partial) {
          double* orow = off + size_t(lane) * RS;
#pragma unroll 4
          for (int r = 0; r < R; ++r) {
            double o = 1.0;
#pragma unroll
            for (int m = 0; m < kMaxOrder; ++m) {
              if (m >= p.order) break;
              if (m != p.n) o *= __ldg(row[m] + r);
            }
            orow[r] = o;
          }
        }
        if (p.obj) {
          if (!(y > 0.0)) bad |= 1u;
          if (x < 0.0) bad |= 2u;
          tj[lane] = (x > 0.0 && y > 0.0) ? x * log(x / y) - x : 0.0;  // + y: closed form
        }
      }
      __syncwarp();
      if (p.partial) {
        if (lane < R) {
#pragma unroll 4
          for (int t = 0; t < cnt; ++t) acc0 = fma(pj[t], off[size_t(t) * RS + lane], acc0);
        }
        if (lane + 32 < R) {
#pragma unroll 4
          for (int t = 0; t < cnt; ++t) acc1 = fma(pj[t], off[size_t(t) * RS + lane + 32], acc1);
        }
      }
      if (p.obj && lane == 0)
        for (int t = 0; t < cnt; ++t) obj += tj[t];
      __syncwarp();
    }
    if (p.partial) {
      if (lane < R) p.partial[pc * R + lane] = acc0;
      if (lane + 32 < R) p.partial[pc * R + lane + 32] = acc1;
    }
    if (p.obj && lane == 0) p.obj[pc] = obj;
  }
  if (bad && p.flags) atomicOr(p.flags, bad);
}

// Num(k, r) = sum of the pieces of key k: 8 warps take pieces k0 + w, k0 + w + 8,
// ... in order, then warps combine in order (fixed shape => deterministic).
static __global__ void __launch_bounds__(256) coo_key_reduce_kernel(const double* partial, const int64_t* key_piece,
                                                                   int64_t keys, int R, double* num) {
  __shared__ double red[8][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t k = blockIdx.x; k < keys; k += gridDim.x) {
    const int64_t p0 = key_piece[k], p1 = key_piece[k + 1];
    for (int r0 = 0; r0 < R; r0 += 64) {
      double s0 = 0.0, s1 = 0.0;
      for (int64_t pc = p0 + warp; pc < p1; pc += 8) {
        if (r0 + lane < R) s0 += partial[pc * R + r0 + lane];
        if (r0 + lane + 32 < R) s1 += partial[pc * R + r0 + lane + 32];
      }
      red[warp][lane] = s0;
      red[warp][lane + 32] = s1;
      __syncthreads();
      if (threadIdx.x < 64 && r0 + int(threadIdx.x) < R) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
        num[k * R + r0 + threadIdx.x] = s;
      }
      __syncthreads();
    }
  }
}

// sum_r colprod[r] (closed-form sum of Xhat over all entries) -> *out
static __global__ void closed_sum_kernel(const double* colprod, int R, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int r = 0; r < R; ++r) s += colprod[r];
    *out = s;
  }
}

}  // namespace ntfg
