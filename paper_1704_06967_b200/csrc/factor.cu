// Dense factorization and solves of the 6F x 6F reduced camera system S (the reference's
// Eigen::LDLT of the Schur complement, solver.cpp:190-194 / :393 and reduced_ldlt_.solve :417).
//
// k_chol_tiles: factor-only tiled Cholesky S = L L^T (tiles of 32 x 32, lower triangle in place)
// as a dataflow over the tiles instead of a sequence of grid-wide phases.  Tile (i, j) is one task
// (left-looking): its owner CTA accumulates sum_k L_ik L_jk^T (k < j) on the FP64 tensor path
// (mma.sync.m8n8k4.f64) as soon as the two source tiles are published, then either factors it
// (i == j: L_jj and Dinv_j = L_jj^-1) or solves it (L_ij = (A_ij - sum) Dinv_j^T), and publishes it
// with a release-store of the call's epoch into the tile's flag.  Tasks are dealt to the persistent
// CTAs in (column, row) order, which is a topological order of the dependencies, so in-order
// processing with all CTAs co-resident (cooperative launch) cannot deadlock, and no CTA ever waits
// at a grid barrier: the critical path is the chain POTRF(j) -> TRSM(j+1, j) -> POTRF(j+1).
// Every tile's sum is formed in the same k order by one CTA: results are bitwise reproducible.
//
// With X given, the same dataflow also forms the explicit inverse X = L^-1 (and X^T) tile by tile
// (inv_task), so every later solve is two GEMVs; the inverse tasks of block row i only need factor
// step i, so they run in the factorization's shadow.

#include <algorithm>
#include <cstdio>

#include "kernels.hpp"

namespace pba_b200 {
namespace {

constexpr int TB = 32;   // tile edge
constexpr int FT = 256;  // threads per CTA (8 warps: two 8x8 DMMA tiles each)

struct TileSmem {
  double a[TB][TB + 1];
  double b[TB][TB + 1];
  double c[TB][TB + 1];
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }

__device__ __forceinline__ void wait_epoch(const int* f, int epoch) {
  int v;
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  } while (v < epoch);
}
__device__ __forceinline__ void publish(int* f, int epoch) {
  __threadfence();
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
}

// tile (r0, c0) of the row-major n x n matrix M (L2 reads: written by other CTAs); outside -> 0
__device__ __forceinline__ void load_tile(double (*t)[TB + 1], const double* __restrict__ M, int n, int r0, int c0,
                                          bool trans) {
#pragma unroll
  for (int q = 0; q < TB * TB / FT; ++q) {
    const int e = threadIdx.x + q * FT, r = e / TB, c = e % TB;
    const int gr = r0 + r, gc = c0 + c;
    const double v = (gr < n && gc < n) ? __ldcg(M + static_cast<int64_t>(gr) * n + gc) : 0.0;
    if (trans) t[c][r] = v; else t[r][c] = v;
  }
}
// d += x y (x[r][p], y[p][c]) in the m8n8k4 fragment layout: warp w covers rows 8 (w >> 1) ..,
// columns 16 (w & 1) .. (two 8x8 output tiles)
__device__ __forceinline__ void mma_tile(const double (*x)[TB + 1], const double (*y)[TB + 1], double (&d)[2][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = warp >> 1, tj0 = 2 * (warp & 1);
#pragma unroll
  for (int p0 = 0; p0 < TB; p0 += 4) {
    const double av = x[8 * ti + (lane >> 2)][p0 + (lane & 3)];
#pragma unroll
    for (int u = 0; u < 2; ++u) dmma(d[u][0], d[u][1], av, y[p0 + (lane & 3)][8 * (tj0 + u) + (lane >> 2)]);
  }
}
__device__ __forceinline__ void frag_to_smem(double (*t)[TB + 1], const double (&d)[2][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = warp >> 1, tj0 = 2 * (warp & 1);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    t[8 * ti + (lane >> 2)][8 * (tj0 + u) + 2 * (lane & 3)] = d[u][0];
    t[8 * ti + (lane >> 2)][8 * (tj0 + u) + 2 * (lane & 3) + 1] = d[u][1];
  }
}

// 1/sqrt(d) for normal d > 0: hardware approximation + two Newton steps, branch-free (the library
// rsqrt's per-lane slow path would split warps)
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

// Factor the updated diagonal tile in sm.a in place (kb valid rows/columns, identity padding):
// L -> A and Dinv = L^-1 -> Dinv.  Blocked by 8 columns: the 8 x 8 diagonal block is factored by
// ONE thread in registers (the pivot chain needs no communication), the panel below it by one
// thread per row (8-step substitution with the block's reciprocal diagonal), the trailing rank-8
// update by all threads (3 CTA barriers per block step; 3.5 us vs 4.8 us for a warp-shuffle
// factorization and 12.5 us with a barrier per column, tools/potrf_micro.cu).  Dinv is then formed
// column-parallel by forward substitution with the reciprocal diagonal.
__device__ void potrf_tile(TileSmem& sm, double* __restrict__ A, int n, int j, int kb, double* __restrict__ Dinv,
                           int* __restrict__ fail) {
  double (*s)[TB + 1] = sm.a;
  double* rd = &sm.c[0][0];  // reciprocal diagonal of L
  const int t = threadIdx.x;
#pragma unroll
  for (int q = 0; q < TB * TB / FT; ++q) {
    const int e = t + q * FT, r = e / TB, c = e % TB;
    if (r >= kb || c >= kb) s[r][c] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
#pragma unroll 1
  for (int k0 = 0; k0 < TB; k0 += 8) {
    if (t == 0) {
      double a[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c) a[i][c] = s[k0 + i][k0 + c];
      bool bad = false;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double d = a[c][c];
        if (!(d > 0.0) || !isfinite(d)) {  // not positive definite (Cholesky of the LDLT's SPD case)
          bad = true;
          d = 1.0;
        }
        const double inv = rsqrt_nr(d);
        a[c][c] = d * inv;
        rd[k0 + c] = inv;
#pragma unroll
        for (int i = c + 1; i < 8; ++i) a[i][c] *= inv;
#pragma unroll
        for (int i = c + 1; i < 8; ++i)
#pragma unroll
          for (int q = c + 1; q <= i; ++q) a[i][q] = fma(-a[i][c], a[q][c], a[i][q]);
      }
      if (bad) *fail = 1;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c) s[k0 + i][k0 + c] = a[i][c];
    }
    __syncthreads();
    const int rows = TB - k0 - 8;
    if (t < rows) {  // panel row r: x L_kk^T = a (x_c = (a_c - sum_{p<c} x_p l_cp) / l_cc)
      const int r = k0 + 8 + t;
      double x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double v = s[r][k0 + c];
#pragma unroll
        for (int p = 0; p < c; ++p) v = fma(-x[p], s[k0 + c][k0 + p], v);
        x[c] = v * rd[k0 + c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) s[r][k0 + c] = x[c];
    }
    __syncthreads();
    for (int e = t; e < rows * rows; e += FT) {  // trailing rank-8 update of the lower part
      const int r = k0 + 8 + e / rows, c = k0 + 8 + e % rows;
      if (c <= r) {
        double v = s[r][c];
#pragma unroll
        for (int p = 0; p < 8; ++p) v = fma(-s[r][k0 + p], s[c][k0 + p], v);
        s[r][c] = v;
      }
    }
    __syncthreads();
  }
  const int j0 = j * TB;
#pragma unroll
  for (int q = 0; q < TB * TB / FT; ++q) {
    const int e = t + q * FT, r = e / TB, c = e % TB;
    if (r < kb && c <= r) A[static_cast<int64_t>(j0 + r) * n + j0 + c] = s[r][c];
  }
  // Dinv = L^-1 by 8 x 8 blocks: the diagonal blocks X_bb by forward substitution (one thread per
  // column of each block), then X_ij = -X_ii sum_{k=j}^{i-1} L_ik X_kj level by level (i - j = 1, 2, 3)
  double (*xs)[TB + 1] = sm.b;
#pragma unroll
  for (int q = 0; q < TB * TB / FT; ++q) {
    const int e = t + q * FT;
    xs[e / TB][e % TB] = 0.0;
  }
  __syncthreads();
  if (t < TB) {
    const int b8 = (t >> 3) * 8, c = t & 7;
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int p = 0; p < r; ++p) v = fma(-s[b8 + r][b8 + p], x[p], v);
      x[r] = r < c ? 0.0 : v * rd[b8 + r];
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) xs[b8 + r][b8 + c] = x[r];
  }
  __syncthreads();
  double (*tt)[TB + 1] = sm.c + 1;  // rows 1.. of sm.c (row 0 holds rd)
#pragma unroll 1
  for (int lv = 1; lv < 4; ++lv) {
    const int nb = 4 - lv;  // blocks (i, j = i - lv), i = lv .. 3
    if (t < nb * 64) {
      const int q = t >> 6, r = (t >> 3) & 7, c = t & 7, i8 = (lv + q) * 8, j8 = q * 8;
      double v = 0.0;
      for (int k8 = j8; k8 < i8; k8 += 8)
#pragma unroll
        for (int p = 0; p < 8; ++p) v = fma(s[i8 + r][k8 + p], xs[k8 + p][j8 + c], v);
      tt[8 * q + r][c] = v;
    }
    __syncthreads();
    if (t < nb * 64) {
      const int q = t >> 6, r = (t >> 3) & 7, c = t & 7, i8 = (lv + q) * 8, j8 = q * 8;
      double v = 0.0;
#pragma unroll
      for (int p = 0; p < 8; ++p) v = fma(xs[i8 + r][i8 + p], tt[8 * q + p][c], v);
      xs[i8 + r][j8 + c] = -v;
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < TB * TB / FT; ++q) {
    const int e = t + q * FT;
    Dinv[static_cast<int64_t>(j) * TB * TB + e] = xs[e / TB][e % TB];
  }
}

#ifdef PBA_CHOL_TRACE
__device__ unsigned long long g_chol_trace[4 * 2048];  // per task: start, accumulated, diag ready, published
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CHOL_TRACE(slot) \
  if (threadIdx.x == 0 && t < 2048) g_chol_trace[4 * t + (slot)] = gtime()
#else
#define CHOL_TRACE(slot)
#endif

// Inverse task (i, j), i > j: X_ij = -Dinv_i sum_{k=j}^{i-1} L_ik X_kj (X_jj = Dinv_j), left-looking
// over k as the tiles are published; stores X_ij and X^T_ji (the two GEMVs of every later solve).
__device__ void inv_task(TileSmem& sm, const double* __restrict__ A, int n, const double* __restrict__ Dinv,
                         double* __restrict__ X, double* __restrict__ XT, const int* __restrict__ flags,
                         int* __restrict__ xflags, int epoch, int i, int j) {
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int k = j; k < i; ++k) {
    if (threadIdx.x == 0) {
      wait_epoch(flags + tri(i, k), epoch);                         // L_ik
      wait_epoch(k == j ? flags + tri(j, j) : xflags + tri(k, j), epoch);  // X_kj
    }
    __syncthreads();
    load_tile(sm.a, A, n, i * TB, k * TB, false);
    if (k == j) {
#pragma unroll
      for (int q = 0; q < TB * TB / FT; ++q) {
        const int e = threadIdx.x + q * FT;
        sm.b[e / TB][e % TB] = __ldcg(Dinv + static_cast<int64_t>(j) * TB * TB + e);
      }
    } else {
      load_tile(sm.b, X, n, k * TB, j * TB, false);
    }
    __syncthreads();
    mma_tile(sm.a, sm.b, d);
    __syncthreads();
  }
  frag_to_smem(sm.c, d);
  if (threadIdx.x == 0) wait_epoch(flags + tri(i, i), epoch);  // Dinv_i
  __syncthreads();
#pragma unroll
  for (int q = 0; q < TB * TB / FT; ++q) {
    const int e = threadIdx.x + q * FT;
    sm.a[e / TB][e % TB] = __ldcg(Dinv + static_cast<int64_t>(i) * TB * TB + e);
  }
  __syncthreads();
  double x[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  mma_tile(sm.a, sm.c, x);
  frag_to_smem(sm.b, x);
  __syncthreads();
  const int i0 = i * TB, j0 = j * TB;
#pragma unroll
  for (int q = 0; q < TB * TB / FT; ++q) {
    const int e = threadIdx.x + q * FT, r = e / TB, c = e % TB;
    if (i0 + r < n && j0 + c < n) {
      X[static_cast<int64_t>(i0 + r) * n + j0 + c] = -sm.b[r][c];
      XT[static_cast<int64_t>(j0 + c) * n + i0 + r] = -sm.b[r][c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) publish(xflags + tri(i, j), epoch);
}

__global__ void __launch_bounds__(FT, 1) k_chol_tiles(double* __restrict__ A, int n, double* __restrict__ Dinv,
                                                      double* __restrict__ X, double* __restrict__ XT,
                                                      int* __restrict__ flags, int* __restrict__ xflags, int epoch,
                                                      int* __restrict__ fail) {
  __shared__ TileSmem sm;
  const int nblk = (n + TB - 1) / TB;
  // Task order (a topological order of the dependencies): step s = the factor tiles of column s (rows
  // s .. nblk-1), then the inverse tiles of row s (columns 0 .. s-1), which need exactly factor
  // step s; nblk tasks per step.
  for (int t = blockIdx.x; t < nblk * nblk; t += gridDim.x) {
    const int step = t / nblk, u = t % nblk;
    if (u >= nblk - step) {
      if (X) inv_task(sm, A, n, Dinv, X, XT, flags, xflags, epoch, step, u - (nblk - step));
      continue;
    }
    const int j = step, i = step + u;
    CHOL_TRACE(0);
    // A_ij is read only by this task (before it is overwritten): load it now, off the critical path
    double aij[TB * TB / FT];
#pragma unroll
    for (int q = 0; q < TB * TB / FT; ++q) {
      const int e = threadIdx.x + q * FT, gr = i * TB + e / TB, gc = j * TB + e % TB;
      aij[q] = (gr < n && gc < n) ? __ldcg(A + static_cast<int64_t>(gr) * n + gc) : 0.0;
    }
    double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int k = 0; k < j; ++k) {  // left-looking: sum_k L_ik L_jk^T in fixed k order
      if (threadIdx.x == 0) {
        wait_epoch(flags + tri(i, k), epoch);
        if (i != j) wait_epoch(flags + tri(j, k), epoch);
      }
      __syncthreads();
      load_tile(sm.a, A, n, i * TB, k * TB, false);
      load_tile(sm.b, A, n, j * TB, k * TB, true);
      __syncthreads();
      mma_tile(sm.a, sm.b, d);
      __syncthreads();
    }
    CHOL_TRACE(1);
    frag_to_smem(sm.c, d);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < TB * TB / FT; ++q) {
      const int e = threadIdx.x + q * FT;
      sm.a[e / TB][e % TB] = aij[q] - sm.c[e / TB][e % TB];
    }
    __syncthreads();
    if (i == j) {
      potrf_tile(sm, A, n, j, min(TB, n - j * TB), Dinv, fail);
      if (X) {  // X_jj = Dinv_j
        __syncthreads();
        const int j0 = j * TB;
#pragma unroll
        for (int q = 0; q < TB * TB / FT; ++q) {
          const int e = threadIdx.x + q * FT, r = e / TB, c = e % TB;
          if (j0 + r < n && j0 + c < n) {
            const double v = sm.b[r][c];  // potrf_tile leaves Dinv_j in sm.b
            X[static_cast<int64_t>(j0 + r) * n + j0 + c] = v;
            XT[static_cast<int64_t>(j0 + c) * n + j0 + r] = v;
          }
        }
      }
    } else {
      if (threadIdx.x == 0) wait_epoch(flags + tri(j, j), epoch);
      __syncthreads();
      CHOL_TRACE(2);
#pragma unroll
      for (int q = 0; q < TB * TB / FT; ++q) {  // Dinv_j^T
        const int e = threadIdx.x + q * FT, r = e / TB, c = e % TB;
        sm.b[c][r] = __ldcg(Dinv + (static_cast<int64_t>(j) * TB + r) * TB + c);
      }
      __syncthreads();
      double x[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      mma_tile(sm.a, sm.b, x);
      frag_to_smem(sm.c, x);
      __syncthreads();
      const int i0 = i * TB, j0 = j * TB;
#pragma unroll
      for (int q = 0; q < TB * TB / FT; ++q) {
        const int e = threadIdx.x + q * FT, r = e / TB, c = e % TB;
        if (i0 + r < n && j0 + c < n) A[static_cast<int64_t>(i0 + r) * n + j0 + c] = sm.c[r][c];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) publish(flags + tri(i, j), epoch);
    CHOL_TRACE(3);
  }
}

int chol_tiles_grid() {
  static int g = [] {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_tiles, FT, 0);
    return std::max(1, sms * std::max(1, per));
  }();
  return g;
}

}  // namespace

#ifdef PBA_CHOL_TRACE
void dump_chol_trace(int n);
#endif
void launch_chol_tiles(double* S, int n, double* Dinv, double* X, double* XT, int* flags, int epoch, int* fail,
                       cudaStream_t s) {
  if (n == 0) return;
  const int nblk = (n + TB - 1) / TB;
  const int grid = std::min(chol_tiles_grid(), nblk * nblk);
  int* xflags = flags + chol_tile_flags(n);
  void* args[] = {&S, &n, &Dinv, &X, &XT, &flags, &xflags, &epoch, &fail};
  // cooperative: every CTA co-resident, so the in-order task waits always resolve
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_chol_tiles), dim3(grid), dim3(FT),
                                                    args, 0, s);
  if (e != cudaSuccess) std::fprintf(stderr, "k_chol_tiles launch: %s\n", cudaGetErrorString(e));
  count_launches(1);
#ifdef PBA_CHOL_TRACE
  static int calls = 0;
  if (++calls == 3) dump_chol_trace(n);  // a warm call
#endif
}

#ifdef PBA_CHOL_TRACE
void dump_chol_trace(int n) {
  const int nblk = (n + TB - 1) / TB;
  static unsigned long long h[4 * 2048];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_chol_trace, sizeof(h));
  unsigned long long t0 = ~0ull;
  for (int t = 0; t < nblk * nblk && t < 2048; ++t)
    if (h[4 * t]) t0 = std::min(t0, h[4 * t]);
  FILE* f = std::fopen("gpurun_out/chol_trace.csv", "w");
  if (!f) return;
  std::fprintf(f, "task,i,j,start_us,acc_us,diag_us,pub_us\n");
  for (int t = 0; t < nblk * nblk && t < 2048; ++t) {
    const int step = t / nblk, u = t % nblk;
    if (u >= nblk - step) continue;  // inverse task (not traced)
    const int i = step + u, j = step;
    std::fprintf(f, "%d,%d,%d,%.3f,%.3f,%.3f,%.3f\n", t, i, j, (h[4 * t] - t0) * 1e-3, (h[4 * t + 1] - t0) * 1e-3,
                 h[4 * t + 2] ? (h[4 * t + 2] - t0) * 1e-3 : -1.0, (h[4 * t + 3] - t0) * 1e-3);
  }
  std::fclose(f);
}
#endif

int chol_tile_flags(int n) {  // per array: the factor's flags, then the inverse's
  const int nblk = (n + TB - 1) / TB;
  return nblk * (nblk + 1) / 2;
}


}  // namespace pba_b200
