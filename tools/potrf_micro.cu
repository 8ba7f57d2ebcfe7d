// Microbenchmark of 32x32 Cholesky (+ triangular inverse) variants inside one CTA (experiments only).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/potrf_micro tools/potrf_micro.cu && /tmp/potrf_micro
#include <cstdio>
#include <cmath>
#include <vector>

constexpr int TB = 32;

__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

template <int JJ>
__device__ __forceinline__ void chol_shfl(double (&a)[TB], int r) {
  if constexpr (JJ < TB) {
    const double dj = __shfl_sync(0xffffffffu, a[JJ], JJ);
    const double inv = rsqrt_nr(dj), piv = dj * inv;
    const double lr = r == JJ ? piv : (r > JJ ? a[JJ] * inv : 0.0);
    a[JJ] = lr;
#pragma unroll
    for (int c = JJ + 1; c < TB; ++c) {
      const double lc = __shfl_sync(0xffffffffu, lr, c);
      if (r >= c) a[c] = fma(-lr, lc, a[c]);
    }
    chol_shfl<JJ + 1>(a, r);
  }
}

// variant 1: one warp, shuffles (launched with 32 threads: no divergence)
// variant 2: one warp, column broadcast through shared memory
// variant 3: 256 threads, one barrier per column (smem right-looking)
template <int V>
__global__ void k(const double* __restrict__ in, double* __restrict__ out, long long* cyc, int reps) {
  __shared__ double s[TB][TB + 1];
  __shared__ double col[TB];
  const int t = threadIdx.x;
  long long best = 1ll << 60;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = t; e < TB * TB; e += blockDim.x) s[e / TB][e % TB] = in[e];
    __syncthreads();
    const long long t0 = clock64();
    if constexpr (V == 1) {
      const int r = t & 31;
      double a[TB];
#pragma unroll
      for (int c = 0; c < TB; ++c) a[c] = s[r][c];
      chol_shfl<0>(a, r);
#pragma unroll
      for (int c = 0; c < TB; ++c) s[r][c] = a[c];
    } else if constexpr (V == 2) {
      if (t < 32) {
        const int r = t;
        double a[TB];
#pragma unroll
        for (int c = 0; c < TB; ++c) a[c] = s[r][c];
#pragma unroll
        for (int jj = 0; jj < TB; ++jj) {
          if (r == jj) col[jj] = a[jj];
          __syncwarp();
          const double dj = col[jj];
          const double inv = rsqrt_nr(dj), piv = dj * inv;
          const double lr = r == jj ? piv : (r > jj ? a[jj] * inv : 0.0);
          a[jj] = lr;
          __syncwarp();
          col[r] = lr;
          __syncwarp();
#pragma unroll
          for (int c = jj + 1; c < TB; ++c)
            if (r >= c) a[c] = fma(-lr, col[c], a[c]);
          __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < TB; ++c) s[r][c] = a[c];
      }
    } else if constexpr (V == 4) {
      // blocked: four 8-column block steps; the 8x8 diagonal block is factored by ONE thread in
      // registers (no communication on the pivot chain), the 24x8 panel by one thread per row
      // (8-step substitution with the block's reciprocal diagonal), the trailing update by all threads
      __shared__ double rd[TB];
#pragma unroll 1
      for (int kb = 0; kb < TB; kb += 8) {
        if (t == 0) {
          double a[8][8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) a[i][j] = s[kb + i][kb + j];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double inv = rsqrt_nr(a[j][j]);
            a[j][j] = a[j][j] * inv;
            rd[kb + j] = inv;
#pragma unroll
            for (int i = j + 1; i < 8; ++i) a[i][j] *= inv;
#pragma unroll
            for (int i = j + 1; i < 8; ++i)
#pragma unroll
              for (int c = j + 1; c <= i; ++c) a[i][c] = fma(-a[i][j], a[c][j], a[i][c]);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) s[kb + i][kb + j] = a[i][j];
        }
        __syncthreads();
        const int rows = TB - kb - 8;
        if (t < rows) {  // panel row r: x L_kk^T = a  (x_c = (a_c - sum_{p<c} x_p l_cp) / l_cc)
          const int r = kb + 8 + t;
          double x[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            double v = s[r][kb + c];
#pragma unroll
            for (int p = 0; p < c; ++p) v = fma(-x[p], s[kb + c][kb + p], v);
            x[c] = v * rd[kb + c];
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) s[r][kb + c] = x[c];
        }
        __syncthreads();
        for (int e = t; e < rows * rows; e += blockDim.x) {  // trailing rank-8 update
          const int r = kb + 8 + e / rows, c = kb + 8 + e % rows;
          if (c <= r) {
            double v = s[r][c];
#pragma unroll
            for (int p = 0; p < 8; ++p) v = fma(-s[r][kb + p], s[c][kb + p], v);
            s[r][c] = v;
          }
        }
        __syncthreads();
      }
    } else {
      for (int jj = 0; jj < TB; ++jj) {
        const double dj = s[jj][jj];
        const double inv = rsqrt_nr(dj), inv2 = inv * inv;
        for (int e = t; e < TB * TB; e += blockDim.x) {
          const int r = e / TB, c = e % TB;
          if (c > jj && r >= c) s[r][c] -= s[r][jj] * s[c][jj] * inv2;
        }
        __syncthreads();
        if (t < TB && t >= jj) s[t][jj] = t == jj ? dj * inv : s[t][jj] * inv;
        __syncthreads();
      }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  for (int e = t; e < TB * TB; e += blockDim.x) out[e] = s[e / TB][e % TB];
  if (t == 0) *cyc = best;
}

int main() {
  std::vector<double> A(TB * TB), L(TB * TB);
  // SPD: M M^T + 32 I
  std::vector<double> M(TB * TB);
  unsigned s = 1;
  for (auto& v : M) { s = s * 1103515245u + 12345u; v = ((s >> 8) & 0xffff) / 65536.0 - 0.5; }
  for (int i = 0; i < TB; ++i)
    for (int j = 0; j < TB; ++j) {
      double v = i == j ? TB : 0.0;
      for (int k = 0; k < TB; ++k) v += M[i * TB + k] * M[j * TB + k];
      A[i * TB + j] = v;
    }
  double *din, *dout;
  long long* dc;
  cudaMalloc(&din, sizeof(double) * TB * TB);
  cudaMalloc(&dout, sizeof(double) * TB * TB);
  cudaMalloc(&dc, sizeof(long long));
  cudaMemcpy(din, A.data(), sizeof(double) * TB * TB, cudaMemcpyHostToDevice);
  auto run = [&](auto kern, int threads, const char* name) {
    kern<<<1, threads>>>(din, dout, dc, 50);
    long long c = 0;
    cudaMemcpy(&c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    cudaMemcpy(L.data(), dout, sizeof(double) * TB * TB, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < TB; ++i)
      for (int j = 0; j <= i; ++j) {
        double v = 0;
        for (int k = 0; k <= j; ++k) v += L[i * TB + k] * L[j * TB + k];
        err = fmax(err, fabs(v - A[i * TB + j]));
      }
    printf("%-28s %8lld cycles  (%.2f us at 1.965 GHz)  max|LL^T-A| %.2e  %s\n", name, c, c / 1965.0, err,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(k<1>, 32, "warp shuffles (32 thr)");
  run(k<2>, 256, "warp smem broadcast (256)");
  run(k<3>, 256, "CTA smem barriers (256)");
  run(k<4>, 256, "blocked 8, 1-thread diag (256)");
  return 0;
}
