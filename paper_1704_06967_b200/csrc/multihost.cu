// Joint multi-host window with per-frame affine brightness on the B200 (include/pba_gpu.h
// pba_gpu_mh_*).  The model and its equations are stated in
// oracle/multihost.cpp, which this path is checked against; the reference has no multi-host
// solver.  Forwards compositional, with the reference's FC LM rules (solver.cpp:685-843).
//
// Device pipeline per candidate evaluation:
//   k_mh_obs     one thread per observation (n, t): warp through T_t T_h^-1, bilinear + image
//                gradient of the target (the FC pass's fused taps), Huber, and the 54-double
//                record of sums in RELATIVE coordinates: z = [J_omega, J_dt, J_d, j_a] of the
//                reference's FC row at the relative pose plus the affine column; Z = sum w z z^T,
//                sum w z, sum w, sum w r z, sum w r; plus energy / counts / max update per obs.
//   k_mh_pair_*  per (host, target) pair: the records of its observations summed in order; the
//                pair's chain matrix T (absolute <- relative increments: [u]x, R_th, alpha, b_h)
//                is a pair constant, so H_FF and g_F come from the pair sums (linearity).
//   k_mh_frames  H_FF and g_F: every entry sums its pairs' mapped blocks in pair order.
//   k_mh_point   per point: b_n (dense over the frame parameters), D_n, g_n from its records.
//   k_mh_schur   S = H_FF + lambda I - sum_n b_n b_n^T / (D_n + lambda), rhs: one thread per
//                entry, points in order (deterministic); then the fused Cholesky + explicit
//                inverse (k_chol_inv) and the triangular GEMVs of the single-host path.
//   k_mh_backsub dx_n, the candidate depths and frame parameters, the gauge mean.
// Every reduction has a fixed order: runs are bitwise reproducible.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"

namespace pba_b200 {

namespace {

constexpr int MH_REC = 54;   // doubles per observation record
constexpr int MH_Z = 8;      // z = [w0 w1 w2 t0 t1 t2 d a]
constexpr int MH_NT = 128;

__host__ __device__ inline int zidx(int i, int j) {  // upper-triangle index of the 8x8 Z
  const int lo = i < j ? i : j, hi = i < j ? j : i;
  return lo * MH_Z - lo * (lo - 1) / 2 + (hi - lo);
}
// record layout
constexpr int R_Z = 0;       // 36
constexpr int R_ZS = 36;     // 8: sum w z
constexpr int R_WS = 44;     // 1: sum w
constexpr int R_GZ = 45;     // 8: sum w r z
constexpr int R_GR = 53;     // 1: sum w r

struct MhDev {
  int K, N, P, Q, nF;
  int64_t NO;
  const FrameD* frames;      // K
  const int32_t* host;       // N
  const int64_t* obs_ptr;    // N+1
  const int32_t* obs_frame;  // NO
  const int32_t* obs_point;  // NO
  const double2* tnorm;      // N*P host-normalized template rays
  const double* tval;        // N*P
};

__device__ __forceinline__ void relative_pose(const PoseD& Tt, const PoseD& Th, PoseD& r) {
  // R_th = R_t R_h^T, t_th = t_t - R_th t_h
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.R[3 * i + j] = Tt.R[3 * i] * Th.R[3 * j] + Tt.R[3 * i + 1] * Th.R[3 * j + 1] + Tt.R[3 * i + 2] * Th.R[3 * j + 2];
  for (int i = 0; i < 3; ++i)
    r.t[i] = Tt.t[i] - (r.R[3 * i] * Th.t[0] + r.R[3 * i + 1] * Th.t[1] + r.R[3 * i + 2] * Th.t[2]);
}

// anchor reprojection (max_reprojection_update_px, solver.cpp:105-131): false = degenerate
__device__ __forceinline__ bool anchor_px(const PoseD& T, const FrameD& fr, double x, double y, double d, double& u,
                                          double& v) {
  double xn, yn, vx, vy, vz;
  if (!warp_point(T, x, y, d, xn, yn, vx, vy, vz)) return false;
  u = fr.fx * xn + fr.cx;
  v = fr.fy * yn + fr.cy;
  return true;
}

// per observation: residuals at (pose, a, b, d); optional record; energy/counts/max update
__global__ void __launch_bounds__(MH_NT) k_mh_obs(const MhDev m, const PoseD* __restrict__ pose,
                                                  const double* __restrict__ a, const double* __restrict__ b,
                                                  const double* __restrict__ d, double gamma, int build,
                                                  double* __restrict__ rec, const PoseD* __restrict__ pose_old,
                                                  const double* __restrict__ d_old, double4* __restrict__ stat) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= m.NO) return;
  const int n = m.obs_point[q], t = m.obs_frame[q], h = m.host[n];
  PoseD T;
  relative_pose(pose[t], pose[h], T);
  const FrameD fr = m.frames[t];
  const double alpha = exp(a[t] - a[h]), bh = b[h], bt = b[t];
  const double dv = d[n];
  double acc[MH_REC];
  if (build)
    for (int i = 0; i < MH_REC; ++i) acc[i] = 0.0;
  double energy = 0.0, nact = 0.0, noob = 0.0;
  for (int k = 0; k < m.P; ++k) {
    const double2 xk = m.tnorm[static_cast<int64_t>(n) * m.P + k];
    double xn, yn, vx, vy, vz;
    if (!warp_point(T, xk.x, xk.y, dv, xn, yn, vx, vy, vz)) {
      noob += 1.0;
      continue;
    }
    const double u = fr.fx * xn + fr.cx, v = fr.fy * yn + fr.cy;
    if (!in_margin(u, v, fr.W, fr.H)) {
      noob += 1.0;
      continue;
    }
    const double tv = m.tval[static_cast<int64_t>(n) * m.P + k];
    double gdu = 0.0, gdv = 0.0;
    const double I = bilinear_grad<true>(fr.img, fr.W, u, v, gdu, gdv);
    const double r = alpha * (tv - bh) + bt - I;
    energy += huber_loss(r, gamma);
    nact += 1.0;
    if (!build) continue;
    // FC row at the relative pose (fc_warp_jacobian geometry.cpp:129-139, solver.cpp:706-709)
    const double gx = gdu * fr.fx, gy = gdv * fr.fy;
    const double Rx0 = T.R[0] * xk.x + T.R[1] * xk.y + T.R[2];
    const double Rx1 = T.R[3] * xk.x + T.R[4] * xk.y + T.R[5];
    const double Rx2 = T.R[6] * xk.x + T.R[7] * xk.y + T.R[8];
    const double iz = 1.0 / vz;
    const double P02 = -vx * iz * iz, P12 = -vy * iz * iz;
    double z[MH_Z];
    z[0] = -(gx * (P02 * Rx1) + gy * (iz * -Rx2 + P12 * Rx1));
    z[1] = -(gx * (iz * Rx2 + P02 * -Rx0) + gy * (P12 * -Rx0));
    z[2] = -(gx * (iz * -Rx1) + gy * (iz * Rx0));
    z[3] = -(gx * (iz * dv));
    z[4] = -(gy * (iz * dv));
    z[5] = -(gx * (P02 * dv) + gy * (P12 * dv));
    z[6] = -(gx * (iz * T.t[0] + P02 * T.t[2]) + gy * (iz * T.t[1] + P12 * T.t[2]));
    z[7] = alpha * (tv - bh);  // d r / d a_t
    const double w = huber_weight(r, gamma);
    const double wr = w * r;
    for (int i = 0; i < MH_Z; ++i) {
      const double wi = w * z[i];
      for (int j = i; j < MH_Z; ++j) acc[R_Z + zidx(i, j)] += wi * z[j];
      acc[R_ZS + i] += wi;
      acc[R_GZ + i] += z[i] * wr;
    }
    acc[R_WS] += w;
    acc[R_GR] += wr;
  }
  if (build)
    for (int i = 0; i < MH_REC; ++i) rec[q * MH_REC + i] = acc[i];
  double mu = 0.0;
  if (pose_old) {  // anchor (pattern pixel 0) displacement between the old and the evaluated parameters
    PoseD To;
    relative_pose(pose_old[t], pose_old[h], To);
    const double2 x0 = m.tnorm[static_cast<int64_t>(n) * m.P];
    double u0, v0, u1, v1;
    const bool ok0 = anchor_px(To, fr, x0.x, x0.y, d_old[n], u0, v0);
    const bool ok1 = anchor_px(T, fr, x0.x, x0.y, dv, u1, v1);
    mu = (ok0 && ok1) ? sqrt((u0 - u1) * (u0 - u1) + (v0 - v1) * (v0 - v1)) : INFINITY;
  }
  stat[q] = make_double4(energy, nact, noob, mu);
}

// fixed-order block partials of the per-observation statistics: {sum e, sum nact, sum noob, max mu}
__global__ void k_mh_stat_partials(int64_t NO, const double4* __restrict__ stat, double4* __restrict__ part) {
  __shared__ double4 sh[MH_NT];
  double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < NO;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double4 s = stat[q];
    acc.x += s.x;
    acc.y += s.y;
    acc.z += s.z;
    acc.w = fmax(acc.w, s.w);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double4 v = sh[0];
    for (int i = 1; i < static_cast<int>(blockDim.x); ++i) {
      v.x += sh[i].x;
      v.y += sh[i].y;
      v.z += sh[i].z;
      v.w = fmax(v.w, sh[i].w);
    }
    part[blockIdx.x] = v;
  }
}

// Chain of a pair (h, t): J_abs = ztilde T with ztilde = [z_w(3) z_t(3) j_a 1 J_d] and
//   frame t:  [z_w + z_t [u]x, z_t, j_a, 1]    frame h: [-(z_w + z_t [u]x) R, -z_t R, -j_a, -alpha]
// col_of(): the coefficients of J_abs column c (c < Q: frame t, Q <= c < 2Q: frame h) on the 9
// components of ztilde.
struct PairMap {
  double C[16][9];  // up to 2Q = 16 absolute columns
  int Q;
};

__device__ void pair_map(const PoseD& Tt, const PoseD& Th, double alpha, int Q, PairMap& pm) {
  PoseD T;
  relative_pose(Tt, Th, T);
  double u[3];
  for (int i = 0; i < 3; ++i) u[i] = T.R[3 * i] * Th.t[0] + T.R[3 * i + 1] * Th.t[1] + T.R[3 * i + 2] * Th.t[2];
  const double S[9] = {0, -u[2], u[1], u[2], 0, -u[0], -u[1], u[0], 0};  // [u]x row-major
  pm.Q = Q;
  for (int c = 0; c < 16; ++c)
    for (int e = 0; e < 9; ++e) pm.C[c][e] = 0.0;
  // frame t rotation column j: z_w[j] + sum_i z_t[i] S[i][j]
  double A[6][3];  // rows: ztilde components 0..5, cols: the 3 rotation columns of frame t
  for (int j = 0; j < 3; ++j) {
    for (int e = 0; e < 3; ++e) A[e][j] = (e == j) ? 1.0 : 0.0;
    for (int i = 0; i < 3; ++i) A[3 + i][j] = S[3 * i + j];
  }
  for (int j = 0; j < 3; ++j) {
    for (int e = 0; e < 6; ++e) pm.C[j][e] = A[e][j];
    pm.C[3 + j][3 + j] = 1.0;
  }
  if (Q == 8) {
    pm.C[6][6] = 1.0;  // j_a
    pm.C[7][7] = 1.0;  // 1
  }
  // frame h: rotation column j = -sum_i (rot col i of t) R[i][j]; translation col j = -sum_i z_t[i] R[i][j]
  for (int j = 0; j < 3; ++j)
    for (int e = 0; e < 6; ++e) {
      double vr = 0.0, vt = 0.0;
      for (int i = 0; i < 3; ++i) {
        vr += pm.C[i][e] * T.R[3 * i + j];
        vt += pm.C[3 + i][e] * T.R[3 * i + j];
      }
      pm.C[Q + j][e] = -vr;
      pm.C[Q + 3 + j][e] = -vt;
    }
  if (Q == 8) {
    pm.C[Q + 6][6] = -1.0;
    pm.C[Q + 7][7] = -alpha;
  }
}

// ztilde moments of a record: M9 (9x9 sum w zt zt^T), gt (9: sum w r zt), with zt = [z0..z5, z7, 1, z6]
__device__ __forceinline__ void moments(const double* rc, double (&M)[9][9], double (&gt)[9]) {
  const int map[9] = {0, 1, 2, 3, 4, 5, 7, -1, 6};  // ztilde index -> z index (-1: the constant 1)
  for (int i = 0; i < 9; ++i) {
    for (int j = 0; j < 9; ++j) {
      const int a = map[i], b = map[j];
      M[i][j] = (a < 0 && b < 0) ? rc[R_WS] : (a < 0 ? rc[R_ZS + b] : (b < 0 ? rc[R_ZS + a] : rc[R_Z + zidx(a, b)]));
    }
    gt[i] = map[i] < 0 ? rc[R_GR] : rc[R_GZ + map[i]];
  }
}

// the chain matrices of every pair at the current parameters (read by k_mh_frames / k_mh_point)
__global__ void k_mh_pairmap(int npairs, int Q, const int2* __restrict__ pairs, const PoseD* __restrict__ pose,
                             const double* __restrict__ a, PairMap* __restrict__ maps) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npairs) return;
  const int h = pairs[p].x, t = pairs[p].y;
  PairMap pm;
  pair_map(pose[t], pose[h], exp(a[t] - a[h]), Q, pm);
  maps[p] = pm;
}

// per pair p = (h, t): records of its observations summed in q order, in two fixed-order levels:
// block (p, s) sums segment s of the pair's list (thread i = record entry i, coalesced 432-byte
// records), then k_mh_pair_sum adds the segments in order
constexpr int MH_SEG = 32;
__global__ void k_mh_pair_seg(const int64_t* __restrict__ pair_ptr, const int64_t* __restrict__ pair_obs,
                              const double* __restrict__ rec, double* __restrict__ seg_rec) {
  const int p = blockIdx.x, sg = blockIdx.y, i = threadIdx.x;
  const int64_t a = pair_ptr[p], len = pair_ptr[p + 1] - a;
  const int64_t j0 = a + len * sg / MH_SEG, j1 = a + len * (sg + 1) / MH_SEG;
  if (i >= MH_REC) return;
  double v = 0.0;
  for (int64_t j = j0; j < j1; ++j) v += rec[pair_obs[j] * MH_REC + i];
  seg_rec[(static_cast<int64_t>(p) * MH_SEG + sg) * MH_REC + i] = v;
}
__global__ void k_mh_pair_sum(const double* __restrict__ seg_rec, double* __restrict__ pair_rec) {
  const int p = blockIdx.x, i = threadIdx.x;
  if (i >= MH_REC) return;
  double v = 0.0;
  for (int sg = 0; sg < MH_SEG; ++sg) v += seg_rec[(static_cast<int64_t>(p) * MH_SEG + sg) * MH_REC + i];
  pair_rec[static_cast<int64_t>(p) * MH_REC + i] = v;
}

// H_FF (nF x nF, full) and g_F: one thread per (entry | gradient row), pairs in order
__global__ void k_mh_frames(const MhDev m, int npairs, const int2* __restrict__ pairs, const PairMap* __restrict__ maps,
                            const double* __restrict__ pair_rec, double* __restrict__ H, double* __restrict__ gF) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int nF = m.nF, Q = m.Q;
  const int nent = nF * nF + nF;
  if (e >= nent) return;
  const bool isg = e >= nF * nF;
  const int r = isg ? e - nF * nF : e / nF, c = isg ? -1 : e % nF;
  const int fr = r / Q + 1, cr = r % Q;
  const int fc = isg ? -1 : c / Q + 1, cc = isg ? 0 : c % Q;
  double v = 0.0;
  for (int p = 0; p < npairs; ++p) {
    const int h = pairs[p].x, t = pairs[p].y;
    // column index of frame parameter (f, comp) in the pair's absolute columns, or -1
    const int ir = fr == t ? cr : (fr == h ? Q + cr : -1);
    if (ir < 0) continue;
    const int ic = isg ? 0 : (fc == t ? cc : (fc == h ? Q + cc : -1));
    if (!isg && ic < 0) continue;
    const PairMap& pm = maps[p];
    double M[9][9], gt[9];
    moments(pair_rec + static_cast<int64_t>(p) * MH_REC, M, gt);
    if (isg) {
      double s = 0.0;
      for (int i = 0; i < 9; ++i) s += pm.C[ir][i] * gt[i];
      v += s;
    } else {
      double s = 0.0;
      for (int i = 0; i < 9; ++i) {
        if (pm.C[ir][i] == 0.0) continue;
        double row = 0.0;
        for (int j = 0; j < 9; ++j) row += M[i][j] * pm.C[ic][j];
        s += pm.C[ir][i] * row;
      }
      v += s;
    }
  }
  if (isg) gF[r] = v;
  else H[static_cast<int64_t>(r) * nF + c] = v;
}

// per point: b_n (nF, dense), D_n, g_n from its observations' records (obs order)
__global__ void k_mh_point(const MhDev m, const int32_t* __restrict__ pair_of, const PairMap* __restrict__ maps,
                           const double* __restrict__ rec, double* __restrict__ Bn, double* __restrict__ D,
                           double* __restrict__ gn) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= m.N) return;
  double* bn = Bn + static_cast<int64_t>(n) * m.nF;
  for (int i = 0; i < m.nF; ++i) bn[i] = 0.0;
  const int h = m.host[n];
  double Dn = 0.0, gd = 0.0;
  for (int64_t q = m.obs_ptr[n]; q < m.obs_ptr[n + 1]; ++q) {
    const int t = m.obs_frame[q];
    const double* rc = rec + q * MH_REC;
    const PairMap& pm = maps[pair_of[static_cast<int64_t>(h) * m.K + t]];
    double M[9][9], gt[9];
    moments(rc, M, gt);
    // b columns: sum w J_abs,c J_d = sum_i C[c][i] M[i][8]
    for (int side = 0; side < 2; ++side) {
      const int f = side == 0 ? t : h;
      if (f == 0) continue;
      for (int cc = 0; cc < m.Q; ++cc) {
        const int c = side * m.Q + cc;
        double s = 0.0;
        for (int i = 0; i < 9; ++i) s += pm.C[c][i] * M[i][8];
        bn[(f - 1) * m.Q + cc] += s;
      }
    }
    Dn += M[8][8];
    gd += gt[8];
  }
  D[n] = Dn;
  gn[n] = gd;
}

// S = H + lambda I - sum_n b_n b_n^T / (D_n + lambda) (upper computed, mirrored); rhs = -g_F + sum_n b_n g_n / (D_n + lambda).
// One block per upper entry / rhs row: thread i sums the points n = i, i + MH_NT, ... in order, then a
// fixed tree over the threads (deterministic).
__global__ void __launch_bounds__(MH_NT) k_mh_schur(int nF, int N, const double* __restrict__ H,
                                                    const double* __restrict__ gF, const double* __restrict__ Bn,
                                                    const double* __restrict__ D, const double* __restrict__ gn,
                                                    double lambda, double* __restrict__ S, double* __restrict__ rhs) {
  __shared__ double sh[MH_NT];
  const int e = blockIdx.x;
  const int nup = nF * (nF + 1) / 2;
  int r, c = -1;
  if (e < nup) {  // e -> (r, c), r <= c
    r = 0;
    int rem = e;
    while (rem >= nF - r) {
      rem -= nF - r;
      ++r;
    }
    c = r + rem;
  } else {
    r = e - nup;
  }
  double v = 0.0;
  for (int n = threadIdx.x; n < N; n += MH_NT) {
    const double br = Bn[static_cast<int64_t>(n) * nF + r];
    if (br == 0.0) continue;
    v += c >= 0 ? br * Bn[static_cast<int64_t>(n) * nF + c] / (D[n] + lambda) : br * (gn[n] / (D[n] + lambda));
  }
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = MH_NT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (c >= 0) {
      const double val = H[static_cast<int64_t>(r) * nF + c] + (r == c ? lambda : 0.0) - sh[0];
      S[static_cast<int64_t>(r) * nF + c] = val;
      S[static_cast<int64_t>(c) * nF + r] = val;
    } else {
      rhs[r] = -gF[r] + sh[0];
    }
  }
}

// dx_n = (-g_n - b_n . xp) / (D_n + lambda); candidate depth; flags {invalid, nonfinite}
__global__ void k_mh_backsub(int nF, int N, const double* __restrict__ Bn, const double* __restrict__ D,
                             const double* __restrict__ gn, const double* __restrict__ xp, double lambda,
                             const double* __restrict__ d, double* __restrict__ d_cand, int* __restrict__ flags) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double acc = -gn[n];
  for (int i = 0; i < nF; ++i) acc -= Bn[static_cast<int64_t>(n) * nF + i] * xp[i];
  const double dx = acc / (D[n] + lambda);
  const double v = d[n] + dx;
  d_cand[n] = v;
  if (v <= 0.0) atomicOr(flags, 1);
  if (!isfinite(dx)) atomicOr(flags, 2);
}

// candidate frames f >= 1: pose_boxplus (geometry.cpp:93-98) and the affine step
__global__ void k_mh_frames_update(int K, int Q, const PoseD* __restrict__ pose, const double* __restrict__ a,
                                   const double* __restrict__ b, const double* __restrict__ xp,
                                   PoseD* __restrict__ pc, double* __restrict__ ac, double* __restrict__ bc) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= K) return;
  if (f == 0) {
    pc[0] = pose[0];
    ac[0] = a[0];
    bc[0] = b[0];
    return;
  }
  const double* x = xp + (f - 1) * Q;
  const double w[3] = {x[0], x[1], x[2]};
  double dR[9];
  so3_exp(w, dR);
  PoseD o;
  mat3_mul(dR, pose[f].R, o.R);
  for (int i = 0; i < 3; ++i) o.t[i] = pose[f].t[i] + x[3 + i];
  pc[f] = o;
  ac[f] = Q == 8 ? a[f] + x[6] : a[f];
  bc[f] = Q == 8 ? b[f] + x[7] : b[f];
}

// normalize_depth_gauge (solver.cpp:135-143) with a given mean (host-reduced, fixed order)
__global__ void k_mh_gauge(int N, int K, double mean, double* __restrict__ d, PoseD* __restrict__ pose) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) d[i] /= mean;
  if (i < K)
    for (int c = 0; c < 3; ++c) pose[i].t[c] *= mean;
}

__global__ void k_mh_template(int N, int P, const int32_t* __restrict__ host, const FrameD* __restrict__ frames,
                              const double2* __restrict__ anc, PatternD pat, double2* __restrict__ tnorm,
                              double* __restrict__ tval, int* __restrict__ bad) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<int64_t>(N) * P) return;
  const int n = static_cast<int>(e / P), k = static_cast<int>(e % P);
  const FrameD fr = frames[host[n]];
  const double pu = anc[n].x + pat.dx[k], pv = anc[n].y + pat.dy[k];
  if (!in_margin(pu, pv, fr.W, fr.H)) {  // build_template (solver.cpp:40-45)
    atomicOr(bad, 1);
    tval[e] = 0.0;
    tnorm[e] = make_double2(0.0, 0.0);
    return;
  }
  tnorm[e] = make_double2((pu - fr.cx) / fr.fx, (pv - fr.cy) / fr.fy);
  tval[e] = bilinear(fr.img, fr.W, pu, pv);
}

}  // namespace

class MhEngine {
 public:
  explicit MhEngine(const pba_mh_problem* p);
  ~MhEngine() {
    if (stream_) {
      cudaStreamSynchronize(stream_);
    }
  }
  void energy(double gamma, pba_energy_result* out);
  void fc_run(const pba_config* cfg, pba_report* rep, double* a_out, double* b_out);
  cudaStream_t stream() const { return sh_.s; }
  std::string last_error;

 private:
  struct StreamHolder {
    cudaStream_t s = nullptr;
    ~StreamHolder() {
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    }
  } sh_;
  cudaStream_t stream_ = nullptr;
  int K_ = 0, N_ = 0, P_ = 0, Q_ = 6, nF_ = 0;
  int64_t NO_ = 0;
  bool template_ok_ = true;
  std::vector<int2> pairs_h_;
  DBuf<float> images_;
  DBuf<FrameD> frames_;
  DBuf<int32_t> host_, obs_frame_, obs_point_;
  DBuf<int64_t> obs_ptr_, pair_ptr_, pair_obs_;
  DBuf<int2> pairs_;
  DBuf<int32_t> pair_of_;   // K*K: pair index of (h, t)
  DBuf<PairMap> maps_;
  DBuf<double2> anchor_, tnorm_;
  DBuf<double> tval_;
  DBuf<PoseD> pose_[2], pose_cand_;
  DBuf<double> a_[2], b_[2], d_[2], a_cand_, b_cand_, d_cand_;
  DBuf<double> rec_, pair_rec_, seg_rec_, H_, gF_, Bn_, D_, gn_, S_, rhs_, X_, XT_, Dinv_, y_, xp_;
  DBuf<double4> stat_, part_;
  DBuf<int> flags_;
  DBuf<unsigned int> bar_;
  MhDev dev_{};
  int nparts_ = 0;

  struct Eval {
    double energy, nact, noob, maxupd;
  };
  Eval evaluate(double gamma, const PoseD* pose, const double* a, const double* b, const double* d, bool build,
                const PoseD* pose_old, const double* d_old);
  void build_system(const PoseD* pose, const double* a);
  bool solve(double lambda, int* flags_out);  // false: factorization failed or non-finite
  void download(int cur, pba_report* rep, double* a_out, double* b_out);
};

MhEngine::MhEngine(const pba_mh_problem* p) {
  if (!p || p->num_frames < 2 || p->num_points < 0 || p->pattern_size < 1 || p->pattern_size > 32 || !p->images ||
      !p->pose_R || !p->pose_t || (p->num_points > 0 && (!p->host || !p->anchors_px || !p->inv_depths)))
    throw PbaError(PBA_E_ARG, "bad multi-host problem");
  ck(cudaStreamCreateWithFlags(&sh_.s, cudaStreamNonBlocking), "stream");
  stream_ = sh_.s;
  set_alloc_stream(stream_);
  K_ = p->num_frames;
  N_ = p->num_points;
  P_ = p->pattern_size;
  Q_ = p->optimize_affine ? 8 : 6;
  nF_ = Q_ * (K_ - 1);
  const int W = p->images[0].width, Hh = p->images[0].height;
  for (int f = 0; f < K_; ++f)
    if (p->images[f].width != W || p->images[f].height != Hh || !p->images[f].data)
      throw PbaError(PBA_E_ARG, "multi-host frames must share one image size");
  const size_t npx = static_cast<size_t>(W) * Hh;
  images_.alloc(npx * K_);
  std::vector<FrameD> fr(K_);
  for (int f = 0; f < K_; ++f) {
    ck(cudaMemcpyAsync(images_.p + npx * f, p->images[f].data, npx * sizeof(float), cudaMemcpyHostToDevice, stream_),
       "images");
    fr[f] = FrameD{images_.p + npx * f, W, Hh, p->images[f].fx, p->images[f].fy, p->images[f].cx, p->images[f].cy};
  }
  frames_.alloc(K_);
  ck(cudaMemcpyAsync(frames_.p, fr.data(), K_ * sizeof(FrameD), cudaMemcpyHostToDevice, stream_), "frames");
  // observations: CSR by point of target frames (default: every frame but the host)
  std::vector<int64_t> optr(N_ + 1, 0);
  std::vector<int32_t> ofr, opt;
  for (int n = 0; n < N_; ++n) {
    const int h = p->host[n];
    if (h < 0 || h >= K_) throw PbaError(PBA_E_ARG, "host frame out of range");
    if (p->obs_ptr) {
      for (int64_t q = p->obs_ptr[n]; q < p->obs_ptr[n + 1]; ++q) {
        const int t = p->obs_frame[q];
        if (t < 0 || t >= K_ || t == h) throw PbaError(PBA_E_ARG, "bad multi-host observation");
        ofr.push_back(t);
        opt.push_back(n);
      }
    } else {
      for (int t = 0; t < K_; ++t)
        if (t != h) {
          ofr.push_back(t);
          opt.push_back(n);
        }
    }
    optr[n + 1] = static_cast<int64_t>(ofr.size());
  }
  NO_ = static_cast<int64_t>(ofr.size());
  // (host, target) pairs and their observation lists (q ascending)
  std::vector<std::vector<int64_t>> plist(static_cast<size_t>(K_) * K_);
  for (int64_t q = 0; q < NO_; ++q) plist[static_cast<size_t>(p->host[opt[q]]) * K_ + ofr[q]].push_back(q);
  std::vector<int64_t> pptr{0}, pobs;
  for (int h = 0; h < K_; ++h)
    for (int t = 0; t < K_; ++t) {
      const auto& L = plist[static_cast<size_t>(h) * K_ + t];
      if (L.empty()) continue;
      pairs_h_.push_back(make_int2(h, t));
      pobs.insert(pobs.end(), L.begin(), L.end());
      pptr.push_back(static_cast<int64_t>(pobs.size()));
    }
  auto up = [&](auto& buf, const auto& vec) {
    using T2 = std::remove_reference_t<decltype(*buf.p)>;
    buf.alloc(std::max<size_t>(vec.size(), 1));
    if (!vec.empty())
      ck(cudaMemcpyAsync(buf.p, vec.data(), vec.size() * sizeof(T2), cudaMemcpyHostToDevice, stream_), "upload");
  };
  up(obs_ptr_, optr);
  up(obs_frame_, ofr);
  up(obs_point_, opt);
  up(pairs_, pairs_h_);
  {
    std::vector<int32_t> pof(static_cast<size_t>(K_) * K_, -1);
    for (size_t i = 0; i < pairs_h_.size(); ++i) pof[static_cast<size_t>(pairs_h_[i].x) * K_ + pairs_h_[i].y] = static_cast<int32_t>(i);
    up(pair_of_, pof);
    maps_.alloc(std::max<size_t>(pairs_h_.size(), 1));
  }
  up(pair_ptr_, pptr);
  up(pair_obs_, pobs);
  std::vector<int32_t> host(p->host, p->host + N_);
  up(host_, host);
  std::vector<double2> anc(N_);
  for (int n = 0; n < N_; ++n) anc[n] = make_double2(p->anchors_px[2 * n], p->anchors_px[2 * n + 1]);
  up(anchor_, anc);
  // parameters
  std::vector<PoseD> poses(K_);
  for (int f = 0; f < K_; ++f) {
    for (int i = 0; i < 9; ++i) poses[f].R[i] = p->pose_R[9 * f + i];
    for (int i = 0; i < 3; ++i) poses[f].t[i] = p->pose_t[3 * f + i];
  }
  up(pose_[0], poses);
  pose_[1].alloc(K_);
  pose_cand_.alloc(K_);
  std::vector<double> av(K_, 0.0), bv(K_, 0.0), dv(p->inv_depths, p->inv_depths + N_);
  if (p->affine_a) av.assign(p->affine_a, p->affine_a + K_);
  if (p->affine_b) bv.assign(p->affine_b, p->affine_b + K_);
  up(a_[0], av);
  up(b_[0], bv);
  up(d_[0], dv);
  for (auto* bf : {&a_[1], &b_[1], &a_cand_, &b_cand_}) bf->alloc(K_);
  d_[1].alloc(std::max(N_, 1));
  d_cand_.alloc(std::max(N_, 1));
  // template (build_template in each host image)
  PatternD pat{};
  pat.P = P_;
  for (int k = 0; k < P_; ++k) {
    pat.dx[k] = p->pattern[2 * k];
    pat.dy[k] = p->pattern[2 * k + 1];
  }
  tnorm_.alloc(std::max<size_t>(static_cast<size_t>(N_) * P_, 1));
  tval_.alloc(std::max<size_t>(static_cast<size_t>(N_) * P_, 1));
  flags_.alloc(4);
  ck(cudaMemsetAsync(flags_.p, 0, 4 * sizeof(int), stream_), "flags");
  if (N_ > 0) {
    const int64_t ne = static_cast<int64_t>(N_) * P_;
    k_mh_template<<<static_cast<int>((ne + 255) / 256), 256, 0, stream_>>>(N_, P_, host_.p, frames_.p, anchor_.p, pat,
                                                                          tnorm_.p, tval_.p, flags_.p);
    count_launches(1);
  }
  int fl = 0;
  ck(cudaMemcpyAsync(&fl, flags_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_), "template flag");
  ck(cudaStreamSynchronize(stream_), "create sync");
  template_ok_ = fl == 0;
  // scratch
  const size_t nO = std::max<int64_t>(NO_, 1);
  rec_.alloc(nO * MH_REC);
  stat_.alloc(nO);
  nparts_ = static_cast<int>(std::min<int64_t>(std::max<int64_t>((NO_ + MH_NT - 1) / MH_NT, 1), 1024));
  part_.alloc(nparts_);
  pair_rec_.alloc(std::max<size_t>(pairs_h_.size(), 1) * MH_REC);
  seg_rec_.alloc(std::max<size_t>(pairs_h_.size(), 1) * MH_SEG * MH_REC);
  H_.alloc(static_cast<size_t>(nF_) * nF_);
  gF_.alloc(nF_);
  Bn_.alloc(std::max<size_t>(static_cast<size_t>(N_) * nF_, 1));
  D_.alloc(std::max(N_, 1));
  gn_.alloc(std::max(N_, 1));
  S_.alloc(static_cast<size_t>(nF_) * nF_);
  X_.alloc(static_cast<size_t>(nF_) * nF_);
  XT_.alloc(static_cast<size_t>(nF_) * nF_);
  Dinv_.alloc(static_cast<size_t>((nF_ + 31) / 32) * 32 * 32);
  rhs_.alloc(nF_);
  y_.alloc(nF_);
  xp_.alloc(nF_);
  bar_.alloc(2);
  ck(cudaMemsetAsync(bar_.p, 0, 2 * sizeof(unsigned int), stream_), "bar");
  dev_ = MhDev{K_, N_, P_, Q_, nF_, NO_, frames_.p, host_.p, obs_ptr_.p, obs_frame_.p, obs_point_.p, tnorm_.p, tval_.p};
}

MhEngine::Eval MhEngine::evaluate(double gamma, const PoseD* pose, const double* a, const double* b, const double* d,
                                  bool build, const PoseD* pose_old, const double* d_old) {
  Eval ev{0.0, 0.0, 0.0, 0.0};
  if (NO_ == 0) return ev;
  k_mh_obs<<<static_cast<int>((NO_ + MH_NT - 1) / MH_NT), MH_NT, 0, stream_>>>(dev_, pose, a, b, d, gamma, build ? 1 : 0,
                                                                             rec_.p, pose_old, d_old, stat_.p);
  k_mh_stat_partials<<<nparts_, MH_NT, 0, stream_>>>(NO_, stat_.p, part_.p);
  count_launches(2);
  std::vector<double4> parts(nparts_);
  ck(cudaMemcpyAsync(parts.data(), part_.p, nparts_ * sizeof(double4), cudaMemcpyDeviceToHost, stream_), "stats");
  ck(cudaStreamSynchronize(stream_), "stats sync");
  for (const double4& v : parts) {  // fixed order
    ev.energy += v.x;
    ev.nact += v.y;
    ev.noob += v.z;
    ev.maxupd = std::max(ev.maxupd, v.w);
  }
  return ev;
}

void MhEngine::build_system(const PoseD* pose, const double* a) {
  const int np = static_cast<int>(pairs_h_.size());
  if (np > 0) {
    k_mh_pair_seg<<<dim3(np, MH_SEG), 64, 0, stream_>>>(pair_ptr_.p, pair_obs_.p, rec_.p, seg_rec_.p);
    k_mh_pair_sum<<<np, 64, 0, stream_>>>(seg_rec_.p, pair_rec_.p);
    count_launches(2);
  }
  const int nent = nF_ * nF_ + nF_;
  if (np > 0) {
    k_mh_pairmap<<<(np + 63) / 64, 64, 0, stream_>>>(np, Q_, pairs_.p, pose, a, maps_.p);
    count_launches(1);
  }
  k_mh_frames<<<(nent + 127) / 128, 128, 0, stream_>>>(dev_, np, pairs_.p, maps_.p, pair_rec_.p, H_.p, gF_.p);
  count_launches(1);
  if (N_ > 0) {
    k_mh_point<<<(N_ + 127) / 128, 128, 0, stream_>>>(dev_, pair_of_.p, maps_.p, rec_.p, Bn_.p, D_.p, gn_.p);
    count_launches(1);
  }
}

bool MhEngine::solve(double lambda, int* flags_out) {
  const int nent = nF_ * (nF_ + 1) / 2 + nF_;
  k_mh_schur<<<nent, MH_NT, 0, stream_>>>(nF_, N_, H_.p, gF_.p, Bn_.p, D_.p, gn_.p, lambda, S_.p, rhs_.p);
  count_launches(1);
  ck(cudaMemsetAsync(flags_.p, 0, 4 * sizeof(int), stream_), "flags");
  launch_chol_inv(S_.p, nF_, Dinv_.p, X_.p, XT_.p, flags_.p, bar_.p, stream_);
  launch_trisolve(X_.p, XT_.p, nF_, rhs_.p, y_.p, xp_.p, flags_.p + 1, stream_);
  int fl[4];
  ck(cudaMemcpyAsync(fl, flags_.p, sizeof(fl), cudaMemcpyDeviceToHost, stream_), "flags");
  ck(cudaStreamSynchronize(stream_), "solve sync");
  if (flags_out) std::memcpy(flags_out, fl, sizeof(fl));
  return fl[0] == 0 && fl[1] == 0;
}

void MhEngine::energy(double gamma, pba_energy_result* out) {
  if (!template_ok_) throw PbaError(PBA_E_OUT_OF_BOUNDS, "template patch pixel outside its host image");
  const Eval ev = evaluate(gamma, pose_[0].p, a_[0].p, b_[0].p, d_[0].p, false, nullptr, nullptr);
  if (ev.nact == 0) throw PbaError(PBA_E_EMPTY_PROBLEM, "no in-bounds residuals");
  if (out) {
    out->energy = ev.energy;
    out->num_active = static_cast<int64_t>(ev.nact);
    out->num_out_of_bounds = static_cast<int64_t>(ev.noob);
  }
}

void MhEngine::download(int cur, pba_report* rep, double* a_out, double* b_out) {
  std::vector<PoseD> poses(K_);
  ck(cudaMemcpy(poses.data(), pose_[cur].p, K_ * sizeof(PoseD), cudaMemcpyDeviceToHost), "poses");
  if (rep && rep->final_R && rep->final_t)
    for (int f = 0; f < K_; ++f) {
      std::memcpy(rep->final_R + 9 * f, poses[f].R, 9 * sizeof(double));
      std::memcpy(rep->final_t + 3 * f, poses[f].t, 3 * sizeof(double));
    }
  if (rep && rep->final_inv_depths && N_ > 0)
    ck(cudaMemcpy(rep->final_inv_depths, d_[cur].p, N_ * sizeof(double), cudaMemcpyDeviceToHost), "depths");
  if (a_out) ck(cudaMemcpy(a_out, a_[cur].p, K_ * sizeof(double), cudaMemcpyDeviceToHost), "a");
  if (b_out) ck(cudaMemcpy(b_out, b_[cur].p, K_ * sizeof(double), cudaMemcpyDeviceToHost), "b");
}

// FcSolver::run (solver.cpp:663-843) on the joint window; see oracle/multihost.cpp mh_fc_solve
void MhEngine::fc_run(const pba_config* cfg_in, pba_report* rep, double* a_out, double* b_out) {
  pba_config cfg;
  if (cfg_in) cfg = *cfg_in;
  else pba_config_default(&cfg);
  if (!template_ok_) throw PbaError(PBA_E_OUT_OF_BOUNDS, "template patch pixel outside its host image");
  const auto t_start = std::chrono::steady_clock::now();
  int cur = 0;
  Eval pass = evaluate(cfg.gamma, pose_[cur].p, a_[cur].p, b_[cur].p, d_[cur].p, true, nullptr, nullptr);
  if (pass.nact == 0) throw PbaError(PBA_E_EMPTY_PROBLEM, "no in-bounds residuals");  // :675
  const double initial_active = pass.nact;
  double energy = pass.energy, lambda = cfg.lambda0;
  double wall_ms = ms_since(t_start);
  int bad = 0, builds = 0, factorizations = 0, rejected = 0, iterations = 0;
  bool converged = false, diverged = false;
  std::string message;
  std::vector<pba_iter_stats> iters;
  std::vector<std::vector<double>> snapR, snapT, snapD;
  auto record = [&](int iter, double e, double mu, double nact, bool acc, int src) {
    pba_iter_stats s{};
    s.iter = iter;
    s.energy = e;
    s.max_update_px = mu;
    s.wall_ms = wall_ms;
    s.hessian_builds = builds;
    s.hessian_factorizations = factorizations;
    s.num_active = static_cast<int64_t>(nact);
    s.accepted = acc ? 1 : 0;
    iters.push_back(s);
    iterations = iter;
    if (cfg.record_snapshots) {
      std::vector<PoseD> poses(K_);
      ck(cudaMemcpy(poses.data(), pose_[src].p, K_ * sizeof(PoseD), cudaMemcpyDeviceToHost), "snap");
      std::vector<double> R(9 * K_), t(3 * K_), d(N_);
      for (int f = 0; f < K_; ++f) {
        std::memcpy(&R[9 * f], poses[f].R, 9 * sizeof(double));
        std::memcpy(&t[3 * f], poses[f].t, 3 * sizeof(double));
      }
      if (N_ > 0) ck(cudaMemcpy(d.data(), d_[src].p, N_ * sizeof(double), cudaMemcpyDeviceToHost), "snap d");
      snapR.push_back(R);
      snapT.push_back(t);
      snapD.push_back(d);
    }
  };
  for (int iter = 1; iter <= cfg.max_iters; ++iter) {
    const auto t_iter = std::chrono::steady_clock::now();
    build_system(pose_[cur].p, a_[cur].p);  // the records of the current pass (:688-724)
    ++builds;
    std::vector<double> gF(nF_);
    if (nF_ > 0) ck(cudaMemcpy(gF.data(), gF_.p, nF_ * sizeof(double), cudaMemcpyDeviceToHost), "gF");
    std::vector<double> gn(N_);
    if (N_ > 0) ck(cudaMemcpy(gn.data(), gn_.p, N_ * sizeof(double), cudaMemcpyDeviceToHost), "gn");
    bool zero_grad = true;
    for (double v : gF)
      if (v != 0.0) zero_grad = false;
    for (double v : gn)
      if (v != 0.0) zero_grad = false;
    bool accepted = false;
    Eval cand{};
    const int nxt = 1 - cur;
    while (!accepted) {
      ++factorizations;  // :732-740
      int fl[4];
      if (!solve(lambda, fl)) {
        lambda *= 10.0;
        ++rejected;
        if (++bad >= cfg.max_bad_steps) break;
        continue;
      }
      k_mh_frames_update<<<(K_ + 127) / 128, 128, 0, stream_>>>(K_, Q_, pose_[cur].p, a_[cur].p, b_[cur].p, xp_.p,
                                                                pose_cand_.p, a_cand_.p, b_cand_.p);
      ck(cudaMemsetAsync(flags_.p, 0, sizeof(int), stream_), "flags");
      if (N_ > 0)
        k_mh_backsub<<<(N_ + 127) / 128, 128, 0, stream_>>>(nF_, N_, Bn_.p, D_.p, gn_.p, xp_.p, lambda, d_[cur].p,
                                                           d_cand_.p, flags_.p);
      count_launches(2);
      int bf = 0;
      ck(cudaMemcpyAsync(&bf, flags_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_), "bs flags");
      ck(cudaStreamSynchronize(stream_), "bs sync");
      if (bf & 2) {  // non-finite depth solution (:195-211)
        lambda *= 10.0;
        ++rejected;
        if (++bad >= cfg.max_bad_steps) break;
        continue;
      }
      bool valid = !(bf & 1);
      if (valid) {
        // normalize_depth_gauge of the candidate before it is evaluated (:807-809; residuals, energy
        // and the reprojection update are gauge-invariant), so the records of an accepted candidate
        // are the next system's
        if (cfg.normalize_depth_gauge && N_ > 0) {
          std::vector<double> d(N_);
          ck(cudaMemcpy(d.data(), d_cand_.p, N_ * sizeof(double), cudaMemcpyDeviceToHost), "gauge");
          double mean = 0.0;
          for (double v : d) mean += v;
          mean /= static_cast<double>(N_);
          if (mean > 0.0 && std::isfinite(mean)) {
            k_mh_gauge<<<(std::max(N_, K_) + 127) / 128, 128, 0, stream_>>>(N_, K_, mean, d_cand_.p, pose_cand_.p);
            count_launches(1);
          }
        }
        // the candidate residuals (+ the next system's records) and the max update vs the current
        cand = evaluate(cfg.gamma, pose_cand_.p, a_cand_.p, b_cand_.p, d_cand_.p, true, pose_[cur].p, d_[cur].p);
        valid = cand.nact > 0;
      }
      if (valid && cand.energy <= energy * (1.0 + 1e-12) + 1e-15) {  // :756-759
        accepted = true;
        bad = 0;
        lambda = std::max(lambda / 10.0, cfg.lambda0);
      } else {
        if (valid && cand.maxupd < cfg.threshold_px) {  // :764-786
          converged = true;
          message = "converged: sub-threshold step rejected";
          wall_ms += ms_since(t_iter);
          record(iter, energy, cand.maxupd, pass.nact, false, cur);
          break;
        }
        lambda *= 10.0;
        ++rejected;
        if (++bad >= cfg.max_bad_steps) break;
      }
    }
    if (!accepted) {  // :792-798
      if (!converged) {
        diverged = true;
        message = "Diverged: " + std::to_string(bad) + " consecutive rejected damped steps";
      }
      break;
    }
    // accept: the candidate becomes current, then the gauge (:800-809)
    ck(cudaMemcpyAsync(pose_[nxt].p, pose_cand_.p, K_ * sizeof(PoseD), cudaMemcpyDeviceToDevice, stream_), "acc");
    ck(cudaMemcpyAsync(a_[nxt].p, a_cand_.p, K_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "acc");
    ck(cudaMemcpyAsync(b_[nxt].p, b_cand_.p, K_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "acc");
    if (N_ > 0)
      ck(cudaMemcpyAsync(d_[nxt].p, d_cand_.p, N_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "acc");
    cur = nxt;
    pass = cand;
    energy = cand.energy;
    wall_ms += ms_since(t_iter);
    record(iter, energy, cand.maxupd, pass.nact, true, cur);
    if (cand.maxupd < cfg.threshold_px) {  // :826-832
      converged = true;
      if (zero_grad) message = "no-progress convergence: zero gradient";
      break;
    }
  }
  if (rep) {
    rep->converged = converged;
    rep->diverged = diverged;
    rep->iterations = iterations;
    rep->hessian_builds = builds;
    rep->hessian_factorizations = factorizations;
    rep->rejected_steps = rejected;
    rep->final_energy = energy;
    rep->total_wall_ms = wall_ms;
    rep->masked_residuals = static_cast<int64_t>(initial_active - pass.nact);
    const int n = std::min<int>(static_cast<int>(iters.size()), std::max(rep->iters_capacity, 0));
    rep->num_iters = n;
    for (int i = 0; i < n; ++i) {
      if (rep->iters) rep->iters[i] = iters[i];
      if (cfg.record_snapshots) {
        if (rep->snap_R) std::memcpy(rep->snap_R + 9 * static_cast<size_t>(K_) * i, snapR[i].data(), 9 * K_ * sizeof(double));
        if (rep->snap_t) std::memcpy(rep->snap_t + 3 * static_cast<size_t>(K_) * i, snapT[i].data(), 3 * K_ * sizeof(double));
        if (rep->snap_d && N_ > 0) std::memcpy(rep->snap_d + static_cast<size_t>(N_) * i, snapD[i].data(), N_ * sizeof(double));
      }
    }
    std::snprintf(rep->message, sizeof(rep->message), "%s", message.c_str());
  }
  download(cur, rep, a_out, b_out);
}

}  // namespace pba_b200

using pba_b200::MhEngine;
using pba_b200::PbaError;

struct pba_mh_handle {
  std::unique_ptr<MhEngine> e;
  std::string err;
};

namespace {
thread_local std::string g_mh_create_error;
template <typename Fn>
int mh_guarded(pba_mh_handle* h, Fn&& fn) {
  if (!h || !h->e) return PBA_E_ARG;
  try {
    pba_b200::set_alloc_stream(h->e->stream());
    fn(*h->e);
    return PBA_OK;
  } catch (const PbaError& ex) {
    h->err = ex.what();
    return ex.code;
  } catch (const std::exception& ex) {
    h->err = ex.what();
    return PBA_E_ARG;
  }
}
}  // namespace

extern "C" {

int pba_gpu_mh_create(const pba_mh_problem* problem, pba_mh_handle** out) {
  if (!out) return PBA_E_ARG;
  *out = nullptr;
  try {
    auto h = std::make_unique<pba_mh_handle>();
    h->e = std::make_unique<MhEngine>(problem);
    *out = h.release();
    return PBA_OK;
  } catch (const PbaError& ex) {
    g_mh_create_error = ex.what();
    return ex.code;
  } catch (const std::exception& ex) {
    g_mh_create_error = ex.what();
    return PBA_E_ARG;
  }
}

void pba_gpu_mh_destroy(pba_mh_handle* h) {
  if (h && h->e) pba_b200::set_alloc_stream(h->e->stream());
  delete h;
}

const char* pba_gpu_mh_last_error(const pba_mh_handle* h) { return h ? h->err.c_str() : g_mh_create_error.c_str(); }

int pba_gpu_mh_energy(pba_mh_handle* h, double gamma, pba_energy_result* out) {
  return mh_guarded(h, [&](MhEngine& e) { e.energy(gamma, out); });
}

int pba_gpu_mh_fc_run(pba_mh_handle* h, const pba_config* cfg, pba_report* rep, double* a_out, double* b_out) {
  return mh_guarded(h, [&](MhEngine& e) { e.fc_run(cfg, rep, a_out, b_out); });
}

}  // extern "C"
