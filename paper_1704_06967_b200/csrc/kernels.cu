// B200 (sm_100a) kernels for the per-iteration photometric bundle adjustment step.
//
// Work decomposition:
//   k_obs_lane / k_obs_lane_tab
//              frame-major fused pass, one lane per observation over its pattern pixels: warp,
//              bilinear (lerp form), Huber residual, Jacobian (IC rows rebuilt from the template
//              records / FC rows / IC build), per-frame J^T W r and J^T W J as per-lane register
//              sums reduced once per tile; tiles launched point-block major (tile_order).
//                                                       solver.cpp:63-103,306-358,450-468,688-724
//   k_obs_energy  residual / Huber only (energy_eval), TMA-staged G-lane pass.   solver.cpp:229-244
//   k_backsub  point-major depth back-substitution + candidate depth.  solver.cpp:418-428,553-560,747-750
//   k_point    point-major gather of per-observation records -> g_n, D_n, s_n.
//   k_cf       frame-major  c_f = sum_n B_nf g_n/(D_n+lambda) + max reprojection update.  solver.cpp:407-416
//   k_finalize deterministic fixed-order reduction of tile partials -> status.
//   k_schur_*  reduced camera system: chunked DMMA SYRK, 64-bit fixed point.  solver.cpp:170-189,375-392
//   k_chol_inv fused blocked Cholesky + explicit L^-1 (stands in for Eigen::LDLT, solver.cpp:190,393).
//   k_tri_gemv two GEMVs per solve with the explicit inverse.   solver.cpp:417
//   k_xreduce / k_rhs / k_gauge_from_sum  rank exchange of point-sharded runs (pba_gpu_set_exchange).
#include <algorithm>
#include <cmath>
#include <cstdio>

#include <atomic>
#include <mutex>

#include "kernels.hpp"

namespace pba_b200 {

namespace {

constexpr int NT = 256;  // threads per block for the observation / tile kernels


// ---------------------------------------------------------------------------------
// k_obs: one block per frame-major tile; G lanes per observation (G = next pow2 >= P)
// ---------------------------------------------------------------------------------
// ---- TMA (cp.async.bulk) + mbarrier helpers -------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "MBAR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// bulk L2 prefetch of [p, p + bytes) (16-byte aligned start, size rounded up to 16)
__device__ __forceinline__ void l2_prefetch(const void* p, int64_t bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + static_cast<uintptr_t>(bytes) + 15) & ~uintptr_t(15);
  for (uintptr_t a = a0; a < a1; a += 65536) {
    const uint32_t n = static_cast<uint32_t>((a1 - a) < 65536 ? (a1 - a) : 65536);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
  }
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Shared-memory staging of one block step (OPS observations).
#ifndef PBA_OBS_STAGES
#define PBA_OBS_STAGES 2
#endif
constexpr int kStages = PBA_OBS_STAGES;
constexpr int kObsStage = 260;  // observation slots per stage: OPS (<=256) + 4 alignment slack
struct StageSmem {
  double2 anc[kObsStage];
  int32_t fmp[kObsStage];
  uint32_t msk[kObsStage];
};

constexpr int NT_OBS = NT + 32;  // 8 consumer warps + 1 producer warp
constexpr size_t kEnergyStageBytes = sizeof(StageSmem);
constexpr size_t kEnergySmem = kStages * kEnergyStageBytes;

#ifndef PBA_OBS_MINB_IC
#define PBA_OBS_MINB_IC 3
#endif
// k_obs_energy: residual / Huber pass (energy_eval, solver.cpp:229-244) with the G lanes of
// an observation over its pattern pixels; a producer warp streams each step's anchors,
// point ids and mask words into shared memory with cp.async.bulk + mbarrier (kStages deep).
template <int G>
__global__ void __launch_bounds__(NT_OBS, PBA_OBS_MINB_IC) k_obs_energy(const ObsArgs a) {
  constexpr int OPS = NT / G;  // observations per block step
  const int t = a.ov.tile_order ? a.ov.tile_order[blockIdx.x] : static_cast<int>(blockIdx.x);  // launch order only
  const int f = a.ov.tile_frame[t];
  const int64_t q0 = a.ov.tile_q0[t];
  const int64_t q1 = a.ov.tile_q1[t];
  const int nsteps = static_cast<int>((q1 - q0 + OPS - 1) / OPS);
  const bool has_mask = a.mask_in != nullptr;
  __shared__ PoseD s_pe;
  __shared__ FrameD s_fr;
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ double red[NT / 32][PT_STRIDE];
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  const int P = a.pat.P;
  if (threadIdx.x == 0) {
    s_fr = a.frames[f];
    s_pe = a.pose_eval[f];
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], NT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  if (warp == NT / 32) {
    // ---------------- producer warp: TMA bulk copies, kStages steps ahead ----------------
    if (lane == 0) {
      for (int s = 0; s < nsteps; ++s) {
        const int st = s % kStages;
        const int round = s / kStages;
        if (round > 0) mbar_wait(&empty_bar[st], static_cast<uint32_t>((round - 1) & 1));
        fence_proxy_async_smem();
        unsigned char* base = dyn_smem + static_cast<size_t>(st) * kEnergyStageBytes;
        const int64_t qs = q0 + static_cast<int64_t>(s) * OPS;
        const int64_t qe = qs + OPS < q1 ? qs + OPS : q1;
        const int64_t i0 = qs & ~int64_t(3), i1 = (qe + 3) & ~int64_t(3);  // 16-byte aligned int32 windows
        const uint32_t tx = static_cast<uint32_t>((qe - qs) * sizeof(double2) + (i1 - i0) * sizeof(int32_t) *
                                                  (has_mask ? 2 : 1));
        mbar_expect_tx(&full_bar[st], tx);
        bulk_g2s(base, a.anchor_fm + qs, static_cast<uint32_t>((qe - qs) * sizeof(double2)), &full_bar[st]);
        bulk_g2s(base + sizeof(double2) * kObsStage, a.ov.fm_point + i0,
                 static_cast<uint32_t>((i1 - i0) * sizeof(int32_t)), &full_bar[st]);
        if (has_mask)
          bulk_g2s(base + (sizeof(double2) + sizeof(int32_t)) * kObsStage, a.mask_in + i0,
                   static_cast<uint32_t>((i1 - i0) * sizeof(uint32_t)), &full_bar[st]);
      }
    }
    __syncthreads();  // matches the consumers' reduction barrier
    return;
  }

  // ---------------- consumer warps ----------------
  const FrameD& fr = s_fr;
  const PoseD& pe = s_pe;
  const FrameD& rf = a.ref;
  const int k = threadIdx.x % G;
  const int j = threadIdx.x / G;
  const bool klive = k < P;
  const double gam = a.gamma;
  double energy = 0.0, nact = 0.0, noob = 0.0;
  for (int s = 0; s < nsteps; ++s) {
    const int st = s % kStages;
    mbar_wait(&full_bar[st], static_cast<uint32_t>((s / kStages) & 1));
    const unsigned char* base = dyn_smem + static_cast<size_t>(st) * kEnergyStageBytes;
    const int64_t qs = q0 + static_cast<int64_t>(s) * OPS;
    const int64_t q = qs + j;
    const bool live = q < q1;
    double2 an = make_double2(0.0, 0.0);
    uint32_t mbits = 0u;
    int n = 0;
    if (live) {
      const int ioff = static_cast<int>(qs & 3);  // skew of the aligned int32 window
      an = reinterpret_cast<const double2*>(base)[j];
      n = reinterpret_cast<const int32_t*>(base + sizeof(double2) * kObsStage)[j + ioff];
      mbits = has_mask ? reinterpret_cast<const uint32_t*>(base + (sizeof(double2) + sizeof(int32_t)) * kObsStage)[j + ioff]
                       : 0xffffffffu;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[st]);  // stage data now lives in registers
    bool act = false;
    if (live && klive && ((mbits >> k) & 1u)) {
      const double dv = __ldg(&a.d_eval[n]);
      // template pixel (solver.cpp:42-49)
      const double pu = an.x + static_cast<double>(a.pat.dx[k]);
      const double pv = an.y + static_cast<double>(a.pat.dy[k]);
      const double x = (pu - rf.cx) * a.ref_ifx;
      const double y = (pv - rf.cy) * a.ref_ify;
      double xn, yn, vx, vy, vz;
      if (!warp_point(pe, x, y, dv, xn, yn, vx, vy, vz)) {
        noob += 1.0;
      } else {
        const double u = fr.fx * xn + fr.cx;
        const double v = fr.fy * yn + fr.cy;
        if (!in_margin(u, v, fr.W, fr.H)) {
          noob += 1.0;
        } else {
          const double r = __ldg(&a.tval[static_cast<int64_t>(n) * P + k]) - bilinear(fr.img, fr.W, u, v);
          act = true;
          energy += huber_loss(r, gam);
          ++nact;
          if (a.r_out) a.r_out[q * P + k] = r;
        }
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (live && k == 0) a.active_out[q] = (G == 32) ? bal : ((bal >> ((lane / G) * G)) & ((1u << G) - 1u));
  }
  // ---- deterministic block reduction ----
  auto put = [&](int slot, double v) {
    v = warp_sum(v);
    if (lane == 0) red[warp][slot] = v;
  };
  put(PT_E, energy);
  put(PT_NACT, static_cast<double>(nact));
  put(PT_NOOB, static_cast<double>(noob));
  __syncthreads();
  if (warp == 0 && lane < PT_STRIDE) {
    double v = 0.0;
    if (lane >= PT_E && lane < PT_MAXUPD)
      for (int w = 0; w < NT / 32; ++w) v += red[w][lane];
    a.partial[static_cast<int64_t>(t) * PT_STRIDE + lane] = v;
  }
}

template <int G>
void launch_energy_g(const ObsArgs& a, cudaStream_t s) {
  static bool attr = [] {
    cudaFuncSetAttribute(k_obs_energy<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kEnergySmem));
    return true;
  }();
  (void)attr;
  k_obs_energy<G><<<a.ov.ntiles, NT_OBS, kEnergySmem, s>>>(a);
}

void launch_energy(const ObsArgs& a, int G, cudaStream_t s) {
  switch (G) {
    case 1: launch_energy_g<1>(a, s); break;
    case 2: launch_energy_g<2>(a, s); break;
    case 4: launch_energy_g<4>(a, s); break;
    case 8: launch_energy_g<8>(a, s); break;
    case 16: launch_energy_g<16>(a, s); break;
    default: launch_energy_g<32>(a, s); break;
  }
}

// ---------------------------------------------------------------------------------
// k_obs_lane: ONE LANE PER OBSERVATION looping over the P pattern pixels; used for every
// pass that touches Jacobian rows (IC candidate pass, IC build, IC refresh, FC build).
// Per-observation sums (B_nf, D, g_n, active bits) and per-frame sums (J^T W r, J^T W J)
// live in the lane's registers: no per-pixel shuffle reductions.
//
// Factored IC Jacobian.  The IC proxy row of pixel k of observation (n, f) at p0 is
// (solver.cpp:331-349)   row = [ R0 x_k  x  m ,  d0 m ,  m . t0 ],   m = zbar0 (a - adt e_z / zbar0)
// where R0 x_k and t0 come from the frozen frame pose p0_f and the pixel ray, d0 from the
// frozen depth of the point, and m (3 doubles) carries the template gradient.  The build
// pass stores m only (24 B instead of 56 B per pixel) and every consumer rebuilds the row
// with the same fused operations (ic_row), so the rows are bitwise the rows the build used
// for H and B.  Layout: blocks of 32 frame-major observations, [block][c][k][lane]
// (coalesced for a warp of consecutive observations, written and read by lane).
// ---------------------------------------------------------------------------------
#ifndef PBA_LANE_MINB
#define PBA_LANE_MINB 2
#endif
#ifndef PBA_IC_MINB
#define PBA_IC_MINB 3
#endif

#ifndef PBA_IC_STORED_PATH
#define PBA_IC_STORED_PATH (!PBA_IC_V2)  // compile the stored-rows body too (PBA_IC_RECOMPUTE=0; the V2 pass never reads m)
#endif
#ifndef PBA_IC_FACT
#define PBA_IC_FACT 1  // IC pass: per-observation factored sums of the d0 m / m.t0 columns
#endif
#ifndef PBA_IC_OBSBASE
#define PBA_IC_OBSBASE 1  // IC pass: per-observation anchor ray and warp base
#endif
#ifndef PBA_IC_TPL_EARLY
#define PBA_IC_TPL_EARLY 1  // IC pass: template record load issued before the warp
#endif
#ifndef PBA_LANE_PREFETCH
#define PBA_LANE_PREFETCH 1
#endif
constexpr int kLanePrefetch = PBA_LANE_PREFETCH;  // block steps of L2 prefetch ahead (0 = off)

__device__ __forceinline__ int64_t jm_index(int64_t q, int c, int k, int P) {
  return ((q >> 5) * 3 + c) * (static_cast<int64_t>(P) * 32) + k * 32 + (q & 31);
}
// 16-byte shared-memory loads of the frame-uniform pose / frame records: one L1 data-pipe
// wavefront per two doubles (the pass is bounded by L1 wavefronts, half of them smem).
__device__ __forceinline__ double2 lds2(const void* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ PoseD lds_pose(const PoseD& s) {
  PoseD r;
  const char* b = reinterpret_cast<const char*>(&s);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double2 v = lds2(b + 16 * i);
    const int j = 2 * i;
    if (j < 9) r.R[j] = v.x; else r.t[j - 9] = v.x;
    if (j + 1 < 9) r.R[j + 1] = v.y; else r.t[j + 1 - 9] = v.y;
  }
  return r;
}
struct FrameL {  // register copy of the FrameD fields a pixel needs
  const float* img;
  int W, H;
  double fx, fy, cx, cy;
};
__device__ __forceinline__ FrameL tab_frame(const FrameRec& r) { return FrameL{r.img, r.W, r.H, r.fsx, r.fsy, r.cx, r.cy}; }
__device__ __forceinline__ FrameL lds_frame(const FrameD& s) {
  static_assert(sizeof(FrameD) == 48, "FrameD layout");
  const char* b = reinterpret_cast<const char*>(&s);
  const double2 v0 = lds2(b), v1 = lds2(b + 16), v2 = lds2(b + 32);
  FrameL f;
  f.img = reinterpret_cast<const float*>(__double_as_longlong(v0.x));
  const long long wh = __double_as_longlong(v0.y);
  f.W = static_cast<int>(wh & 0xffffffffll);
  f.H = static_cast<int>(wh >> 32);
  f.fx = v1.x;
  f.fy = v1.y;
  f.cx = v2.x;
  f.cy = v2.y;
  return f;
}

// one 256-bit read-only load (LDG.256) of a template record
__device__ __forceinline__ double4 ld_tpl(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// R0 x_k for the pixel ray (x, y, 1), explicit fused order shared by build and consumers
__device__ __forceinline__ void rot_ray(const PoseD& p0, double x, double y, double (&R0x)[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) R0x[i] = fma(p0.R[3 * i], x, fma(p0.R[3 * i + 1], y, p0.R[3 * i + 2]));
}
// m of the closed-form IC row (solver.cpp:331-349) from the frozen template gradient (gx, gy) of
// the pixel, its ray (x, y), the frozen frame pose p0 and the frozen depth d0.  The build and
// every consumer evaluate this same function, so the rebuilt rows are bitwise the build's rows.
// m = zbar0 a - (0, 0, a.t0) with a = R0 g3 / zbar0 and g3 = (gx, gy, -(gx x + gy y)):
// zbar0 cancels in the first term, m = R0 g3 - (0, 0, (R0 g3).t0 d0 / vz0) (one reciprocal;
// equal to the reference's order of operations up to roundoff).
__device__ __forceinline__ void ic_m(const PoseD& p0, const double (&R0x)[3], double d0, double x, double y,
                                     double gxi, double gyi, double& m0, double& m1, double& m2) {
  const double vz0 = R0x[2] + d0 * p0.t[2];
  const double g32 = -(gxi * x + gyi * y);
  const double h0 = p0.R[0] * gxi + p0.R[1] * gyi + p0.R[2] * g32;
  const double h1 = p0.R[3] * gxi + p0.R[4] * gyi + p0.R[5] * g32;
  const double h2 = p0.R[6] * gxi + p0.R[7] * gyi + p0.R[8] * g32;
  const double hdt = h0 * p0.t[0] + h1 * p0.t[1] + h2 * p0.t[2];
  m0 = h0;
  m1 = h1;
  m2 = h2 - hdt * (d0 * rcp_nr(vz0));  // |vz0| >= 1e-12 (degenerate pixels are masked at the build)
}
__device__ __forceinline__ void ic_row(const PoseD& p0, const double (&R0x)[3], double d0, double m0, double m1,
                                       double m2, double (&row)[7]);
// the frozen row of pixel k: read from the stored m (blocked layout, jm = the observation's block
// base) or, kRecompute (no store: large problems), rebuilt from the frozen template gradient
template <bool kRecompute>
__device__ __forceinline__ void ic_jrow(const PoseD& p0, const double (&R0x)[3], double d0, double x, double y,
                                        double gx, double gy, int k, const double* __restrict__ jm, int P,
                                        double (&row)[7]) {
  double m0, m1, m2;
  if (kRecompute) {
    ic_m(p0, R0x, d0, x, y, gx, gy, m0, m1, m2);
  } else {
    m0 = __ldg(jm + k * 32);
    m1 = __ldg(jm + (P + k) * 32);
    m2 = __ldg(jm + (2 * P + k) * 32);
  }
  ic_row(p0, R0x, d0, m0, m1, m2, row);
}
__device__ __forceinline__ void ic_row(const PoseD& p0, const double (&R0x)[3], double d0, double m0, double m1,
                                       double m2, double (&row)[7]) {
  row[0] = fma(R0x[1], m2, -(R0x[2] * m1));
  row[1] = fma(R0x[2], m0, -(R0x[0] * m2));
  row[2] = fma(R0x[0], m1, -(R0x[1] * m0));
  row[3] = d0 * m0;
  row[4] = d0 * m1;
  row[5] = d0 * m2;
  row[6] = fma(m0, p0.t[0], fma(m1, p0.t[1], m2 * p0.t[2]));
}

__constant__ FrameRec c_tab[kTabSlots][kTabFrames];  // the IC pass's frame records (launch_obs_ic_tab)

// kTab: the frame-uniform records (candidate pose, frozen pose, intrinsics) come from a
// kernel-parameter table (constant bank, read through the constant cache) instead of shared
// memory: the per-pixel re-reads of the pose then cost no L1 data-pipe wavefronts, which
// bound the shared-memory variant.
template <int MODE, int PT, int LPO, bool kTab, bool kRc>
__device__ __forceinline__ void obs_lane_body(const ObsArgs& a, const FrameTab& tab) {
  static_assert(LPO == 1 || (PT > 0 && PT % LPO == 0), "LPO lanes split a compile-time pattern evenly");
  constexpr int OPB = NT / LPO;  // observations per block step
  constexpr bool kH = (MODE != OBS_IC);         // builds J^T W J, B, D
  // J^T W r per frame: the IC / FC passes, and the IC build, whose rows, residuals and mask are those
  // of IcSolver::run's initial pass at the same parameters (solver.cpp:487-495): the build hands that
  // pass's gradient, energy and active count to the run (Engine::begin), which then skips it
  constexpr bool kG = (MODE == OBS_IC || MODE == OBS_FC || MODE == OBS_BUILD);
  const int tb = kTab ? tab.tile0 + static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x);
  const int t = a.ov.tile_order ? a.ov.tile_order[tb] : tb;  // launch order only: partials stay per tile
  const int f = a.ov.tile_frame[t];
  const int64_t q0 = a.ov.tile_q0[t], q1 = a.ov.tile_q1[t];
  __shared__ __align__(16) PoseD s_pe, s_p0;
  __shared__ __align__(16) FrameD s_fr;
  __shared__ double red[NT / 32][PT_STRIDE];
  // kV2 (IC pass): J^T W r accumulated in the frame-factored form.  With h = R0 g3, tau = R0^T t0,
  // s = d0 / vz0 and wq = w r (g3 . tau) s, the frozen row [R0x x m, d0 m, m . t0] of
  // m = h - e_z (h . t0) s (solver.cpp:331-349) sums over a frame's pixels to
  //   rot   = R0 sum w r (x~ x g3)  -  ((R0 sum wq x~)_y, -(R0 sum wq x~)_x, 0)
  //   trans = R0 sum d0 w r g3      -  e_z sum d0 wq
  //   g_n   = sum (w r (g3 . tau) - t0z wq)
  // (R0 (x~ x g3) = R0x~ x R0 g3): R0 is applied once per tile, a pixel needs only vz0, one
  // reciprocal and 10 FMA-class accumulations (equal to the per-pixel rows up to roundoff).
  constexpr bool kV2 = PBA_IC_V2 && MODE == OBS_IC;
  __shared__ double s_tau[4];
  if (threadIdx.x == 0) {
    s_fr = a.frames[f];
    s_pe = a.pose_eval[f];
    if (MODE != OBS_FC) s_p0 = a.pose0[f];
    if (kV2 && !kTab) {
      const PoseD& q = s_p0;
#pragma unroll
      for (int j = 0; j < 3; ++j) s_tau[j] = q.R[j] * q.t[0] + q.R[3 + j] * q.t[1] + q.R[6 + j] * q.t[2];
      s_tau[3] = q.t[2];
    }
  }
  __syncthreads();
  double v2a[kV2 ? 10 : 1];  // ac[3] = sum wr (x~ x g3), aq[3] = sum wq x~, ag[3] = sum d0 wr g3, adq = sum d0 wq
#pragma unroll
  for (int i = 0; i < (kV2 ? 10 : 1); ++i) v2a[i] = 0.0;
  const FrameD& rf = a.ref;
  const int P = PT > 0 ? PT : a.pat.P;
  const double gam = a.gamma;
  double hacc[kH ? 21 : 1], gacc[6];
#pragma unroll
  for (int i = 0; i < (kH ? 21 : 1); ++i) hacc[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) gacc[i] = 0.0;
  double energy = 0.0;
  int nact = 0, noob = 0;  // integer counters: off the FP64 pipe
  double energy_m = 0.0;   // OBS_BUILD: energy and count over the pixels that enter the sticky mask
  int nact_m = 0;
  (void)energy_m;
  (void)nact_m;
  // L2 prefetch of the streamed per-observation inputs, kLanePrefetch block steps ahead
  auto prefetch_step = [&](int64_t qs) {
    if (qs >= q1) return;
    const int64_t qe = qs + OPB < q1 ? qs + OPB : q1;
    if (threadIdx.x == 0) l2_prefetch(a.anchor_fm + qs, (qe - qs) * sizeof(double2));
    if (threadIdx.x == 32) l2_prefetch(a.ov.fm_point + qs, (qe - qs) * sizeof(int32_t));
    if (threadIdx.x == 64 && a.mask_in && (MODE == OBS_IC || MODE == OBS_REFRESH))
      l2_prefetch(a.mask_in + qs, (qe - qs) * sizeof(uint32_t));
    if (threadIdx.x == 96 && !kRc && (MODE == OBS_IC || MODE == OBS_REFRESH)) {
      const int64_t b0 = jm_index(qs, 0, 0, P), b1 = jm_index(qe - 1, 0, 0, P) - ((qe - 1) & 31) + 3 * P * 32;
      l2_prefetch(a.Jm + b0 - (qs & 31), (b1 - (b0 - (qs & 31))) * sizeof(double));
    }
  };
  // bulk L2 prefetch one block step ahead; off for the IC passes that rebuild the rows (not
  // HBM-bound: the prefetch instructions cost more than they hide there)
  constexpr bool kPf = kLanePrefetch > 0 && !((MODE == OBS_IC || MODE == OBS_REFRESH) && kRc);
  if (kPf) {
    for (int i = 0; i < kLanePrefetch; ++i) prefetch_step(q0 + static_cast<int64_t>(i) * OPB);
  }
  const int sub = LPO > 1 ? static_cast<int>(threadIdx.x % LPO) : 0;
  constexpr int KP = PT > 0 ? PT / LPO : 0;  // pixels per lane (compile time), 0 = all P
  for (int64_t base = q0; base < q1; base += OPB) {
    if (kPf) prefetch_step(base + static_cast<int64_t>(kLanePrefetch) * OPB);
    const int64_t q = base + threadIdx.x / LPO;
    const bool live = q < q1;
    const int64_t qc = live ? q : q1 - 1;  // clamped for the loads of idle lanes
    const double2 an = a.anchor_fm[qc];
    const int n = a.ov.fm_point[qc];
    const double dv = __ldg(&a.d_eval[n]);
    const double* tv = a.tval + static_cast<int64_t>(n) * P;
    const uint32_t mbits = !live ? 0u
                           : ((MODE == OBS_IC || MODE == OBS_REFRESH) && a.mask_in ? a.mask_in[q] : 0xffffffffu);
    const double d0n = (MODE == OBS_IC || MODE == OBS_REFRESH) ? __ldg(&a.d0[n]) : dv;
    const double* jm = (MODE == OBS_FC || kRc) ? nullptr : a.Jm + jm_index(qc, 0, 0, P);
    const double4* tpl = a.tgrad + static_cast<int64_t>(n) * P;  // frozen {tval, gx, gy} of the point
    double b6[6] = {0, 0, 0, 0, 0, 0};
    double dc = 0.0, gnc = 0.0;
    double gterm = 0.0;  // OBS_BUILD: the observation's g_n term of the initial pass
    (void)gterm;
    double mw[3] = {0.0, 0.0, 0.0};  // PBA_IC_FACT: sum over the observation's pixels of wr m
    (void)mw;
    uint32_t bits = 0u;
    bool obs_ok = true;
    if constexpr (MODE == OBS_BUILD) {
      const PoseD p0 = kTab ? c_tab[tab.slot][f - tab.f0].p0 : lds_pose(s_p0);
      // make_proxy_constants at the anchor (geometry.cpp:141-160): masks the whole obs
      const double xa = ((an.x + static_cast<double>(a.pat.dx[0])) - rf.cx) * a.ref_ifx;
      const double ya = ((an.y + static_cast<double>(a.pat.dy[0])) - rf.cy) * a.ref_ify;
      const double vza = p0.R[6] * xa + p0.R[7] * ya + p0.R[8] + dv * p0.t[2];
      obs_ok = (dv > 0.0) && !(vza < kDegenerateDepthEps);
    }
    // kOB (IC pass, compile-time pattern): the observation's anchor ray and the pixel-invariant
    // part of the warp, R e_z + d t, are formed once per observation; a pixel then costs one add
    // per ray coordinate and two FMAs per warp component (equal up to roundoff)
    constexpr bool kOB = PBA_IC_OBSBASE && MODE == OBS_IC && PT > 0;
    double xa = 0.0, ya = 0.0, bx = 0.0, by = 0.0, bz = 0.0, c8 = 0.0;
    if constexpr (kV2) {  // pixel-invariant part of the frozen depth vz0 = R0[6] x + R0[7] y + R0[8] + d0 t0z
      const double r8 = kTab ? c_tab[tab.slot][f - tab.f0].p0.R[8] : s_p0.R[8];
      const double t0z = kTab ? c_tab[tab.slot][f - tab.f0].t0z : s_tau[3];
      c8 = fma(d0n, t0z, r8);
    }
    if constexpr (kOB) {
      const PoseD pe = kTab ? c_tab[tab.slot][f - tab.f0].pe : lds_pose(s_pe);
      xa = (an.x - rf.cx) * a.ref_ifx;
      ya = (an.y - rf.cy) * a.ref_ify;
      bx = fma(dv, pe.t[0], pe.R[2]);
      by = fma(dv, pe.t[1], pe.R[5]);
      bz = fma(dv, pe.t[2], pe.R[8]);
    }
#pragma unroll (PT > 0 ? KP : 1)
    for (int kk = 0; kk < (PT > 0 ? KP : P); ++kk) {
      const int k = PT > 0 ? sub * KP + kk : kk;
      if (!((mbits >> k) & 1u)) continue;
      // template pixel (solver.cpp:42-49)
      double x, y;
      if constexpr (kOB) {
        x = xa + a.pat_n[k].x;
        y = ya + a.pat_n[k].y;
      } else {
        const double pu = an.x + (PT > 0 ? a.pat_d[k].x : static_cast<double>(a.pat.dx[k]));  // no I2F when unrolled
        const double pv = an.y + (PT > 0 ? a.pat_d[k].y : static_cast<double>(a.pat.dy[k]));
        x = (pu - rf.cx) * a.ref_ifx;
        y = (pv - rf.cy) * a.ref_ify;
      }
      double xn, yn, vx, vy, vz, r = 0.0;
      bool act = false;
      double4 T = make_double4(0.0, NAN, NAN, 0.0);  // template record {tval, gx, gy} (non-FC modes)
      const PoseD pe = kTab ? c_tab[tab.slot][f - tab.f0].pe : lds_pose(s_pe);
      const FrameL fr = kTab ? tab_frame(c_tab[tab.slot][f - tab.f0]) : lds_frame(s_fr);
      constexpr bool kTplEarly = PBA_IC_TPL_EARLY && MODE == OBS_IC;
      if constexpr (kTplEarly) T = ld_tpl(tpl + k);  // issued ahead of the warp: its latency overlaps it
      bool wok;
      if constexpr (kOB) {
        vx = fma(pe.R[0], x, fma(pe.R[1], y, bx));
        vy = fma(pe.R[3], x, fma(pe.R[4], y, by));
        vz = fma(pe.R[6], x, fma(pe.R[7], y, bz));
        wok = !(fabs(vz) < kDegenerateDepthEps);
        if (wok) {
          const double iz = rcp_nr(vz);
          xn = vx * iz;
          yn = vy * iz;
        }
      } else {
        wok = warp_point(pe, x, y, dv, xn, yn, vx, vy, vz);
      }
      if (!wok) {
        ++noob;
      } else {
        // scaled table (IC pass): pe rows 0/1 carry fx/fy, and fr.fx/fr.fy hold W - 3 / H - 3
        constexpr bool kSc = kTab && PBA_TAB_SCALED;
        const double u = kSc ? xn + fr.cx : fr.fx * xn + fr.cx;
        const double v = kSc ? yn + fr.cy : fr.fy * yn + fr.cy;
        const bool inm = kSc ? (u >= 1.0 && u <= fr.fx && v >= 1.0 && v <= fr.fy) : in_margin(u, v, fr.W, fr.H);
        if (!inm) {
          ++noob;
        } else {
          double gdu = 0.0, gdv = 0.0;
          if constexpr (MODE == OBS_FC) {
            r = __ldg(tv + k) - bilinear_grad<true>(fr.img, fr.W, u, v, gdu, gdv);  // + image_gradient taps
          } else {
            if constexpr (!kTplEarly) T = ld_tpl(tpl + k);
            r = T.x - bilinear(fr.img, fr.W, u, v);
          }
          act = true;
          if constexpr (MODE != OBS_BUILD) energy += huber_loss(r, gam);  // the build reports the masked energy only
          ++nact;
          if (a.r_out) a.r_out[q * P + k] = r;
          if constexpr (kV2) {
            // fresh weights (solver.cpp:461): w(r) r = r or gamma * sign(r) (no division)
            const double wr = fabs(r) <= gam ? r : copysign(gam, r);
            const double* R0 = kTab ? c_tab[tab.slot][f - tab.f0].p0.R : s_p0.R;
            const double* tau = kTab ? c_tab[tab.slot][f - tab.f0].p0.t : s_tau;
            const double t0z = kTab ? c_tab[tab.slot][f - tab.f0].t0z : s_tau[3];
            const double vz0 = fma(R0[6], x, fma(R0[7], y, c8));
            const double s0 = d0n * rcp_nr(vz0);  // |vz0| >= 1e-12: degenerate pixels are masked at the build
            const double g3z = T.w;               // -(gx x + gy y) of the template record
            const double hdt = fma(T.y, tau[0], fma(T.z, tau[1], g3z * tau[2]));
            const double wh = wr * hdt;
            const double wq = wh * s0;
            v2a[3] = fma(wq, x, v2a[3]);
            v2a[4] = fma(wq, y, v2a[4]);
            v2a[5] += wq;
            v2a[0] = fma(wr, fma(y, g3z, -T.z), v2a[0]);
            v2a[1] = fma(wr, fma(-x, g3z, T.y), v2a[1]);
            v2a[2] = fma(wr, fma(x, T.z, -(y * T.y)), v2a[2]);
            const double wd = wr * d0n;
            v2a[6] = fma(wd, T.y, v2a[6]);
            v2a[7] = fma(wd, T.z, v2a[7]);
            v2a[8] = fma(wd, g3z, v2a[8]);
            v2a[9] = fma(d0n, wq, v2a[9]);
            gnc = fma(-t0z, wq, gnc + wh);
            bits |= 1u << k;
          } else if constexpr (MODE == OBS_IC) {
            // fresh weights (solver.cpp:461): w(r) r = r or gamma * sign(r) (no division)
            const double wr = fabs(r) <= gam ? r : copysign(gam, r);
            const PoseD p0 = kTab ? c_tab[tab.slot][f - tab.f0].p0 : lds_pose(s_p0);
            double R0x[3], row[7];
            rot_ray(p0, x, y, R0x);
#if PBA_IC_FACT
            // factored: the d0 m and m.t0 columns are linear in m, so only sum wr m per
            // observation (3 FMAs) and apply d0 and t0 once per observation below
            double m0, m1, m2;
            if (kRc) {
              ic_m(p0, R0x, d0n, x, y, T.y, T.z, m0, m1, m2);
            } else {
              m0 = __ldg(jm + k * 32);
              m1 = __ldg(jm + (P + k) * 32);
              m2 = __ldg(jm + (2 * P + k) * 32);
            }
            gacc[0] += fma(R0x[1], m2, -(R0x[2] * m1)) * wr;
            gacc[1] += fma(R0x[2], m0, -(R0x[0] * m2)) * wr;
            gacc[2] += fma(R0x[0], m1, -(R0x[1] * m0)) * wr;
            mw[0] = fma(m0, wr, mw[0]);
            mw[1] = fma(m1, wr, mw[1]);
            mw[2] = fma(m2, wr, mw[2]);
            (void)row;
#else
            ic_jrow<kRc>(p0, R0x, d0n, x, y, T.y, T.z, k, jm, P, row);
#pragma unroll
            for (int c = 0; c < 6; ++c) gacc[c] += row[c] * wr;
            gnc += row[6] * wr;
#endif
            bits |= 1u << k;
          } else if constexpr (MODE == OBS_REFRESH) {
            const PoseD p0 = kTab ? c_tab[tab.slot][f - tab.f0].p0 : lds_pose(s_p0);
            double R0x[3], row[7];
            rot_ray(p0, x, y, R0x);
            ic_jrow<kRc>(p0, R0x, d0n, x, y, T.y, T.z, k, jm, P, row);
            const double w = huber_weight(r, gam);
            int h = 0;
#pragma unroll
            for (int i2 = 0; i2 < 6; ++i2) {
              const double wi = w * row[i2];
#pragma unroll
              for (int j2 = i2; j2 < 6; ++j2) hacc[h++] += wi * row[j2];
              b6[i2] += wi * row[6];
            }
            dc += w * row[6] * row[6];
            bits |= 1u << k;
          } else if constexpr (MODE == OBS_FC) {
            // image_gradient on the target at the warped point (image.cpp:36-49)
            const double gx = gdu * fr.fx, gy = gdv * fr.fy;
            // fc_warp_jacobian (geometry.cpp:129-139); row = -(grad^T J_img)
            const double Rx0 = pe.R[0] * x + pe.R[1] * y + pe.R[2];
            const double Rx1 = pe.R[3] * x + pe.R[4] * y + pe.R[5];
            const double Rx2 = pe.R[6] * x + pe.R[7] * y + pe.R[8];
            const double iz = rcp_nr(vz);  // |vz| >= 1e-12 here (warp_point); <= 1 ulp from 1 / vz
            const double P02 = -vx * iz * iz, P12 = -vy * iz * iz;
            double row[7];
            row[0] = -(gx * (P02 * Rx1) + gy * (iz * -Rx2 + P12 * Rx1));
            row[1] = -(gx * (iz * Rx2 + P02 * -Rx0) + gy * (P12 * -Rx0));
            row[2] = -(gx * (iz * -Rx1) + gy * (iz * Rx0));
            row[3] = -(gx * (iz * dv));
            row[4] = -(gy * (iz * dv));
            row[5] = -(gx * (P02 * dv) + gy * (P12 * dv));
            row[6] = -(gx * (iz * pe.t[0] + P02 * pe.t[2]) + gy * (iz * pe.t[1] + P12 * pe.t[2]));
            const double w = huber_weight(r, gam);
            const double wr = w * r;
            int h = 0;
#pragma unroll
            for (int i2 = 0; i2 < 6; ++i2) {
              const double wi = w * row[i2];
#pragma unroll
              for (int j2 = i2; j2 < 6; ++j2) hacc[h++] += wi * row[j2];
              b6[i2] += wi * row[6];
              gacc[i2] += row[i2] * wr;
            }
            dc += w * row[6] * row[6];
            gnc += row[6] * wr;
            bits |= 1u << k;
          }
        }
      }
      if constexpr (MODE == OBS_BUILD) {
        // IcSolver::build per-pixel rows (solver.cpp:306-356); evaluation point is p0
        double m0 = 0.0, m1 = 0.0, m2 = 0.0;
        if (act && obs_ok) {
          const PoseD p0 = kTab ? c_tab[tab.slot][f - tab.f0].p0 : lds_pose(s_p0);
          // template gradient image_gradient(ref, x) (image.cpp:36-49): computed once per (n, k)
          // with the template values (solver.cpp:296-304), NaN when its footprint leaves the image
          const double2 tg = make_double2(T.y, T.z);
          const bool grad_ok = !isnan(tg.x);
          double R0x[3];
          rot_ray(p0, x, y, R0x);
          const double vz0 = R0x[2] + dv * p0.t[2];
          if (grad_ok && !(vz0 < kDegenerateDepthEps)) {
            bits |= 1u << k;
            ic_m(p0, R0x, dv, x, y, tg.x, tg.y, m0, m1, m2);
            double row[7];
            ic_row(p0, R0x, dv, m0, m1, m2, row);
            const double w = huber_weight(r, gam);  // W0 (solver.cpp:279)
            int h = 0;
#pragma unroll
            for (int i2 = 0; i2 < 6; ++i2) {
              const double wi = w * row[i2];
#pragma unroll
              for (int j2 = i2; j2 < 6; ++j2) hacc[h++] += wi * row[j2];
              b6[i2] += wi * row[6];
            }
            dc += w * row[6] * row[6];
            gnc += fabs(row[6]);  // bound of the IC g_n terms: |w r| <= gamma (k_point PT_DONLY)
            // the run's initial pass (fresh weights at the same residual, solver.cpp:461): w(r) r
            const double wr = fabs(r) <= gam ? r : copysign(gam, r);
#pragma unroll
            for (int c = 0; c < 6; ++c) gacc[c] = fma(row[c], wr, gacc[c]);
            gterm = fma(row[6], wr, gterm);
            energy_m += huber_loss(r, gam);
            ++nact_m;
          }
        }
        if (a.Jmw) {  // store m unless the consumers rebuild it
          double* jw = a.Jmw + jm_index(q, 0, k, P);
          jw[0] = m0;
          jw[P * 32] = m1;
          jw[2 * P * 32] = m2;
        }
      }
    }
#if PBA_IC_FACT
    if constexpr (MODE == OBS_IC && !kV2) {  // apply the per-observation factors: [.., d0 sum wr m, t0 . sum wr m]
      const PoseD p0 = kTab ? c_tab[tab.slot][f - tab.f0].p0 : lds_pose(s_p0);
      gacc[3] = fma(d0n, mw[0], gacc[3]);
      gacc[4] = fma(d0n, mw[1], gacc[4]);
      gacc[5] = fma(d0n, mw[2], gacc[5]);
      gnc = fma(mw[0], p0.t[0], fma(mw[1], p0.t[1], mw[2] * p0.t[2]));
    }
#endif
    if constexpr (LPO > 1) {  // per-observation sums over the LPO lanes of the observation
#pragma unroll
      for (int o = 1; o < LPO; o <<= 1) {
        gnc += __shfl_xor_sync(0xffffffffu, gnc, o);
        dc += __shfl_xor_sync(0xffffffffu, dc, o);
        bits |= __shfl_xor_sync(0xffffffffu, bits, o);
        if constexpr (kH) {
#pragma unroll
          for (int i2 = 0; i2 < 6; ++i2) b6[i2] += __shfl_xor_sync(0xffffffffu, b6[i2], o);
        }
      }
    }
    if (live && sub == 0) {
      a.active_out[q] = bits;
      if (MODE == OBS_IC && a.gfix) {  // exact, order-free fixed-point sum per point (L2-resident RED)
        const double v = gnc * __ldg(a.gscale + n);
        if (fabs(v) < 0x1p62) atomicAdd(a.gfix + n, static_cast<unsigned long long>(llrint(v)));
        else *a.gfix_bad = 1;  // non-finite or beyond the bound: the engine re-runs the pass unscaled
      } else if (MODE == OBS_IC && a.rec_g) a.rec_g[q] = gnc;  // IC needs the g_n term only (D is frozen)
      else a.rec[q] = make_double2(gnc, dc);
      if (MODE == OBS_BUILD && a.rec_g) a.rec_g[q] = gterm;
      if constexpr (kH) {
#pragma unroll
        for (int i2 = 0; i2 < 6; ++i2) a.B_out[q * 6 + i2] = b6[i2];
        if (MODE == OBS_BUILD && a.Bpm_out) {  // the point-major copy k_backsub streams
          double2* dst = reinterpret_cast<double2*>(a.Bpm_out + static_cast<int64_t>(__ldg(a.fm2pm + q)) * 6);
          dst[0] = make_double2(b6[0], b6[1]);
          dst[1] = make_double2(b6[2], b6[3]);
          dst[2] = make_double2(b6[4], b6[5]);
        }
        if (a.B_dense) {  // the Schur chunk row slot of (n, f): 16-byte aligned (rows are 64-double multiples)
          double2* dst = reinterpret_cast<double2*>(a.B_dense + a.dense_row[n] + 6 * f);
          dst[0] = make_double2(b6[0], b6[1]);
          dst[1] = make_double2(b6[2], b6[3]);
          dst[2] = make_double2(b6[4], b6[5]);
        }
      }
    }
  }
  // ---- deterministic block reduction of the per-lane frame accumulators ----
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto put = [&](int slot, double v) {
    v = warp_sum(v);
    if (lane == 0) red[warp][slot] = v;
  };
  if constexpr (kV2) {  // the frame-factored sums to J^T W r of the frame (R0 is uniform over the tile)
    const double* R0 = kTab ? c_tab[tab.slot][f - tab.f0].p0.R : s_p0.R;
    double rc[3], rq[3], rg[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rc[i] = fma(R0[3 * i], v2a[0], fma(R0[3 * i + 1], v2a[1], R0[3 * i + 2] * v2a[2]));
      rq[i] = fma(R0[3 * i], v2a[3], fma(R0[3 * i + 1], v2a[4], R0[3 * i + 2] * v2a[5]));
      rg[i] = fma(R0[3 * i], v2a[6], fma(R0[3 * i + 1], v2a[7], R0[3 * i + 2] * v2a[8]));
    }
    gacc[0] = rc[0] - rq[1];
    gacc[1] = rc[1] + rq[0];
    gacc[2] = rc[2];
    gacc[3] = rg[0];
    gacc[4] = rg[1];
    gacc[5] = rg[2] - v2a[9];
  }
  if constexpr (kG) {
#pragma unroll
    for (int i = 0; i < 6; ++i) put(PT_G + i, gacc[i]);
  }
  if constexpr (kH) {
#pragma unroll
    for (int i = 0; i < 21; ++i) put(PT_H + i, hacc[i]);
  }
  put(PT_E, energy);
  put(PT_NACT, static_cast<double>(nact));
  put(PT_NOOB, static_cast<double>(noob));
  if constexpr (MODE == OBS_BUILD) {  // the initial pass's energy and active count (slots PT_MAXUPD, + 1)
    put(PT_MAXUPD, energy_m);
    put(PT_MAXUPD + 1, static_cast<double>(nact_m));
  }
  __syncthreads();
  if (warp == 0) {
    const bool used = (lane >= PT_E && lane < PT_MAXUPD) || (kG && lane < 6) || (kH && lane >= PT_H && lane < PT_H + 21) ||
                      (MODE == OBS_BUILD && lane >= PT_MAXUPD);
    double v = 0.0;
    if (used)
      for (int w = 0; w < NT / 32; ++w) v += red[w][lane];
    a.partial[static_cast<int64_t>(t) * PT_STRIDE + lane] = v;
  }
}

__device__ FrameTab g_no_tab;  // bound to the table parameter of the shared-memory variant, never read

template <int MODE, int PT, int LPO>
__global__ void __launch_bounds__(NT, MODE == OBS_IC ? PBA_IC_MINB : PBA_LANE_MINB) k_obs_lane(const ObsArgs a) {
  if (MODE == OBS_IC || MODE == OBS_REFRESH) {
    if (PBA_IC_STORED_PATH && a.Jm) obs_lane_body<MODE, PT, LPO, false, false>(a, g_no_tab);
    else obs_lane_body<MODE, PT, LPO, false, true>(a, g_no_tab);
  } else {
    obs_lane_body<MODE, PT, LPO, false, false>(a, g_no_tab);
  }
}
template <int MODE, int PT, int LPO>
__global__ void __launch_bounds__(NT, MODE == OBS_IC ? PBA_IC_MINB : PBA_LANE_MINB)
    k_obs_lane_tab(const ObsArgs a, const FrameTab tab) {
  if (PBA_IC_STORED_PATH && a.Jm) obs_lane_body<MODE, PT, LPO, true, false>(a, tab);
  else obs_lane_body<MODE, PT, LPO, true, true>(a, tab);
}

// ---------------------------------------------------------------------------------
// k_pose_update
// ---------------------------------------------------------------------------------
__global__ void k_pose_update(int ic, int F, const PoseD* __restrict__ cur, const PoseD* __restrict__ pose0,
                              const double* __restrict__ xp, PoseD* __restrict__ cand) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const PoseD pk = cur[f];
  const double w[3] = {xp[6 * f], xp[6 * f + 1], xp[6 * f + 2]};
  const double dt[3] = {xp[6 * f + 3], xp[6 * f + 4], xp[6 * f + 5]};
  double dR[9];
  so3_exp(w, dR);
  PoseD out;
  if (ic) {
    // apply_ic_update (geometry.cpp:197-209): R = R_k R0^T dR^T R0; t = t_k - R_k R0^T dt
    const PoseD p0 = pose0[f];
    double R0T[9], dRT[9], A[9], Bm[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        R0T[3 * r + c] = p0.R[3 * c + r];
        dRT[3 * r + c] = dR[3 * c + r];
      }
    mat3_mul(pk.R, R0T, A);   // R_k R0^T
    mat3_mul(A, dRT, Bm);     // (R_k R0^T) dR^T
    mat3_mul(Bm, p0.R, out.R);
    for (int r = 0; r < 3; ++r) out.t[r] = pk.t[r] - (A[3 * r] * dt[0] + A[3 * r + 1] * dt[1] + A[3 * r + 2] * dt[2]);
  } else {
    // pose_boxplus (geometry.cpp:93-98)
    mat3_mul(dR, pk.R, out.R);
    for (int r = 0; r < 3; ++r) out.t[r] = pk.t[r] + dt[r];
  }
  cand[f] = out;
}

// ---------------------------------------------------------------------------------
// Point-major reduction kernels (k_backsub, k_point).  A warp task is kPPW consecutive
// internal points; their observations [pm_ptr[n0], pm_ptr[n0 + kPPW]) are contiguous in
// point-major order, so the warp streams them flat (coalesced, kUnroll independent loads
// in flight per lane) and keeps one register accumulator per point (the segment of an
// observation is found from the kPPW - 1 inner boundaries).  Persistent grid of
// reduce_blocks(N) blocks (a fixed function of N: the per-block partials and therefore
// every reduction order are reproducible).
// ---------------------------------------------------------------------------------
constexpr int kPPW = 4;
#ifndef PBA_BS_UNROLL
#define PBA_BS_UNROLL 2
#endif
#ifndef PBA_BS_MINB
#define PBA_BS_MINB 4
#endif
#ifndef PBA_PT_UNROLL
#define PBA_PT_UNROLL 4
#endif
#ifndef PBA_PT_MINB
#define PBA_PT_MINB 4
#endif
constexpr int kBsUnroll = PBA_BS_UNROLL, kBsMinB = PBA_BS_MINB;  // k_backsub: loads in flight per lane, blocks/SM
constexpr int kPtUnroll = PBA_PT_UNROLL, kPtMinB = PBA_PT_MINB;  // k_point

struct WarpTask {
  int n0, np;              // first point, number of points (<= kPPW)
  int64_t O0, Oe;          // observation range
  int64_t b1, b2, b3;      // inner boundaries (points 1..3 start)
};

__device__ __forceinline__ WarpTask warp_task(const ObsView& ov, int task, int lane) {
  WarpTask t;
  t.n0 = task * kPPW;
  t.np = min(kPPW, ov.N - t.n0);
  const int64_t bj = ov.pm_ptr[t.n0 + min(lane, t.np)];
  t.O0 = __shfl_sync(0xffffffffu, bj, 0);
  t.b1 = __shfl_sync(0xffffffffu, bj, 1);
  t.b2 = __shfl_sync(0xffffffffu, bj, 2);
  t.b3 = __shfl_sync(0xffffffffu, bj, 3);
  t.Oe = __shfl_sync(0xffffffffu, bj, kPPW);
  return t;
}

__device__ __forceinline__ void seg_add(double (&acc)[kPPW], const WarpTask& t, int64_t o, double v) {
  const int seg = (o >= t.b1) + (o >= t.b2) + (o >= t.b3);
#pragma unroll
  for (int p = 0; p < kPPW; ++p)
    if (seg == p) acc[p] += v;
}

// lane p < kPPW receives the warp total of acc[p]
__device__ __forceinline__ double seg_reduce(double (&acc)[kPPW], int lane) {
  double mine = 0.0;
#pragma unroll
  for (int p = 0; p < kPPW; ++p) {
    const double v = warp_sum(acc[p]);
    if (lane == p) mine = v;
  }
  return mine;
}

// Block-level fixed-order reduction of NV per-thread values into partial[blockIdx.x * NV + i]
// (slot NV-1 is a max when LAST_MAX).
template <int NV, bool LAST_MAX>
__device__ __forceinline__ void block_partial(double (&v)[NV], double* __restrict__ partial) {
  __shared__ double red[NT / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double x = (LAST_MAX && i == NV - 1) ? warp_max(v[i]) : warp_sum(v[i]);
    if (lane == 0) red[warp][i] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double x = 0.0;
    for (int w = 0; w < NT / 32; ++w)
      x = (LAST_MAX && threadIdx.x == NV - 1) ? fmax(x, red[w][threadIdx.x]) : x + red[w][threadIdx.x];
    partial[blockIdx.x * NV + threadIdx.x] = x;
  }
}

// Grid ticket: returns true in the last block to finish (after every block's partial is
// visible); that block resets the counter for the next launch.
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) *ticket = 0u;
  }
  __syncthreads();
  return s_last;
}

// k_backsub: dx_n = (-g_n - sum_f B_nf . xp_f) / (D_n + lambda) and the candidate depth
// (solver.cpp:418-428, :553-560 / :747-750); the last block also forms the depth-gauge
// scale of the candidate (mean of d_cand, normalize_depth_gauge solver.cpp:135-143).
__global__ void __launch_bounds__(NT, kBsMinB) k_backsub(const BacksubArgs a) {
  extern __shared__ double s_xp[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* __restrict__ xp = a.xp;
  if (a.xp_smem) {
    for (int i = threadIdx.x; i < 6 * a.ov.F; i += NT) s_xp[i] = a.xp[i];
    __syncthreads();
    xp = s_xp;
  }
  double st[3] = {0.0, 0.0, 0.0};  // sum d_cand, #invalid, #nonfinite
  const int ntask = (a.ov.N + kPPW - 1) / kPPW;
  for (int task = blockIdx.x * (NT / 32) + warp; task < ntask; task += gridDim.x * (NT / 32)) {
    const WarpTask t = warp_task(a.ov, task, lane);
    // per-point scalars, issued before the observation stream
    const int np_ = lane < t.np ? t.n0 + lane : t.n0;
    const double Dn = a.D[np_], gn = a.g_n[np_], dc = a.d_cur[np_];
    const double d0n = a.ic ? a.d0[np_] : 0.0;
    double acc[kPPW] = {0.0, 0.0, 0.0, 0.0};
    if (a.Bpm) {  // frozen IC blocks: flat stream of the task's observations, 3 x 16 B per lane
      const int ne = static_cast<int>(t.Oe - t.O0);
      const int r1 = static_cast<int>(t.b1 - t.O0), r2 = static_cast<int>(t.b2 - t.O0),
                r3 = static_cast<int>(t.b3 - t.O0);
      const double2* __restrict__ bp = reinterpret_cast<const double2*>(a.Bpm) + 3 * t.O0;
      const int32_t* __restrict__ fp = a.ov.pm_frame + t.O0;
      for (int i0 = lane; i0 < ne; i0 += 32 * kBsUnroll) {
        double2 bv[kBsUnroll][3];
        int fr[kBsUnroll];
#pragma unroll
        for (int u = 0; u < kBsUnroll; ++u) {
          const int i = i0 + 32 * u;
          const bool ok = i < ne;
#pragma unroll
          for (int c = 0; c < 3; ++c) bv[u][c] = ok ? __ldcs(bp + 3 * i + c) : make_double2(0.0, 0.0);
          fr[u] = ok ? fp[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < kBsUnroll; ++u) {
          const int i = i0 + 32 * u;
          const double* x = xp + 6 * fr[u];
          const double v = bv[u][0].x * x[0] + bv[u][0].y * x[1] + bv[u][1].x * x[2] + bv[u][1].y * x[3] +
                           bv[u][2].x * x[4] + bv[u][2].y * x[5];
          const int seg = (i >= r1) + (i >= r2) + (i >= r3);
#pragma unroll
          for (int p = 0; p < kPPW; ++p)
            if (seg == p) acc[p] += v;
        }
      }
    } else if (a.tq) {  // FC: per-observation dots B_nf . xp_f from the frame-major k_bdot sweep
      for (int64_t o0 = t.O0 + lane; o0 < t.Oe; o0 += 32 * 4) {
        double tv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t o = o0 + 32 * u;
          tv[u] = o < t.Oe ? a.tq[a.ov.pm2fm[o]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) seg_add(acc, t, o0 + 32 * u, tv[u]);
      }
    } else {  // gather the frame-major blocks
      for (int64_t o = t.O0 + lane; o < t.Oe; o += 32) {
        const int f = a.ov.pm_frame[o];
        const double* b = a.B + static_cast<int64_t>(a.ov.pm2fm[o]) * 6;
        double dot = 0.0;
#pragma unroll
        for (int c = 0; c < 6; ++c) dot += b[c] * xp[6 * f + c];
        seg_add(acc, t, o, dot);
      }
    }
    const double sum = seg_reduce(acc, lane);
    if (lane < t.np) {
      const int n = t.n0 + lane;
      const double dx = (-gn - sum) / (Dn + a.lambda);
      const double dn = a.ic ? ((d0n - dx) / d0n) * dc : dc + dx;
      a.d_cand[n] = dn;
      if (a.dx_out) a.dx_out[n] = dx;
      st[0] += dn;
      if (dn <= 0.0) st[1] += 1.0;
      if (!isfinite(dx)) st[2] += 1.0;
    }
  }
  double v4[4] = {st[0], st[1], st[2], 0.0};
  block_partial<4, false>(v4, a.partial);
  if (!last_block(a.ticket)) return;
  if (warp == 0) {  // same fixed order as k_finalize's sum of slot 0
    double v = 0.0;
    for (int b = lane; b < gridDim.x; b += 32) v += __ldcg(a.partial + 4 * b);
    v = warp_sum(v);
    if (lane == 0) {
      if (a.gauge_sum) *a.gauge_sum = v;
      const double mean = v / static_cast<double>(a.ov.N);
      *a.gauge_scale = (a.gauge_enabled && mean > 0.0 && isfinite(mean)) ? mean : 1.0;
    }
  }
}

// k_bdot: tq[q] = B_q . xp_f over the frame-major tiles (coalesced B; xp_f frame-uniform)
__global__ void __launch_bounds__(NT) k_bdot(const ObsView ov, const double* __restrict__ B,
                                             const double* __restrict__ xp, double* __restrict__ tq) {
  const int t = blockIdx.x;
  const int f = ov.tile_frame[t];
  const int64_t q0 = ov.tile_q0[t], q1 = ov.tile_q1[t];
  double x[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) x[c] = __ldg(xp + 6 * f + c);
  const double2* __restrict__ B2 = reinterpret_cast<const double2*>(B);
  for (int64_t q = q0 + threadIdx.x; q < q1; q += NT) {
    const double2 b0 = __ldcs(B2 + 3 * q), b1 = __ldcs(B2 + 3 * q + 1), b2 = __ldcs(B2 + 3 * q + 2);
    double dot = 0.0;
    dot += b0.x * x[0];
    dot += b0.y * x[1];
    dot += b1.x * x[2];
    dot += b1.y * x[3];
    dot += b2.x * x[4];
    dot += b2.y * x[5];
    tq[q] = dot;
  }
}

// Template values tval[n*P + k] = bilinear(ref, anchor_n + offset_k) (build_template,
// solver.cpp:33-53): fixed for the whole solve, computed once per handle.
__global__ void k_template_values(int N, PatternD pat, FrameD ref, double ref_ifx, double ref_ify,
                                  const double2* __restrict__ anc, double* __restrict__ tval,
                                  double4* __restrict__ tgrad) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<int64_t>(N) * pat.P) return;
  const int n = static_cast<int>(e / pat.P), k = static_cast<int>(e % pat.P);
  const double pu = anc[n].x + static_cast<double>(pat.dx[k]);
  const double pv = anc[n].y + static_cast<double>(pat.dy[k]);
  // a template pixel outside the image is refused at build (OutOfBounds, solver.cpp:43-45): never sample it
  tval[e] = in_bounds_px(pu, pv, ref.W, ref.H) ? bilinear(ref.img, ref.W, pu, pv) : NAN;
  // template gradient at to_pixel(to_normalized(px)) (solver.cpp:296-304, image.cpp:36-49), the
  // same expressions the IC build used per pixel; NaN marks a footprint outside the image
  const double x = (pu - ref.cx) * ref_ifx, y = (pv - ref.cy) * ref_ify;
  const double gu = ref.fx * x + ref.cx, gvp = ref.fy * y + ref.cy;
  const bool ok = in_bounds_px(gu - 0.5, gvp, ref.W, ref.H) && in_bounds_px(gu + 0.5, gvp, ref.W, ref.H) &&
                  in_bounds_px(gu, gvp - 0.5, ref.W, ref.H) && in_bounds_px(gu, gvp + 0.5, ref.W, ref.H);
  double4 g = make_double4(tval[e], NAN, NAN, 0.0);  // {template value, gx, gy, g3z}: one 32-byte load
  if (ok) {
    g.y = (bilinear(ref.img, ref.W, gu + 0.5, gvp) - bilinear(ref.img, ref.W, gu - 0.5, gvp)) * ref.fx;
    g.z = (bilinear(ref.img, ref.W, gu, gvp + 0.5) - bilinear(ref.img, ref.W, gu, gvp - 0.5)) * ref.fy;
    // g3 = (gx, gy, -(gx x + gy y)) at the ray the IC pass forms (anchor ray + pattern offset)
    const double xo = (anc[n].x - ref.cx) * ref_ifx + static_cast<double>(pat.dx[k]) * ref_ifx;
    const double yo = (anc[n].y - ref.cy) * ref_ify + static_cast<double>(pat.dy[k]) * ref_ify;
    g.w = -(g.y * xo + g.z * yo);
  }
  tgrad[e] = g;
}

// Bpm[o] = B[pm2fm[o]] (point-major copy of the frozen IC pose-depth blocks): three threads per
// observation, one 16-byte move each (a warp reads ~11 whole 48-byte blocks, stores coalesced)
__global__ void k_b_to_pm(const ObsView ov, const double* __restrict__ B, double* __restrict__ Bpm) {
  const double2* __restrict__ src = reinterpret_cast<const double2*>(B);
  double2* __restrict__ dst = reinterpret_cast<double2*>(Bpm);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ov.NO * 3;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = e / 3, c = e - 3 * o;
    __stcs(dst + e, __ldcs(src + 3 * static_cast<int64_t>(ov.pm2fm[o]) + c));
  }
}

// ---------------------------------------------------------------------------------
// k_point: point-major gather of the per-observation records (flat warp tasks)
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, kPtMinB) k_point(const PointArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double g2 = 0.0;
  if (a.mode == PT_GRAD && a.gfix) {  // g_n from the IC pass's fixed-point sums (cleared for the next pass)
    for (int n = blockIdx.x * NT + threadIdx.x; n < a.ov.N; n += gridDim.x * NT) {
      const long long v = static_cast<long long>(a.gfix[n]);
      a.gfix[n] = 0ull;
      const double g = static_cast<double>(v) * (1.0 / a.gscale[n]);  // S_n is a power of two: exact inverse
      a.g_n[n] = g;
      if (a.s_n) a.s_n[n] = g / (a.D[n] + a.lambda);
      g2 += g * g;
    }
    double v2[2] = {g2, 0.0};
    block_partial<2, false>(v2, a.partial);
    return;
  }
  const int ntask = (a.ov.N + kPPW - 1) / kPPW;
  for (int task = blockIdx.x * (NT / 32) + warp; task < ntask; task += gridDim.x * (NT / 32)) {
    const WarpTask t = warp_task(a.ov, task, lane);
    const int np_ = lane < t.np ? t.n0 + lane : t.n0;
    double gs = 0.0, ds = 0.0, Dn = 0.0;
    if (a.mode == PT_GRAD || a.mode == PT_RESCALE) Dn = a.D[np_];
    if (a.mode == PT_RESCALE) gs = a.g_n[np_];
    if (a.mode == PT_GRAD && a.rec_g) {  // 8-byte g_n terms (IC)
      double ag[kPPW] = {0.0, 0.0, 0.0, 0.0};
      for (int64_t o0 = t.O0 + lane; o0 < t.Oe; o0 += 32 * kPtUnroll) {
        double rg[kPtUnroll];
#pragma unroll
        for (int u = 0; u < kPtUnroll; ++u) {
          const int64_t o = o0 + 32 * u;
          rg[u] = o < t.Oe ? a.rec_g[a.ov.pm2fm[o]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kPtUnroll; ++u) seg_add(ag, t, o0 + 32 * u, rg[u]);
      }
      gs = seg_reduce(ag, lane);
    } else if (a.mode != PT_RESCALE) {
      double ag[kPPW] = {0.0, 0.0, 0.0, 0.0}, ad[kPPW] = {0.0, 0.0, 0.0, 0.0};
      for (int64_t o0 = t.O0 + lane; o0 < t.Oe; o0 += 32 * kPtUnroll) {
        double2 rc[kPtUnroll];
#pragma unroll
        for (int u = 0; u < kPtUnroll; ++u) {
          const int64_t o = o0 + 32 * u;
          rc[u] = o < t.Oe ? a.rec[a.ov.pm2fm[o]] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kPtUnroll; ++u) {
          const int64_t o = o0 + 32 * u;
          seg_add(ag, t, o, rc[u].x);
          seg_add(ad, t, o, rc[u].y);
        }
      }
      gs = seg_reduce(ag, lane);
      ds = seg_reduce(ad, lane);
    }
    if (lane < t.np) {
      const int n = t.n0 + lane;
      double g = gs, D = Dn;
      switch (a.mode) {
        case PT_GRAD: a.g_n[n] = g; break;
        case PT_FCH: a.g_n[n] = g; a.D[n] = ds; D = ds; break;
        case PT_DONLY:
          a.D[n] = ds;
          D = ds;
          if (a.gscale) {  // S_n = 2^(59 - e) with gamma sum |Jd| < 2^e: the IC pass's sums stay below 2^60
            // (two bits of headroom over the int64 range for rounding of the factored terms; the
            // exponent is clamped so tiny bounds cannot make S_n infinite)
            const double bound = a.gbound * g;
            a.gscale[n] = (bound > 0.0 && isfinite(bound)) ? ldexp(1.0, min(a.gexp - (ilogb(bound) + 1), 1000)) : 1.0;
          }
          g = 0.0;
          break;
        default: break;  // PT_RESCALE
      }
      if (a.s_n && a.mode != PT_DONLY) a.s_n[n] = g / (D + a.lambda);
      g2 += g * g;
    }
  }
  double v2[2] = {g2, 0.0};
  block_partial<2, false>(v2, a.partial);
}

// ---------------------------------------------------------------------------------
// k_cf: c_f partial per tile (solver.cpp:407-416 Schur right-hand-side term)
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_cf(const ObsView ov, const double* __restrict__ B,
                                           const double* __restrict__ s_n, double* __restrict__ partial,
                                           const MaxUpdArgs mu) {
  const int t = ov.tile_order ? ov.tile_order[blockIdx.x] : static_cast<int>(blockIdx.x);  // launch order only
  const int64_t q0 = ov.tile_q0[t], q1 = ov.tile_q1[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool want_upd = mu.pose_cand != nullptr;
  // max_reprojection_update_px (solver.cpp:105-131): the tile's frame is uniform
  __shared__ PoseD s_po, s_pn;
  __shared__ FrameD s_fr;
  if (want_upd && threadIdx.x == 0) {
    const int f = ov.tile_frame[t];
    s_po = mu.pose_cur[f];
    s_pn = mu.pose_cand[f];
    s_fr = mu.frames[f];
  }
  __syncthreads();
  double c[6] = {0, 0, 0, 0, 0, 0};
  double mupd = 0.0;
  const double2* __restrict__ B2 = reinterpret_cast<const double2*>(B);
  for (int64_t q = q0 + threadIdx.x; q < q1; q += NT) {
    const int n = ov.fm_point[q];
    const double s = __ldg(&s_n[n]);
    const double2 b0 = __ldcs(B2 + 3 * q), b1 = __ldcs(B2 + 3 * q + 1), b2 = __ldcs(B2 + 3 * q + 2);
    c[0] += b0.x * s;
    c[1] += b0.y * s;
    c[2] += b1.x * s;
    c[3] += b1.y * s;
    c[4] += b2.x * s;
    c[5] += b2.y * s;
    if (want_upd) {
      const double2 an = __ldg(&mu.anchor[n]);
      const double xa = ((an.x + static_cast<double>(mu.dx0)) - mu.ref_cx) * mu.ref_ifx;
      const double ya = ((an.y + static_cast<double>(mu.dy0)) - mu.ref_cy) * mu.ref_ify;
      double xo, yo, xn2, yn2, t0_, t1_, t2_;
      const bool oka = warp_point(s_po, xa, ya, __ldg(&mu.d_cur[n]), xo, yo, t0_, t1_, t2_);
      const bool okb = warp_point(s_pn, xa, ya, __ldg(&mu.d_cand[n]), xn2, yn2, t0_, t1_, t2_);
      if (!oka || !okb) {
        mupd = INFINITY;
      } else {
        const double du = (s_fr.fx * xo + s_fr.cx) - (s_fr.fx * xn2 + s_fr.cx);
        const double dv = (s_fr.fy * yo + s_fr.cy) - (s_fr.fy * yn2 + s_fr.cy);
        mupd = fmax(mupd, du * du + dv * dv);  // squared: sqrt is monotone, taken once per tile
      }
    }
  }
  mupd = sqrt(mupd);
  __shared__ double red[NT / 32][7];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double v = warp_sum(c[i]);
    if (lane == 0) red[warp][i] = v;
  }
  {
    const double v = warp_max(mupd);
    if (lane == 0) red[warp][6] = v;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double v = 0.0;
    for (int w = 0; w < NT / 32; ++w) v = threadIdx.x == 6 ? fmax(v, red[w][6]) : v + red[w][threadIdx.x];
    partial[static_cast<int64_t>(t) * 8 + threadIdx.x] = v;
  }
}

// ---------------------------------------------------------------------------------
// k_finalize: blocks 0..F-1 reduce the tiles of frame f; block F the scalars.
// Fixed strided order + warp tree: bitwise reproducible for a given tiling.
// ---------------------------------------------------------------------------------
__device__ double tile_sum(const double* part, int stride, int slot, int t0, int t1, int lane, bool is_max) {
  double v = 0.0;
  for (int t = t0 + lane; t < t1; t += 32) {
    const double x = part[static_cast<int64_t>(t) * stride + slot];
    v = is_max ? fmax(v, x) : v + x;
  }
  return is_max ? warp_max(v) : warp_sum(v);
}

__global__ void __launch_bounds__(NT) k_finalize(const FinalizeArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int F = a.ov.F;
  if (blockIdx.x < F) {
    const int f = blockIdx.x;
    const int t0 = a.ov.ftile_ptr[f], t1 = a.ov.ftile_ptr[f + 1];
    __shared__ double vals[6 + 6 + 21 + 4];
    // components: 0..5 g, 6..11 cf, 12..32 H, 33 energy, 34 #active, 35 #oob, 36 max update
    for (int c = warp; c < 37; c += NT / 32) {
      double v = 0.0;
      if (c < 6) {
        v = a.partial ? tile_sum(a.partial, PT_STRIDE, PT_G + c, t0, t1, lane, false)
                      : (a.g_f_in ? a.g_f_in[6 * f + c] : 0.0);
      } else if (c < 12) {
        if (a.partial_cf) v = tile_sum(a.partial_cf, 8, c - 6, t0, t1, lane, false);
      } else if (c < 33) {
        if (a.want_h && a.partial) v = tile_sum(a.partial, PT_STRIDE, PT_H + (c - 12), t0, t1, lane, false);
      } else if (c < 36) {
        // e_slot: the energy and active count sit in other slots (the IC build's initial-pass sums; no oob count)
        if (a.partial && a.e_slot) v = c < 35 ? tile_sum(a.partial, PT_STRIDE, a.e_slot + (c - 33), t0, t1, lane, false) : 0.0;
        else if (a.partial) v = tile_sum(a.partial, PT_STRIDE, PT_E + (c - 33), t0, t1, lane, false);
      } else {
        if (a.partial_cf) v = tile_sum(a.partial_cf, 8, 6, t0, t1, lane, true);
      }
      if (lane == 0) vals[c] = v;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      const double g = vals[threadIdx.x];
      if (a.g_f) a.g_f[6 * f + threadIdx.x] = g;
      if (a.rhs) a.rhs[6 * f + threadIdx.x] = -g + vals[6 + threadIdx.x];
    }
    if (a.cf_out && threadIdx.x < 6) a.cf_out[6 * f + threadIdx.x] = vals[6 + threadIdx.x];
    if (a.want_h && a.H && threadIdx.x < 21) a.H[21 * f + threadIdx.x] = vals[12 + threadIdx.x];
    if (threadIdx.x < 4) a.fscal[4 * f + threadIdx.x] = vals[33 + threadIdx.x];
  }
  // the last block to finish reduces the per-frame scalars and the point-kernel partials
  if (!last_block(a.ticket) || !a.status) return;
  __shared__ double sc[8];
  double v = 0.0;
  if (warp < 4) {
    const bool mx = warp == 3;
    for (int f = lane; f < F; f += 32) {
      const double x = __ldcg(a.fscal + 4 * f + warp);
      v = mx ? fmax(v, x) : v + x;
    }
    v = mx ? warp_max(v) : warp_sum(v);
  } else if (warp < 7) {
    if (a.partial_bs) {
      for (int b = lane; b < a.nbs; b += 32) v += a.partial_bs[4 * b + (warp - 4)];
      v = warp_sum(v);
    }
  } else if (a.partial_pt) {
    for (int b = lane; b < a.npt; b += 32) v += a.partial_pt[2 * b];
    v = warp_sum(v);
  }
  if (lane == 0) sc[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    Status s;
    s.energy = sc[0];
    s.num_active = sc[1];
    s.num_oob = sc[2];
    s.max_upd = sc[3];
    s.sum_d = sc[4];
    s.invalid = sc[5];
    s.nonfinite = sc[6];
    s.gnorm2_n = sc[7];
    *a.status = s;
  }
}

// ---------------------------------------------------------------------------------
// k_commit (normalize_depth_gauge, solver.cpp:135-143, applied on accept)
// ---------------------------------------------------------------------------------
__global__ void k_commit(int N, int F, const double* __restrict__ d_cand, const PoseD* __restrict__ pose_cand,
                         double mean, double tscale, double* __restrict__ d_cur, PoseD* __restrict__ pose_cur) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) d_cur[i] = d_cand[i] / mean;
  if (i < F) {
    PoseD p = pose_cand[i];
    for (int r = 0; r < 3; ++r) p.t[r] = p.t[r] * tscale;
    pose_cur[i] = p;
  }
}

// ---------------------------------------------------------------------------------
// Depth gauge of the candidate (normalize_depth_gauge, solver.cpp:135-143, applied by the
// reference after acceptance at :618-620 / :807-809).  The candidate is normalized BEFORE
// it is evaluated: residuals, energy and the reprojection update are gauge-invariant, and
// the FC Jacobian/Hessian built in the same pass then sits in the normalized
// parametrization exactly like the reference's next-iteration build (:688-724).
// ---------------------------------------------------------------------------------
__global__ void k_gauge_apply(int N, int F, const double* __restrict__ scale, double* __restrict__ d,
                              PoseD* __restrict__ pose) {
  const double m = *scale;
  if (m == 1.0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) d[i] = d[i] / m;
  if (i < F)
    for (int r = 0; r < 3; ++r) pose[i].t[r] = pose[i].t[r] * m;
}

// ---------------------------------------------------------------------------------
// k_max_reproj: standalone max_reprojection_update_px over point-major obs
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_max_reproj(const ObsView ov, const FrameD* __restrict__ frames, const FrameD ref,
                                                   const double2* __restrict__ anchor, int dx0, int dy0,
                                                   const PoseD* __restrict__ pa,
                                                   const double* __restrict__ da, const PoseD* __restrict__ pb,
                                                   const double* __restrict__ db, double* __restrict__ partial) {
  double m = 0.0;
  for (int64_t o = blockIdx.x * static_cast<int64_t>(NT) + threadIdx.x; o < ov.NO;
       o += static_cast<int64_t>(gridDim.x) * NT) {
    // point of obs o: binary search in pm_ptr
    int lo = 0, hi = ov.N - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ov.pm_ptr[mid] <= o) lo = mid; else hi = mid - 1;
    }
    const int n = lo;
    const int f = ov.pm_frame[o];
    const double2 an = anchor[n];
    const double x = ((an.x + static_cast<double>(dx0)) - ref.cx) / ref.fx;
    const double y = ((an.y + static_cast<double>(dy0)) - ref.cy) / ref.fy;
    double xa, ya, xb, yb, t0, t1, t2;
    const bool oka = warp_point(pa[f], x, y, da[n], xa, ya, t0, t1, t2);
    const bool okb = warp_point(pb[f], x, y, db[n], xb, yb, t0, t1, t2);
    if (!oka || !okb) {
      m = INFINITY;
    } else {
      const FrameD fr = frames[f];
      const double du = (fr.fx * xa + fr.cx) - (fr.fx * xb + fr.cx);
      const double dv = (fr.fy * ya + fr.cy) - (fr.fy * yb + fr.cy);
      m = fmax(m, sqrt(du * du + dv * dv));
    }
  }
  __shared__ double red[NT / 32];
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < NT / 32; ++w) v = fmax(v, red[w]);
    partial[blockIdx.x] = v;
  }
}

// ---------------------------------------------------------------------------------
// Schur complement, deterministic: the update sum_n B_nf B_nf'^T / (D_n + lambda) is
// accumulated in 64-bit fixed point with per-row scale s_r = 2^30 / sqrt(H_rr).
// Because S = H_pp - B D^-1 B^T is PSD, sum_n |B_nf,i B_nf',j| / D_n <= sqrt(H_ii H_jj)
// (Cauchy-Schwarz), so the scaled sum of |terms| stays below 2^60: no overflow, integer
// atomics are associative (bitwise reproducible), and the resolution 2^-60 sqrt(H_ii H_jj)
// is finer than an fp64 accumulation of the same terms.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ int h21_index(int i, int j) {
  const int lo = i < j ? i : j, hi = i < j ? j : i;
  return lo * 6 - lo * (lo - 1) / 2 + (hi - lo);  // upper-triangle packing of k_obs
}

__global__ void k_schur_scale(int F, const double* __restrict__ H21, double* __restrict__ scale,
                              unsigned long long* __restrict__ acc, int64_t nacc, const int32_t* __restrict__ chunk_pts,
                              int npts, const double* __restrict__ D, double lambda, double* __restrict__ wsort,
                              const double* __restrict__ scale_in) {
  const int64_t e0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t e = e0; e < nacc; e += static_cast<int64_t>(gridDim.x) * blockDim.x) acc[e] = 0ull;
  for (int64_t p = e0; p < npts; p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    wsort[p] = 1.0 / (D[chunk_pts[p]] + lambda);  // Schur weight of the p-th window-sorted point
  if (e0 < 6 * F) {
    const int r = static_cast<int>(e0);
    const double h = H21[21 * (r / 6) + h21_index(r % 6, r % 6)];
    scale[r] = scale_in ? scale_in[r] : h > 0.0 ? 1073741824.0 / sqrt(h) : 1073741824.0;
  }
}

__global__ void __launch_bounds__(NT) k_schur_pts(const ObsView ov, const double* __restrict__ B,
                                                  const double* __restrict__ D, double lambda,
                                                  const double* __restrict__ scale,
                                                  unsigned long long* __restrict__ acc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = blockIdx.x * (NT / 32) + warp;
  if (n >= ov.N) return;
  const int64_t o0 = ov.pm_ptr[n], o1 = ov.pm_ptr[n + 1];
  const int kn = static_cast<int>(o1 - o0);
  const double Dn = D[n] + lambda;
  const int ld = 6 * ov.F;
  for (int a = 0; a < kn; ++a) {
    const int fa = ov.pm_frame[o0 + a];
    const double* Ba = B + static_cast<int64_t>(ov.pm2fm[o0 + a]) * 6;
    bool za = true;
    for (int c = 0; c < 6; ++c) za = za && (Ba[c] == 0.0);
    if (za) continue;  // Bf.isZero(0.0) (solver.cpp:181,384)
    const int items = (kn - a) * 36;
    for (int it = lane; it < items; it += 32) {
      const int b = a + it / 36, ij = it % 36, i = ij / 6, jj = ij % 6;
      const int fb = ov.pm_frame[o0 + b];
      const double* Bb = B + static_cast<int64_t>(ov.pm2fm[o0 + b]) * 6;
      bool zb = true;
      for (int c = 0; c < 6; ++c) zb = zb && (Bb[c] == 0.0);
      if (zb) continue;
      if (b == a && i > jj) continue;  // upper triangle only (k_schur_final mirrors)
      const int r = 6 * fa + i, c = 6 * fb + jj;
      const double v = Ba[i] * Bb[jj] / Dn;
      const long long q = llrint(v * scale[r] * scale[c]);
      atomicAdd(&acc[static_cast<int64_t>(r) * ld + c], static_cast<unsigned long long>(q));
    }
  }
}

// Chunked dense Schur update on the FP64 tensor path (DMMA, mma.sync.m8n8k4.f64).
// Points are sorted by visibility window and cut into chunks; a chunk's scaled blocks
// b_n / sqrt(D_n + lambda) form a dense [points x 6W] matrix over its frame window, and
// one CTA computes one SCH_TB x SCH_TB tile-block of its Gram matrix (upper triangle of tile-blocks),
// K-looping over the chunk's points through shared memory.  4 warps x SY_NT^2 DMMA 8x8 tiles.
// Results enter S through the same deterministic fixed-point RED as k_schur_pts.
constexpr int SCH_TB = kSchurTB;      // tile-block edge (window-local dimensions)
constexpr int SY_NT = PBA_SY_NT;      // 8x8 DMMA tiles per warp-quadrant side
constexpr int SY_QW = 8 * SY_NT;      // warp-quadrant edge
constexpr int SY_PPR = SCH_TB / 2;    // 16-byte pieces per chunk row of a tile-block

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Densify once per B (independent of D and lambda): row p of chunk c = b_n^T over the chunk's
// frame window (zero where the point does not observe a frame), LD_c = roundup(6 W_c, SCH_TB).
__global__ void __launch_bounds__(256) k_schur_densify(const ObsView ov, const double* __restrict__ B,
                                                       const int32_t* __restrict__ chunk_pts, int npts,
                                                       const int32_t* __restrict__ chunk_of,
                                                       const int4* __restrict__ chunks,
                                                       const int64_t* __restrict__ chunk_off, double* __restrict__ dense) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= npts) return;
  const int c = chunk_of[warp];
  const int4 ch = chunks[c];  // {begin, end, fmin, LD}
  const int fmin = ch.z, LD = ch.w;
  double* row = dense + chunk_off[c] + static_cast<int64_t>(warp - ch.x) * LD;
  for (int d = lane; d < LD; d += 32) row[d] = 0.0;
  __syncwarp();
  const int n = chunk_pts[warp];
  for (int64_t o = ov.pm_ptr[n] + lane; o < ov.pm_ptr[n + 1]; o += 32) {
    const int lf = ov.pm_frame[o] - fmin;
    const double* b = B + static_cast<int64_t>(ov.pm2fm[o]) * 6;
#pragma unroll
    for (int i = 0; i < 6; ++i) row[6 * lf + i] = b[i];
  }
}

// One SCH_TB x SCH_TB upper tile-block of a chunk's weighted Gram matrix  sum_p w_p a_p a_p^T  on DMMA.
// 4 warps, each an SY_QW x SY_QW quadrant (SY_NT^2 DMMA 8x8 tiles, 2 SY_NT^2 fp64 accumulators per lane); the
// K loop streams SY_KB points per stage into shared memory with cp.async (2 stages,
// zero-filled past the chunk end); the weight w_p = 1/(D_n + lambda) scales the A fragment.
#ifndef PBA_SY_KB
#define PBA_SY_KB 32
#endif
#ifndef PBA_SY_STAGES
#define PBA_SY_STAGES 2
#endif
constexpr int SY_KB = PBA_SY_KB;  // points per stage
constexpr int SY_LDS = SCH_TB + 4;  // smem row stride (doubles): = 4 mod 16 puts the 4 k-rows of a half-warp fragment load on distinct banks (2 wavefronts)
constexpr int SY_STAGES = PBA_SY_STAGES;
constexpr int SY_THREADS = 128;
constexpr size_t SY_SMEM = static_cast<size_t>(SY_STAGES) * (2 * SY_KB * SY_LDS + SY_KB) * sizeof(double);

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(SY_THREADS) k_schur_syrk(const ObsView ov, const int4* __restrict__ blocks,
                                                           const int4* __restrict__ chunks,
                                                           const int64_t* __restrict__ chunk_off,
                                                           const double* __restrict__ dense,
                                                           const double* __restrict__ wsort,
                                                           const double* __restrict__ scale,
                                                           unsigned long long* __restrict__ acc) {
  extern __shared__ __align__(16) double sy_smem[];
  // blocks[b] = {chunk id, valid columns V (unused here), 0, rb | cb << 16}
  const int4 blk = blocks[blockIdx.x];
  const int4 ch = chunks[blk.x];
  const int p0 = ch.x, p1 = ch.y, fmin = ch.z, LD = ch.w;
  const int rb = blk.w & 0xffff, cb = blk.w >> 16;
  const int r0 = rb * SCH_TB, c0 = cb * SCH_TB;
  const bool diag = rb == cb;
  const double* base = dense + chunk_off[blk.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1;
  const bool active = !(diag && wr > wc);  // strictly-lower quadrant of a diagonal block: mirrored
  double* As = sy_smem;                                   // [stage][KB][LDS]
  double* Bs = As + SY_STAGES * SY_KB * SY_LDS;           // [stage][KB][LDS]
  double* Ws = Bs + SY_STAGES * SY_KB * SY_LDS;           // [stage][KB]
  auto issue = [&](int stage, int pb) {
    double* as = As + stage * SY_KB * SY_LDS;
    double* bs = Bs + stage * SY_KB * SY_LDS;
    // KB rows x SY_PPR 16-byte pieces for each of A and B
    static_assert((2 * SY_KB * SY_PPR) % SY_THREADS == 0, "whole pieces per thread");
#pragma unroll
    for (int it = 0; it < (2 * SY_KB * SY_PPR) / SY_THREADS; ++it) {
      const int idx = tid + it * SY_THREADS;
      const int isb = idx >= SY_KB * SY_PPR;
      const int j = idx - isb * SY_KB * SY_PPR;
      const int pp = j / SY_PPR, piece = j % SY_PPR;
      const bool valid = pb + pp < p1;
      const double* src = base + static_cast<int64_t>(valid ? pb - p0 + pp : 0) * LD + (isb ? c0 : r0) + 2 * piece;
      cp_async16((isb ? bs : as) + pp * SY_LDS + 2 * piece, src, valid);
    }
    if (tid < SY_KB) cp_async8(Ws + stage * SY_KB + tid, wsort + min(pb + tid, p1 - 1), pb + tid < p1);
    cp_async_commit();
  };
  double accd[SY_NT][SY_NT][2];
#pragma unroll
  for (int i = 0; i < SY_NT; ++i)
#pragma unroll
    for (int j = 0; j < SY_NT; ++j) accd[i][j][0] = accd[i][j][1] = 0.0;
  const int nsb = (p1 - p0 + SY_KB - 1) / SY_KB;
  // SY_STAGES-deep cp.async pipeline: SY_STAGES - 1 stages in flight while one is consumed (an
  // empty commit group past the end keeps the wait count uniform)
#pragma unroll
  for (int i = 0; i < SY_STAGES - 1; ++i) {
    if (i < nsb) issue(i, p0 + i * SY_KB);
    else cp_async_commit();
  }
  for (int sb = 0; sb < nsb; ++sb) {
    const int stage = sb % SY_STAGES;
    const int nxt = sb + SY_STAGES - 1;
    if (nxt < nsb) issue(nxt % SY_STAGES, p0 + nxt * SY_KB);
    else cp_async_commit();
    cp_async_wait<SY_STAGES - 1>();
    __syncthreads();
    if (active) {
      const double* as = As + stage * SY_KB * SY_LDS + wr * SY_QW + (lane >> 2);
      const double* bs = Bs + stage * SY_KB * SY_LDS + wc * SY_QW + (lane >> 2);
      const double* ws = Ws + stage * SY_KB;
#pragma unroll
      for (int kk = 0; kk < SY_KB; kk += 4) {
        const int k = kk + (lane & 3);
        const double w = ws[k];
        double a[SY_NT], b[SY_NT];
#pragma unroll
        for (int i = 0; i < SY_NT; ++i) a[i] = as[k * SY_LDS + 8 * i] * w;
#pragma unroll
        for (int j = 0; j < SY_NT; ++j) b[j] = bs[k * SY_LDS + 8 * j];
#pragma unroll
        for (int i = 0; i < SY_NT; ++i)
#pragma unroll
          for (int j = 0; j < SY_NT; ++j)
            dmma_8x8x4(accd[i][j][0], accd[i][j][1], a[i], b[j]);
      }
    }
    __syncthreads();  // the stage is overwritten by the next issue
  }
  if (!active) return;
  // fold into the upper triangle of S (window-local -> global), fixed point
  const int ld = 6 * ov.F;
  const int gbase = 6 * fmin;
#pragma unroll
  for (int i = 0; i < SY_NT; ++i)
#pragma unroll
    for (int j = 0; j < SY_NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = r0 + wr * SY_QW + 8 * i + (lane >> 2);
        const int lc = c0 + wc * SY_QW + 8 * j + (lane & 3) * 2 + h;
        if (lr > lc || lc >= LD) continue;  // padded rows/cols are zero
        const int r = gbase + lr, c = gbase + lc;
        if (c >= ld) continue;
        const long long qv = llrint(accd[i][j][h] * scale[r] * scale[c]);
        if (qv != 0) atomicAdd(&acc[static_cast<int64_t>(r) * ld + c], static_cast<unsigned long long>(qv));
      }
}

__global__ void k_schur_final(int F, const double* __restrict__ H21, double lambda, const double* __restrict__ scale,
                              const unsigned long long* __restrict__ acc, double* __restrict__ S) {
  const int n = 6 * F;
  const int64_t total = static_cast<int64_t>(n) * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / n), c = static_cast<int>(e % n);
    double v = 0.0;
    if (r / 6 == c / 6) v = H21[21 * (r / 6) + h21_index(r % 6, c % 6)] + (r == c ? lambda : 0.0);
    const int64_t eu = r <= c ? e : static_cast<int64_t>(c) * n + r;  // upper-triangle accumulator
    const double upd = static_cast<double>(static_cast<long long>(acc[eu])) / (scale[r] * scale[c]);
    S[e] = v - upd;
  }
}

// ---------------------------------------------------------------------------------
// Blocked right-looking Cholesky, NB = 32, lower factor in place.
// ---------------------------------------------------------------------------------
constexpr int NB = 32;

__global__ void __launch_bounds__(1024) k_chol_diag(double* __restrict__ A, int n, int j0, int nb, int* fail) {
  __shared__ double a[NB][NB + 1];
  const int r = threadIdx.y, c = threadIdx.x;
  if (r < nb && c < nb && c <= r) a[r][c] = A[static_cast<int64_t>(j0 + r) * n + j0 + c];
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (r == 0 && c == 0) {
      const double d = a[j][j];
      if (!(d > 0.0) || !isfinite(d)) {
        *fail = 1;
        a[j][j] = 1.0;
      } else {
        a[j][j] = sqrt(d);
      }
    }
    __syncthreads();
    if (c == j && r > j && r < nb) a[r][j] = a[r][j] / a[j][j];
    __syncthreads();
    if (r > j && r < nb && c > j && c <= r) a[r][c] -= a[r][j] * a[c][j];
    __syncthreads();
  }
  if (r < nb && c < nb && c <= r) A[static_cast<int64_t>(j0 + r) * n + j0 + c] = a[r][c];
}

__global__ void __launch_bounds__(256) k_chol_panel(double* __restrict__ A, int n, int j0, int nb) {
  __shared__ double l11[NB][NB + 1];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    l11[r][c] = (r < nb && c <= r) ? A[static_cast<int64_t>(j0 + r) * n + j0 + c] : 0.0;
  }
  __syncthreads();
  const int i = j0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* row = A + static_cast<int64_t>(i) * n + j0;
  double l[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    if (c < nb) {
      double v = row[c];
      for (int p = 0; p < c; ++p) v -= l[p] * l11[c][p];
      l[c] = v / l11[c][c];
      row[c] = l[c];
    }
  }
}

// trailing update of the lower triangle: A[i][c] -= sum_p L[i][p] L[c][p], 32x32 tiles
__global__ void __launch_bounds__(256) k_chol_update(double* __restrict__ A, int n, int j0, int nb) {
  const int base = j0 + nb;
  const int m = (n - base + NB - 1) / NB;
  // map blockIdx.x -> (ti, tj) with tj <= ti
  int tid = blockIdx.x, ti = 0;
  while (tid > ti) {
    tid -= ti + 1;
    ++ti;
  }
  const int tj = tid;
  if (ti >= m) return;
  __shared__ double Li[NB][NB + 1], Lj[NB][NB + 1];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, p = e % NB;
    const int gi = base + ti * NB + r, gj = base + tj * NB + r;
    Li[r][p] = (gi < n && p < nb) ? A[static_cast<int64_t>(gi) * n + j0 + p] : 0.0;
    Lj[r][p] = (gj < n && p < nb) ? A[static_cast<int64_t>(gj) * n + j0 + p] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    const int gi = base + ti * NB + r, gj = base + tj * NB + c;
    if (gi >= n || gj >= n || gj > gi) continue;
    double s = 0.0;
#pragma unroll 8
    for (int p = 0; p < NB; ++p) s += Li[r][p] * Lj[c][p];
    A[static_cast<int64_t>(gi) * n + gj] -= s;
  }
}

// ---------------------------------------------------------------------------------
// Triangular solves through an explicit inverse of the Cholesky factor.
// The factor is frozen between factorizations (IC: once per solve + once per rejection),
// so L^-1 is formed once per factorization (blocked triangular inversion, one CTA per
// block column) and every solve is two row-parallel GEMVs spread over all SMs instead
// of a latency-bound single-CTA substitution (solver.cpp:417 reduced_ldlt_.solve).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_tri_diag_inv(const double* __restrict__ L, int n, double* __restrict__ Dinv) {
  // inverse of the lower-triangular diagonal block bi (32x32), forward substitution per column
  const int bi = blockIdx.x;
  const int j0 = bi * NB, nb = min(NB, n - j0);
  __shared__ double l[NB][NB + 1];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    l[r][c] = (r < nb && c <= r) ? L[static_cast<int64_t>(j0 + r) * n + j0 + c] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  const int c = threadIdx.x;
  if (c < NB) {
    double x[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      double v = (r == c) ? 1.0 : 0.0;
      for (int p = 0; p < r; ++p) v -= l[r][p] * x[p];
      x[r] = (r < c) ? 0.0 : v / l[r][r];
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) Dinv[(static_cast<int64_t>(bi) * NB + r) * NB + c] = x[r];
  }
}

// Block column bj of L^-1:  X_jj = Dinv_j;  X_ij = -Dinv_i * sum_{k=j}^{i-1} L_ik X_kj.
// Writes X (row-major lower) and X^T (row-major upper).
__global__ void __launch_bounds__(256) k_tri_inv_col(const double* __restrict__ L, int n, const double* __restrict__ Dinv,
                                                     double* __restrict__ X, double* __restrict__ XT) {
  const int bj = blockIdx.x;
  const int nblk = (n + NB - 1) / NB;
  const int j0 = bj * NB;
  __shared__ double A[NB][NB + 1], Bm[NB][NB + 1], T[NB][NB + 1];
  const int tid = threadIdx.x;
  auto store = [&](int bi, double (*blk)[NB + 1]) {
    for (int e = tid; e < NB * NB; e += blockDim.x) {
      const int r = e / NB, c = e % NB;
      const int gr = bi * NB + r, gc = j0 + c;
      if (gr < n && gc < n) {
        X[static_cast<int64_t>(gr) * n + gc] = blk[r][c];
        XT[static_cast<int64_t>(gc) * n + gr] = blk[r][c];
      }
    }
  };
  // diagonal block
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    T[r][c] = Dinv[(static_cast<int64_t>(bj) * NB + r) * NB + c];
  }
  __syncthreads();
  store(bj, T);
  for (int bi = bj + 1; bi < nblk; ++bi) {
    // T = sum_k L_ik X_kj  (4 outputs per thread)
    double acc[4] = {0, 0, 0, 0};
    for (int bk = bj; bk < bi; ++bk) {
      __syncthreads();
      for (int e = tid; e < NB * NB; e += blockDim.x) {
        const int r = e / NB, c = e % NB;
        const int gr = bi * NB + r, gk = bk * NB + c;
        A[r][c] = (gr < n && gk < n) ? L[static_cast<int64_t>(gr) * n + gk] : 0.0;
        const int kr = bk * NB + r, jc = j0 + c;
        Bm[r][c] = (kr < n && jc < n) ? X[static_cast<int64_t>(kr) * n + jc] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = tid + q * 256, r = e / NB, c = e % NB;
        double s2 = 0.0;
#pragma unroll 8
        for (int p = 0; p < NB; ++p) s2 += A[r][p] * Bm[p][c];
        acc[q] += s2;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + q * 256;
      Bm[e / NB][e % NB] = acc[q];
    }
    for (int e = tid; e < NB * NB; e += blockDim.x) {
      const int r = e / NB, c = e % NB;
      A[r][c] = Dinv[(static_cast<int64_t>(bi) * NB + r) * NB + c];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + q * 256, r = e / NB, c = e % NB;
      double s2 = 0.0;
#pragma unroll 8
      for (int p = 0; p < NB; ++p) s2 += A[r][p] * Bm[p][c];
      T[r][c] = -s2;
    }
    __syncthreads();
    store(bi, T);
    __threadfence_block();
  }
}

// ---------------------------------------------------------------------------------
// k_chol_inv: the whole factorization in ONE persistent cooperative kernel.
// Right-looking blocked Cholesky (NB = 32) of the lower triangle of S in place, fused with
// the explicit inverse X = L^-1 (block rows X_k. = Dinv_k (I - sum_{m<k} L_km X_m.), the sum
// accumulated right-looking in the not-yet-final block rows of X) and X^T.  Per block step k:
//   phase A (all CTAs): panel L_ik = A_ik Dinv_k^T (i > k); X_kj = -Dinv_k R_kj (j < k), X_kk
//   phase B (all CTAs): trailing A_ij -= L_ik L_jk^T (k < j <= i); R_ij += L_ik X_kj (j <= k);
//                       CTA 0 updates A_{k+1,k+1} first and factors it (look-ahead) -> L, Dinv
// with a software grid barrier between phases (co-residency from the cooperative launch).
// Replaces ~3 launches per block column + the per-column inverse CTAs of the earlier path.
// ---------------------------------------------------------------------------------
constexpr int CI_THREADS = 256;
#ifndef PBA_CI_PER_SM
#define PBA_CI_PER_SM 1
#endif

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int g = gen;
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicExch(&bar[1], g + 1u);
    } else {
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
      } while (v == g);
    }
    gen = g + 1u;
  }
  __syncthreads();
}

struct CiSmem {
  double a[NB][NB + 1];
  double b[NB][NB + 1];
  double d[NB][NB + 1];
  double c[NB][NB + 1];  // DMMA product tile of ci_mm
};

// load a 32x32 block (rows r0.., cols c0..) of an n x n row-major matrix; out of range -> 0.
// trans: t[c][r] = M[r0 + r][c0 + c]
__device__ __forceinline__ void ci_load(double (*t)[NB + 1], const double* __restrict__ M, int n, int r0, int c0,
                                        bool trans) {
  for (int e = threadIdx.x; e < NB * NB; e += CI_THREADS) {
    const int r = e / NB, c = e % NB;
    const int gr = r0 + r, gc = c0 + c;
    const double v = (gr < n && gc < n) ? __ldcg(M + static_cast<int64_t>(gr) * n + gc) : 0.0;
    if (trans) t[c][r] = v; else t[r][c] = v;
  }
}
// acc[q] (element e = tid + 256 q, r = e / 32, c = e % 32) = sum_p x[r][p] * y[p][c]
// acc[q] (element e = tid + 256 q, r = e / 32, c = e % 32) = sum_p x[r][p] * y[p][c], on the FP64 tensor
// path: 8 warps x two 8x8 tiles, 8 k-steps of mma.sync.m8n8k4.f64 each, through the shared tile ct.
// Callers synchronise before (x, y written) and after (ct reused by the next product).
__device__ __forceinline__ void ci_mm(const double (*x)[NB + 1], const double (*y)[NB + 1], double (*ct)[NB + 1],
                                      double (&acc)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = warp >> 1, tj0 = 2 * (warp & 1);
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int p0 = 0; p0 < NB; p0 += 4) {
    const double av = x[8 * ti + (lane >> 2)][p0 + (lane & 3)];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double bv = y[p0 + (lane & 3)][8 * (tj0 + u) + (lane >> 2)];
      dmma_8x8x4(d[u][0], d[u][1], av, bv);
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    ct[8 * ti + (lane >> 2)][8 * (tj0 + u) + 2 * (lane & 3)] = d[u][0];
    ct[8 * ti + (lane >> 2)][8 * (tj0 + u) + 2 * (lane & 3) + 1] = d[u][1];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * CI_THREADS;
    acc[q] = ct[e / NB][e % NB];
  }
}
__device__ __forceinline__ void ci_store(double* __restrict__ M, int n, int r0, int c0, const double (&acc)[4],
                                         double sign, double* __restrict__ MT) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * CI_THREADS, r = e / NB, c = e % NB;
    const int gr = r0 + r, gc = c0 + c;
    if (gr < n && gc < n) {
      M[static_cast<int64_t>(gr) * n + gc] = sign * acc[q];
      if (MT) MT[static_cast<int64_t>(gc) * n + gr] = sign * acc[q];
    }
  }
}

// Factor the diagonal block k in shared memory: L_kk into A, Dinv_k = L_kk^-1 into Dinv.
// One CTA barrier per column: every thread derives the pivot itself, the trailing update reads the
// unscaled column j (l_rj l_cj = a_rj a_cj / d_j) and the scaled column goes to a second buffer, so
// the update and the scaling of column j do not conflict.
__device__ void ci_diag(CiSmem& sm, double* __restrict__ A, int n, int k, double* __restrict__ Dinv, int* fail) {
  const int k0 = k * NB, kb = min(NB, n - k0);
  double (*a)[NB + 1] = sm.a;
  double (*l)[NB + 1] = sm.b;
  for (int e = threadIdx.x; e < NB * NB; e += CI_THREADS) {
    const int r = e / NB, c = e % NB;
    a[r][c] = (r < kb && c < kb && c <= r) ? __ldcg(A + static_cast<int64_t>(k0 + r) * n + k0 + c)
                                           : (r == c ? 1.0 : 0.0);
    l[r][c] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < NB; ++j) {
    double dj = a[j][j];
    if (!(dj > 0.0) || !isfinite(dj)) {
      if (threadIdx.x == 0) *fail = 1;
      dj = 1.0;
    }
    const double piv = sqrt(dj), inv = 1.0 / piv, inv2 = inv * inv;
    if (threadIdx.x < NB && threadIdx.x >= j) l[threadIdx.x][j] = threadIdx.x == j ? piv : a[threadIdx.x][j] * inv;
    for (int e = threadIdx.x; e < NB * NB; e += CI_THREADS) {
      const int r = e / NB, c = e % NB;
      if (c > j && r >= c) a[r][c] -= a[r][j] * a[c][j] * inv2;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NB * NB; e += CI_THREADS) {
    const int r = e / NB, c = e % NB;
    a[r][c] = l[r][c];
    if (r < kb && c <= r) A[static_cast<int64_t>(k0 + r) * n + k0 + c] = l[r][c];
  }
  __syncthreads();
  // Dinv_k: forward substitution, one column per thread
  if (threadIdx.x < NB) {
    const int c = threadIdx.x;
    double x[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int p = 0; p < r; ++p) v -= a[r][p] * x[p];
      x[r] = (r < c) ? 0.0 : v / a[r][r];
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) Dinv[(static_cast<int64_t>(k) * NB + r) * NB + c] = x[r];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(CI_THREADS) k_chol_inv(double* __restrict__ A, int n, double* __restrict__ X,
                                                         double* __restrict__ XT, double* __restrict__ Dinv,
                                                         int* __restrict__ fail, unsigned int* __restrict__ bar) {
  __shared__ CiSmem sm;
  unsigned int gen = 0;
  if (threadIdx.x == 0) gen = *reinterpret_cast<volatile unsigned int*>(bar + 1);
  const int nblk = (n + NB - 1) / NB;
  const int G = gridDim.x, cta = blockIdx.x;
  if (cta == 0) ci_diag(sm, A, n, 0, Dinv, fail);
  grid_barrier(bar, gen);
  for (int k = 0; k < nblk; ++k) {
    const int k0 = k * NB;
    // ---- phase A: panel + block row k of X ----
    const int npanel = nblk - k - 1;
    const int itemsA = npanel + k + 1;
    bool dl = false;
    for (int it = cta; it < itemsA; it += G) {
      if (!dl) {  // Dinv_k^T (panel) -- loaded once per CTA and step
        for (int e = threadIdx.x; e < NB * NB; e += CI_THREADS) {
          const int r = e / NB, c = e % NB;
          sm.d[r][c] = __ldcg(Dinv + (static_cast<int64_t>(k) * NB + r) * NB + c);
        }
        dl = true;
      }
      __syncthreads();
      double acc[4];
      if (it < npanel) {  // L_ik = A_ik Dinv_k^T
        const int i0 = (k + 1 + it) * NB;
        ci_load(sm.a, A, n, i0, k0, false);
        for (int e = threadIdx.x; e < NB * NB; e += CI_THREADS) sm.b[e % NB][e / NB] = sm.d[e / NB][e % NB];
        __syncthreads();
        ci_mm(sm.a, sm.b, sm.c, acc);
        ci_store(A, n, i0, k0, acc, 1.0, nullptr);
      } else {
        const int j = it - npanel;  // 0..k
        if (j == k) {               // X_kk = Dinv_k
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + q * CI_THREADS;
            acc[q] = sm.d[e / NB][e % NB];
          }
          ci_store(X, n, k0, k0, acc, 1.0, XT);
        } else {  // X_kj = -Dinv_k R_kj
          ci_load(sm.b, X, n, k0, j * NB, false);
          __syncthreads();
          ci_mm(sm.d, sm.b, sm.c, acc);
          ci_store(X, n, k0, j * NB, acc, -1.0, XT);
        }
      }
      __syncthreads();
    }
    grid_barrier(bar, gen);
    if (k + 1 >= nblk) break;
    // ---- phase B: trailing update of A, right-looking accumulation of R; look-ahead on CTA 0 ----
    const int m = nblk - k - 1;                 // trailing block rows k+1 .. nblk-1
    const int ntrail = m * (m + 1) / 2;         // tiles (i, j), k < j <= i
    const int nr = m * (k + 1);                 // tiles (i, j), i > k, j <= k
    const int items = ntrail + nr;
    auto do_item = [&](int it) {
      double acc[4];
      if (it < ntrail) {
        int t = it, ti = 0;
        while (t > ti) {
          t -= ti + 1;
          ++ti;
        }
        const int i0 = (k + 1 + ti) * NB, j0 = (k + 1 + t) * NB;
        ci_load(sm.a, A, n, i0, k0, false);     // L_ik
        ci_load(sm.b, A, n, j0, k0, true);      // L_jk^T
        __syncthreads();
        ci_mm(sm.a, sm.b, sm.c, acc);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = threadIdx.x + q * CI_THREADS, r = e / NB, c = e % NB;
          const int gr = i0 + r, gc = j0 + c;
          if (gr < n && gc < n && gc <= gr) A[static_cast<int64_t>(gr) * n + gc] -= acc[q];
        }
      } else {
        const int u = it - ntrail;
        const int ti = u / (k + 1), j = u % (k + 1);
        const int i0 = (k + 1 + ti) * NB, j0 = j * NB;
        ci_load(sm.a, A, n, i0, k0, false);     // L_ik
        ci_load(sm.b, X, n, k0, j0, false);     // X_kj
        __syncthreads();
        ci_mm(sm.a, sm.b, sm.c, acc);
        const bool first = j == k;              // R_ij starts at step k = j
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = threadIdx.x + q * CI_THREADS, r = e / NB, c = e % NB;
          const int gr = i0 + r, gc = j0 + c;
          if (gr < n && gc < n) {
            double* dst = X + static_cast<int64_t>(gr) * n + gc;
            *dst = first ? acc[q] : *dst + acc[q];
          }
        }
      }
      __syncthreads();
    };
    if (cta == 0) {
      do_item(0);                               // tile (k+1, k+1)
      ci_diag(sm, A, n, k + 1, Dinv, fail);     // look-ahead factorization of the next diagonal block
    }
    if (G > 1) {
      for (int it = 1 + (cta + G - 1) % G; it < items; it += G - 1)
        if (cta != 0) do_item(it);
    } else {
      for (int it = 1; it < items; ++it) do_item(it);
    }
    grid_barrier(bar, gen);
  }
}

// y = M b for a triangular row-major M (lower: columns <= row; upper: columns >= row).
__global__ void __launch_bounds__(256) k_tri_gemv(const double* __restrict__ M, int n, int lower,
                                                  const double* __restrict__ b, double* __restrict__ y,
                                                  int* __restrict__ nonfinite) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n) return;
  const int c0 = lower ? 0 : r, c1 = lower ? r + 1 : n;
  const double* row = M + static_cast<int64_t>(r) * n;
  double s2 = 0.0;
  for (int c = c0 + lane; c < c1; c += 32) s2 += row[c] * b[c];
  s2 = warp_sum(s2);
  if (lane == 0) {
    y[r] = s2;
    if (nonfinite && !isfinite(s2)) atomicOr(nonfinite, 1);
  }
}

int next_pow2(int p) {
  int g = 1;
  while (g < p) g <<= 1;
  return g;
}

}  // namespace

// ================================ launchers =========================================

namespace {
std::atomic<int64_t> g_launches{0};
}
void count_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

#ifndef PBA_IC_LPO
#define PBA_IC_LPO 1
#endif
template <int MODE>
void launch_lane(const ObsArgs& a, cudaStream_t s) {
  // compile-time pattern (unrolled pixel loop) for the IC pass on 8-pixel patterns; the
  // Hessian-building passes stay rolled (register pressure)
  if (MODE == OBS_IC && a.pat.P == 8) k_obs_lane<MODE, (MODE == OBS_IC ? 8 : 0), (MODE == OBS_IC ? PBA_IC_LPO : 1)><<<a.ov.ntiles, NT, 0, s>>>(a);
  else k_obs_lane<MODE, 0, 1><<<a.ov.ntiles, NT, 0, s>>>(a);
}

// IC frame records from the candidate poses (PBA_TAB_SCALED: rows 0/1 of the candidate pose
// pre-multiplied by fx, fy; (fsx, fsy) = in-margin bounds W - 3, H - 3; PBA_IC_V2: tau = R0^T t0)
__global__ void k_frame_recs(int F, const PoseD* __restrict__ pe, const PoseD* __restrict__ p0,
                             const FrameD* __restrict__ frames, FrameRec* __restrict__ recs) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const FrameD fr = frames[f];
  FrameRec r;
  r.pe = pe[f];
  r.p0 = p0[f];
  r.t0z = r.p0.t[2];
#if PBA_IC_V2
  const PoseD q = p0[f];
#pragma unroll
  for (int j = 0; j < 3; ++j) r.p0.t[j] = q.R[j] * q.t[0] + q.R[3 + j] * q.t[1] + q.R[6 + j] * q.t[2];
#endif
#if PBA_TAB_SCALED
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    r.pe.R[c] *= fr.fx;
    r.pe.R[3 + c] *= fr.fy;
  }
  r.pe.t[0] *= fr.fx;
  r.pe.t[1] *= fr.fy;
  r.fsx = static_cast<double>(fr.W - 3);
  r.fsy = static_cast<double>(fr.H - 3);
#else
  r.fsx = fr.fx;
  r.fsy = fr.fy;
#endif
  r.cx = fr.cx;
  r.cy = fr.cy;
  r.img = fr.img;
  r.W = fr.W;
  r.H = fr.H;
  recs[f] = r;
}

void launch_frame_recs(int F, const PoseD* pose_eval, const PoseD* pose0, const FrameD* frames, FrameRec* recs,
                       cudaStream_t s) {
  if (F <= 0) return;
  k_frame_recs<<<(F + 127) / 128, 128, 0, s>>>(F, pose_eval, pose0, frames, recs);
  count_launches(1);
}

namespace {
// The constant tables are one per process: passes of different handles (e.g. the shards of one
// process on their own streams) take turns per slot, ordered by an event and a host mutex.
std::mutex g_tab_mutex;
cudaEvent_t g_tab_free[kTabSlots] = {};
}  // namespace

void launch_obs_ic_tab(const ObsArgs& a, const FrameTab* tabs, int ntabs, const FrameRec* recs, cudaStream_t s,
                       cudaStream_t side, cudaEvent_t fork, cudaEvent_t join) {
  // the frame chunks are independent (disjoint tiles): chunks after the first run on a side
  // stream so their launches overlap instead of serialising tail effects
  const bool fan = ntabs > 1 && side && fork && join;
  if (fan) {
    cudaEventRecord(fork, s);
    cudaStreamWaitEvent(side, fork, 0);
  }
  std::lock_guard<std::mutex> lk(g_tab_mutex);
  for (int i = 0; i < ntabs; ++i) {
    const int nb = tabs[i].ntiles;
    if (nb == 0) continue;
    cudaStream_t st = (fan && i > 0) ? side : s;
    const int slot = tabs[i].slot;
    if (!g_tab_free[slot]) cudaEventCreateWithFlags(&g_tab_free[slot], cudaEventDisableTiming);
    cudaStreamWaitEvent(st, g_tab_free[slot], 0);  // the slot's previous pass (any handle) is done
    cudaMemcpyToSymbolAsync(c_tab, recs + tabs[i].f0, tabs[i].nf * sizeof(FrameRec),
                            static_cast<size_t>(slot) * kTabFrames * sizeof(FrameRec), cudaMemcpyDeviceToDevice, st);
    if (a.pat.P == 8) k_obs_lane_tab<OBS_IC, 8, PBA_IC_LPO><<<nb, NT, 0, st>>>(a, tabs[i]);
    else k_obs_lane_tab<OBS_IC, 0, 1><<<nb, NT, 0, st>>>(a, tabs[i]);
    cudaEventRecord(g_tab_free[slot], st);
    count_launches(2);
  }
  if (fan) {
    cudaEventRecord(join, side);
    cudaStreamWaitEvent(s, join, 0);
  }
}

void launch_obs(int mode, const ObsArgs& a, cudaStream_t s) {
  if (a.ov.ntiles == 0) return;
  const int G = next_pow2(a.pat.P);
  count_launches(1);
  switch (mode) {
    case OBS_ENERGY: launch_energy(a, G, s); break;
    case OBS_IC: launch_lane<OBS_IC>(a, s); break;
    case OBS_FC: k_obs_lane<OBS_FC, 0, 1><<<a.ov.ntiles, NT, 0, s>>>(a); break;
    case OBS_BUILD: launch_lane<OBS_BUILD>(a, s); break;
    default: launch_lane<OBS_REFRESH>(a, s); break;
  }
}

void launch_pose_update(int ic, int F, const PoseD* cur, const PoseD* pose0, const double* xp, PoseD* cand,
                        cudaStream_t s) {
  k_pose_update<<<(F + 127) / 128, 128, 0, s>>>(ic, F, cur, pose0, xp, cand);
  count_launches(1);
}

static int reduce_blocks(int N, int minb) {
  const int ntask = (N + kPPW - 1) / kPPW;
  const int nb = (ntask + NT / 32 - 1) / (NT / 32);
  return std::max(1, std::min(nb, 148 * minb));
}
int backsub_blocks(int N) { return reduce_blocks(N, kBsMinB); }
int point_blocks(int N) { return reduce_blocks(N, kPtMinB); }

void launch_bdot(const ObsView& ov, const double* B, const double* xp, double* tq, cudaStream_t s) {
  if (ov.ntiles == 0) return;
  k_bdot<<<ov.ntiles, NT, 0, s>>>(ov, B, xp, tq);
  count_launches(1);
}

void launch_backsub(const BacksubArgs& a, cudaStream_t s) {
  const int nb = backsub_blocks(a.ov.N);
  if (nb > 0) {
    const size_t smem = a.xp_smem ? 6 * static_cast<size_t>(a.ov.F) * sizeof(double) : 0;
    k_backsub<<<nb, NT, smem, s>>>(a);
    count_launches(1);
  }
}

void launch_point(const PointArgs& a, cudaStream_t s) {
  const int nb = point_blocks(a.ov.N);
  if (nb > 0) {
    k_point<<<nb, NT, 0, s>>>(a);
    count_launches(1);
  }
}

void launch_template_values(int N, const PatternD& pat, const FrameD& ref, const double2* anc, double* tval,
                            double4* tgrad, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(N) * pat.P;
  if (n == 0) return;
  k_template_values<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(N, pat, ref, 1.0 / ref.fx, 1.0 / ref.fy, anc,
                                                                       tval, tgrad);
  count_launches(1);
}

void launch_b_to_pm(const ObsView& ov, const double* B, double* Bpm, cudaStream_t s) {
  if (ov.NO == 0) return;
  const int g = static_cast<int>(std::min<int64_t>((ov.NO * 3 + 255) / 256, 148 * 32));
  k_b_to_pm<<<g, 256, 0, s>>>(ov, B, Bpm);
  count_launches(1);
}

void launch_cf(const ObsView& ov, const double* B, const double* s_n, double* partial_cf, cudaStream_t s,
               const MaxUpdArgs* mu) {
  if (ov.ntiles > 0) {
    k_cf<<<ov.ntiles, NT, 0, s>>>(ov, B, s_n, partial_cf, mu ? *mu : MaxUpdArgs{});
    count_launches(1);
  }
}

void launch_finalize(const FinalizeArgs& a, cudaStream_t s) {
  k_finalize<<<std::max(a.ov.F, 1), NT, 0, s>>>(a);
  count_launches(1);
}

void launch_commit(int N, int F, const double* d_cand, const PoseD* pose_cand, double scale_d, double scale_t,
                   double* d_cur, PoseD* pose_cur, cudaStream_t s) {
  const int m = N > F ? N : F;
  k_commit<<<(m + 255) / 256, 256, 0, s>>>(N, F, d_cand, pose_cand, scale_d, scale_t, d_cur, pose_cur);
  count_launches(1);
}

void launch_gauge(int N, int F, const double* scale, double* d, PoseD* pose, cudaStream_t s) {
  const int m = N > F ? N : F;
  if (m == 0) return;
  k_gauge_apply<<<(m + 255) / 256, 256, 0, s>>>(N, F, scale, d, pose);
  count_launches(1);
}

void launch_max_reproj(const ObsView& ov, const FrameD* frames, const FrameD& ref, const double2* anchor, int dx0,
                       int dy0, const PoseD* pa, const double* da, const PoseD* pb, const double* db, double* partial,
                       int nblocks, cudaStream_t s) {
  k_max_reproj<<<nblocks, NT, 0, s>>>(ov, frames, ref, anchor, dx0, dy0, pa, da, pb, db, partial);
  count_launches(1);
}

__global__ void k_dense_rows(const int32_t* __restrict__ chunk_pts, int npts, const int32_t* __restrict__ chunk_of,
                             const int4* __restrict__ chunks, const int64_t* __restrict__ chunk_off,
                             int64_t* __restrict__ dense_row) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  const int c = chunk_of[p];
  const int4 ch = chunks[c];
  dense_row[chunk_pts[p]] = chunk_off[c] + static_cast<int64_t>(p - ch.x) * ch.w - 6 * ch.z;
}

__global__ void k_tile_first_point(int ntiles, const int64_t* __restrict__ tile_q0, const int32_t* __restrict__ fm_point,
                                   int32_t* __restrict__ key) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntiles) key[t] = fm_point[tile_q0[t]];
}
void launch_tile_first_point(int ntiles, const int64_t* tile_q0, const int32_t* fm_point, int32_t* key, cudaStream_t s) {
  if (ntiles <= 0) return;
  k_tile_first_point<<<(ntiles + 255) / 256, 256, 0, s>>>(ntiles, tile_q0, fm_point, key);
  count_launches(1);
}

void launch_dense_rows(const SchurPlan& plan, int64_t* dense_row, cudaStream_t s) {
  if (plan.npts <= 0) return;
  k_dense_rows<<<(plan.npts + 255) / 256, 256, 0, s>>>(plan.chunk_pts, plan.npts, plan.chunk_of, plan.chunks,
                                                       plan.chunk_off, dense_row);
  count_launches(1);
}

void launch_schur_acc(const ObsView& ov, const double* H21, const double* B, const double* D, double lambda,
                      double* scale, unsigned long long* acc, const SchurPlan* plan, bool densify, cudaStream_t s,
                      const double* scale_in) {
  const int n = 6 * ov.F;
  const int64_t total = static_cast<int64_t>(n) * n;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16)));
  const bool dense = plan && plan->nblocks > 0;
  k_schur_scale<<<blocks, 256, 0, s>>>(ov.F, H21, scale, acc, total, dense ? plan->chunk_pts : nullptr,
                                       dense ? plan->npts : 0, D, lambda, dense ? plan->wsort : nullptr, scale_in);
  int launched = 1;
  if (dense) {
    if (densify) {
      k_schur_densify<<<(plan->npts * 32 + 255) / 256, 256, 0, s>>>(ov, B, plan->chunk_pts, plan->npts, plan->chunk_of,
                                                                    plan->chunks,
                                                                    plan->chunk_off, plan->dense);
      ++launched;
    }
    static bool attr = [] {
      cudaFuncSetAttribute(k_schur_syrk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SY_SMEM));
      return true;
    }();
    (void)attr;
    k_schur_syrk<<<plan->nblocks, SY_THREADS, SY_SMEM, s>>>(ov, plan->blocks, plan->chunks, plan->chunk_off,
                                                            plan->dense, plan->wsort, scale, acc);
    ++launched;
  } else {
    const int pb = (ov.N + (NT / 32) - 1) / (NT / 32);
    if (pb > 0) {
      k_schur_pts<<<pb, NT, 0, s>>>(ov, B, D, lambda, scale, acc);
      ++launched;
    }
  }
  count_launches(launched);
}

void launch_schur_final(const ObsView& ov, const double* H21, double lambda, const double* scale,
                        const unsigned long long* acc, double* S, cudaStream_t s) {
  const int n = 6 * ov.F;
  const int64_t total = static_cast<int64_t>(n) * n;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16)));
  k_schur_final<<<blocks, 256, 0, s>>>(ov.F, H21, lambda, scale, acc, S);
  count_launches(1);
}

void launch_schur(const ObsView& ov, const double* H21, const double* B, const double* D, double lambda, double* S,
                  double* scale, unsigned long long* acc, const SchurPlan* plan, bool densify, cudaStream_t s) {
  launch_schur_acc(ov, H21, B, D, lambda, scale, acc, plan, densify, s);
  launch_schur_final(ov, H21, lambda, scale, acc, S, s);
}

__global__ void k_xreduce(const double* __restrict__ in, int world, int K, const XPlan plan, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  int sg = 0;
  while (sg < plan.nseg - 1 && k >= plan.seg_end[sg]) ++sg;
  const bool mx = plan.seg_max[sg] != 0;
  double v = in[k];
  for (int r = 1; r < world; ++r) {
    const double x = in[static_cast<int64_t>(r) * K + k];
    v = mx ? fmax(v, x) : v + x;
  }
  out[k] = v;
}

void launch_xreduce(const double* in, int world, int K, const XPlan& plan, double* out, cudaStream_t s) {
  if (K <= 0) return;
  k_xreduce<<<(K + 255) / 256, 256, 0, s>>>(in, world, K, plan, out);
  count_launches(1);
}

__global__ void k_rhs(int n, const double* __restrict__ g, const double* __restrict__ cf, double* __restrict__ rhs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rhs[i] = -g[i] + cf[i];
}

void launch_rhs(int n, const double* g, const double* cf, double* rhs, cudaStream_t s) {
  if (n <= 0) return;
  k_rhs<<<(n + 255) / 256, 256, 0, s>>>(n, g, cf, rhs);
  count_launches(1);
}

__global__ void k_gauge_from_sum(const double* __restrict__ sum, double n_total, int enabled, double* __restrict__ gauge) {
  const double mean = *sum / n_total;
  *gauge = (enabled && mean > 0.0 && isfinite(mean)) ? mean : 1.0;
}

void launch_gauge_from_sum(const double* sum, double n_total, int enabled, double* gauge, cudaStream_t s) {
  k_gauge_from_sum<<<1, 1, 0, s>>>(sum, n_total, enabled, gauge);
  count_launches(1);
}

void launch_cholesky(double* S, int n, int* fail, cudaStream_t s) {
  for (int j0 = 0; j0 < n; j0 += NB) {
    const int nb = std::min(NB, n - j0);
    k_chol_diag<<<1, dim3(NB, NB), 0, s>>>(S, n, j0, nb, fail);
    count_launches(1);
    const int rest = n - j0 - nb;
    if (rest > 0) {
      k_chol_panel<<<(rest + 255) / 256, 256, 0, s>>>(S, n, j0, nb);
      const int m = (rest + NB - 1) / NB;
      k_chol_update<<<m * (m + 1) / 2, 256, 0, s>>>(S, n, j0, nb);
      count_launches(2);
    }
  }
}

void launch_tri_inverse(const double* L, int n, double* Dinv, double* X, double* XT, cudaStream_t s) {
  const int nblk = (n + NB - 1) / NB;
  if (nblk == 0) return;
  k_tri_diag_inv<<<nblk, 256, 0, s>>>(L, n, Dinv);
  k_tri_inv_col<<<nblk, 256, 0, s>>>(L, n, Dinv, X, XT);
  count_launches(2);
}

int chol_inv_grid() {
  static int g = [] {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_inv, CI_THREADS, 0);
    int g0 = std::max(1, sms * std::max(1, std::min(per, PBA_CI_PER_SM)));
    if (const char* e = std::getenv("PBA_CI_GRID")) g0 = std::max(1, std::min(g0, std::atoi(e)));  // experiments
    return g0;
  }();
  return g;
}

void launch_chol_inv(double* S, int n, double* Dinv, double* X, double* XT, int* fail, unsigned int* bar,
                     cudaStream_t s) {
  if (n == 0) return;
  const int nblk = (n + NB - 1) / NB;
  const int items = std::max(nblk * (nblk + 1) / 2, 1);
  int grid = std::min(chol_inv_grid(), items);
  void* args[] = {&S, &n, &X, &XT, &Dinv, &fail, &bar};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_chol_inv), dim3(grid),
                                                    dim3(CI_THREADS), args, 0, s);
  if (e != cudaSuccess) std::fprintf(stderr, "k_chol_inv launch: %s\n", cudaGetErrorString(e));
  count_launches(1);
}

// internal <-> user point order: to_user ? dst[perm[i]] = src[i] : dst[i] = src[perm[i]]
__global__ void k_permute(int N, const int32_t* __restrict__ perm, const double* __restrict__ src,
                          double* __restrict__ dst, int to_user) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (to_user) dst[perm[i]] = src[i]; else dst[i] = src[perm[i]];
}
void launch_permute(int N, const int32_t* perm, const double* src, double* dst, bool to_user, cudaStream_t s) {
  if (N == 0) return;
  k_permute<<<(N + 255) / 256, 256, 0, s>>>(N, perm, src, dst, to_user ? 1 : 0);
  count_launches(1);
}

// Compact the user indices of the points with D == 0 (order fixed afterwards on the host).
__global__ void k_zero_d(int N, const double* __restrict__ D, const int32_t* __restrict__ perm,
                         int32_t* __restrict__ out, unsigned int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool z = i < N && D[i] == 0.0;
  const unsigned m = __ballot_sync(0xffffffffu, z);
  if (m == 0u) return;
  const int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(cnt, static_cast<unsigned>(__popc(m)));
  base = __shfl_sync(m, base, __ffs(m) - 1);
  if (z) out[base + __popc(m & ((1u << lane) - 1u))] = perm[i];
}

int64_t launch_zero_d(int N, const double* D, const int32_t* perm, int32_t* out, cudaStream_t s) {
  unsigned int* cnt = reinterpret_cast<unsigned int*>(out + N);
  cudaMemsetAsync(cnt, 0, sizeof(unsigned int), s);
  k_zero_d<<<(N + 255) / 256, 256, 0, s>>>(N, D, perm, out, cnt);
  count_launches(1);
  unsigned int h = 0;
  cudaMemcpyAsync(&h, cnt, sizeof(unsigned int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return static_cast<int64_t>(h);
}

void launch_trisolve(const double* X, const double* XT, int n, const double* b, double* y, double* x, int* nonfinite,
                     cudaStream_t s) {
  const int nb = (n + 7) / 8;
  if (nb == 0) return;
  k_tri_gemv<<<nb, 256, 0, s>>>(X, n, 1, b, y, nullptr);    // y = L^-1 b
  k_tri_gemv<<<nb, 256, 0, s>>>(XT, n, 0, y, x, nonfinite);  // x = L^-T y
  count_launches(2);
}

}  // namespace pba_b200
