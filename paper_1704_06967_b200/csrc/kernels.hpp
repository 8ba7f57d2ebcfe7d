// Host-side launchers for the B200 PBA kernels (implemented in kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace pba_b200 {

// Observation-pass modes (see kernels.cu k_obs).
enum ObsMode : int {
  OBS_ENERGY = 0,   // residual / Huber only              (energy_eval, solver.cpp:229-244)
  OBS_IC = 1,       // + J^T W r with frozen J rows        (solver.cpp:436-468)
  OBS_FC = 2,       // + FC Jacobian, J^T W J, J^T W r     (solver.cpp:688-724)
  OBS_BUILD = 3,    // IC build at p0: J rows, W0, H       (solver.cpp:273-358)
  OBS_REFRESH = 4   // IC Hessian refresh with fresh W     (solver.cpp:505-531)
};

// Per-tile partial layout of the observation pass (doubles).
constexpr int PT_G = 0;       // 6: sum J_pose^T w r
constexpr int PT_H = 6;       // 21: upper triangle of sum w J_pose J_pose^T
constexpr int PT_E = 27;      // energy
constexpr int PT_NACT = 28;   // active residual count
constexpr int PT_NOOB = 29;   // out-of-bounds count
constexpr int PT_MAXUPD = 30; // max anchor reprojection update
constexpr int PT_STRIDE = 32;

struct ObsArgs {
  ObsView ov;
  double2 pat_d[8];            // pattern offsets as doubles (compile-time 8-pixel passes)
  double2 pat_n[8];            // pattern offsets in normalised reference coordinates (dx / fx, dy / fy)
  FrameD ref;
  double ref_ifx, ref_ify;     // 1 / ref.fx, 1 / ref.fy (template normalization)
  const FrameD* frames;        // F
  PatternD pat;
  const double2* anchor_fm;    // NO: anchor pixel of obs q (frame-major copy, static, TMA-staged)
  const double* tval;          // N*P: template values (internal point order)
  const double4* tgrad;        // N*P: template records {tval, gx, gy, 0} (IC modes), gx NaN = footprint outside
  const double* d_eval;        // N: inverse depths at the evaluation parameters (internal order)
  const double* d_old;         // N or null: inverse depths at the old parameters (max update)
  double gamma;
  const PoseD* pose_eval;      // F
  const PoseD* pose_old;       // F or null (max reprojection update)
  const PoseD* pose0;          // F (IC build)
  const uint32_t* mask_in;     // NO bit words or null (= all pixels)
  uint32_t* active_out;        // NO bit words
  double* r_out;               // NO*P or null
  const double* Jm;            // factored IC Jacobian m (3 per pixel, see k_obs_lane), IC / REFRESH read
  double* Jmw;                 // BUILD output of m
  const double* d0;            // N: frozen depths of the IC build (IC / REFRESH)
  double* B_out;               // NO*6 (FC/BUILD/REFRESH)
  double* B_dense;             // or null: also scatter b_n into the Schur chunk rows (SchurPlan::dense)
  double* Bpm_out;             // or null: also write b_n point-major (at fm2pm[q]; the IC build: no k_b_to_pm)
  const int32_t* fm2pm;
  const int64_t* dense_row;    // N: offset of point n's chunk row minus 6 fmin (slot of frame f at + 6 f)
  double2* rec;                // NO: {sum_k Jd w r, sum_k w Jd^2}
  double* rec_g;               // NO or null: IC pass g_n terms only (sum_k Jd w r)
  unsigned long long* gfix;    // N or null: IC pass g_n accumulated as 64-bit fixed point (RED), scaled by gscale
  const double* gscale;        // N: per-point power-of-two scale S_n (gamma sum |Jd| S_n < 2^61, set at the build)
  int* gfix_bad;               // set when a term is non-finite or outside the fixed-point range (engine re-runs the pass)
  double* partial;             // ntiles * PT_STRIDE
};

void launch_obs(int mode, const ObsArgs& a, cudaStream_t s);

// Frame table of the IC pass for frames [f0, f0 + nf) (tiles [tile0, tile0 + ntiles)), passed
// as a kernel parameter: the frame-uniform records are then read through the constant cache.
#ifndef PBA_TAB_SCALED
#define PBA_TAB_SCALED 1
#endif
#ifndef PBA_IC_V2
#define PBA_IC_V2 1  // IC pass: gradient accumulated in the frame-factored form (see kernels.cu obs_lane_body)
#endif
#ifndef PBA_SY_NT
#define PBA_SY_NT 3  // Schur SYRK: 8x8 DMMA tiles per warp-quadrant side (tile-block edge 16 * PBA_SY_NT)
#endif
constexpr int kSchurTB = 16 * PBA_SY_NT;  // Schur chunk rows are padded to multiples of this (48: 6 W = 240 at C4 fits exactly)
// IC-pass frame record.  With PBA_TAB_SCALED the candidate pose's first two rows (R and t) are
// pre-multiplied by fx and fy, so the warped pixel is u = (fx v_x) / v_z + cx, and (fsx, fsy) hold
// the in-margin bounds (W - 3, H - 3) as doubles; otherwise pe is the plain pose and (fsx, fsy) = (fx, fy).
// With PBA_IC_V2 the frozen pose's translation slot holds tau = R0^T t0 and t0z its z component.
struct FrameRec {
  PoseD pe;                 // evaluation (candidate) pose
  PoseD p0;                 // frozen IC pose (PBA_IC_V2: {R0, tau = R0^T t0})
  double fsx, fsy, cx, cy;
  double t0z;               // frozen translation z (PBA_IC_V2)
  const float* img;
  int W, H;
};
// The IC pass reads its frame records from constant memory: kTabSlots tables of kTabFrames records
// (the frame chunks of one pass run concurrently, one slot each).  The records are built on the
// device from the candidate poses (k_frame_recs) and copied into the slot on the launching stream,
// so the pass needs no host read-back of the poses.
#ifndef PBA_TAB_FRAMES
#define PBA_TAB_FRAMES 240  // one constant table (and one IC-pass launch) for up to 240 frames
#endif
constexpr int kTabFrames = PBA_TAB_FRAMES;
constexpr int kTabSlots = 240 / PBA_TAB_FRAMES;  // kTabSlots * kTabFrames * 248 B of the 64 KB constant bank
struct FrameTab {             // kernel parameter: which frames / tiles / constant slot
  int f0, nf, tile0, ntiles, slot;
};
// records of frames [0, F) into recs (device): scaled candidate rows, {R0, tau}, t0z, intrinsics
void launch_frame_recs(int F, const PoseD* pose_eval, const PoseD* pose0, const FrameD* frames, FrameRec* recs,
                       cudaStream_t s);
void launch_obs_ic_tab(const ObsArgs& a, const FrameTab* tabs, int ntabs, const FrameRec* recs, cudaStream_t s,
                       cudaStream_t side, cudaEvent_t fork, cudaEvent_t join);
// doubles of the factored IC Jacobian store for NO observations of P pixels
inline int64_t jm_doubles(int64_t NO, int P) { return ((NO + 31) / 32) * 3 * static_cast<int64_t>(P) * 32; }

// Candidate poses (IC: apply_ic_update geometry.cpp:197-209 with pc.d0 = 1;
// FC: pose_boxplus geometry.cpp:93-98) from the pose step xp (6F).
void launch_pose_update(int ic, int F, const PoseD* cur, const PoseD* pose0, const double* xp,
                        PoseD* cand, cudaStream_t s);

// Depth back-substitution + candidate depth (solver.cpp:418-428 / 198-208 and
// :553-560 / :747-750).  partial: per block {sum d_cand, #invalid, #nonfinite}.
struct BacksubArgs {
  ObsView ov;
  int ic;
  const double* xp;       // 6F
  const double* B;        // NO*6 frame-major
  const double* D;        // N (without lambda)
  const double* g_n;      // N
  double lambda;
  const double* d_cur;    // N
  const double* d0;       // N (IC)
  double* d_cand;         // N
  double* dx_out;         // N or null
  double* partial;        // nblocks * 4: {sum d_cand, #invalid, #nonfinite, unused}
  const double* Bpm;      // NO*6 point-major copy of B, or null (gather through pm2fm)
  int xp_smem;            // stage xp in shared memory (6F doubles <= 48 KB)
  unsigned int* ticket;   // grid ticket (zero between launches)
  double* gauge_scale;    // out: mean of d_cand (1 when disabled / not positive-finite)
  int gauge_enabled;
  const double* tq = nullptr;  // NO or null: per-observation B_nf . xp_f (k_bdot) instead of B / Bpm
  double* gauge_sum = nullptr; // or null: also the raw sum of d_cand (sharded runs form the mean over ranks)
};
int backsub_blocks(int N);
// tval[n*P + k] = bilinear(ref, anchor_n + offset_k) (build_template, solver.cpp:33-53)
// and tgrad[n*P + k] = image_gradient(ref, .) at the template pixel (NaN: footprint outside)
void launch_template_values(int N, const PatternD& pat, const FrameD& ref, const double2* anc, double* tval,
                            double4* tgrad, cudaStream_t s);
void launch_b_to_pm(const ObsView& ov, const double* B, double* Bpm, cudaStream_t s);
void launch_backsub(const BacksubArgs& a, cudaStream_t s);
// tq[q] = B_q . xp_f over the frame-major observations (FC back-substitution without B gathers)
void launch_bdot(const ObsView& ov, const double* B, const double* xp, double* tq, cudaStream_t s);

// Point-major gather of the per-observation records.
enum PointMode : int { PT_GRAD = 0, PT_FCH = 1, PT_DONLY = 2, PT_RESCALE = 3 };
struct PointArgs {
  ObsView ov;
  int mode;
  const double2* rec;     // NO
  double* g_n;            // N (out for GRAD/FCH; in for RESCALE)
  double* D;              // N (out for FCH/DONLY; in otherwise)
  double lambda;          // damping used for s_n
  double* s_n;            // N out: g_n / (D_n + lambda)
  double* partial;        // nblocks * 2 {sum g_n^2, 0}
  const double* rec_g = nullptr;  // NO or null: PT_GRAD reads these 8-byte g_n terms instead of rec
  unsigned long long* gfix = nullptr;  // N or null: PT_GRAD converts (and clears) the fixed-point g_n sums
  double* gscale = nullptr;            // N: PT_GRAD reads S_n; PT_DONLY writes it (gbound * sum rec.x * S_n < 2^59)
  double gbound = 0.0;                 // PT_DONLY: Huber threshold gamma (|w r| <= gamma in the IC pass)
  int gexp = 59;                       // PT_DONLY: S_n = 2^(gexp - e) (tests raise it to force the overflow fallback)
};
int point_blocks(int N);
void launch_point(const PointArgs& a, cudaStream_t s);

// max_reprojection_update_px (solver.cpp:105-131) between (pose_cur, d_cur) and
// (pose_cand, d_cand) over every observed anchor, fused into k_cf (null pose_cand = skip).
struct MaxUpdArgs {
  const PoseD* pose_cur;
  const PoseD* pose_cand;
  const double* d_cur;
  const double* d_cand;
  const FrameD* frames;
  const double2* anchor;     // N: anchor pixel (internal point order, L2-resident)
  double ref_cx, ref_cy, ref_ifx, ref_ify;
  int dx0, dy0;              // pattern offset 0 (the anchor pixel)
};

// Frame-major  c_f = sum_n B_nf s_n  per tile (partial slots 0..5), max update (slot 6).
void launch_cf(const ObsView& ov, const double* B, const double* s_n, double* partial_cf,
               cudaStream_t s, const MaxUpdArgs* mu = nullptr);

// Reduction of tile partials.  Writes g_f (6F), rhs = -g_f + c_f (6F) when
// partial_cf != null, H (21F upper) when want_h, and the scalar Status.
struct Status {
  double energy;
  double num_active;
  double num_oob;
  double max_upd;
  double sum_d;
  double invalid;
  double nonfinite;
  double gnorm2_n;
};
struct FinalizeArgs {
  ObsView ov;
  const double* partial;      // ntiles * PT_STRIDE (obs pass) or null
  const double* partial_cf;   // ntiles * 8 or null
  const double* partial_bs;   // backsub blocks * 4 or null
  int nbs;
  const double* partial_pt;   // point blocks * 2 or null
  int npt;
  int want_h;
  double* g_f;                // 6F or null
  double* rhs;                // 6F or null (requires partial_cf; uses g_f_in if partial==null)
  const double* g_f_in;       // 6F: gradient when the obs partial is absent (rescale)
  double* H;                  // 21F or null
  double* cf_out;             // 6F or null: the Schur rhs term c_f itself (sharded runs sum it over ranks)
  Status* status;             // or null
  double* fscal;              // F*4 scratch: per-frame {energy, #active, #oob, max update}
  unsigned int* ticket;       // grid ticket (zero between launches)
  int e_slot;                 // 0 = energy / #active / #oob at PT_E..; else energy, #active at e_slot, e_slot + 1
};
void launch_finalize(const FinalizeArgs& a, cudaStream_t s);

// Accept: d_cur = d_cand / mean, t_cur = t_cand * mean (solver.cpp:135-143).
void launch_commit(int N, int F, const double* d_cand, const PoseD* pose_cand, double scale_d,
                   double scale_t, double* d_cur, PoseD* pose_cur, cudaStream_t s);

// Depth-gauge normalization of a candidate with the scale formed by k_backsub (solver.cpp:135-143).
void launch_gauge(int N, int F, const double* scale, double* d, PoseD* pose, cudaStream_t s);

// Max reprojection update between two parameter sets (solver.cpp:105-131).
void launch_max_reproj(const ObsView& ov, const FrameD* frames, const FrameD& ref,
                       const double2* anchor, int dx0, int dy0, const PoseD* pa, const double* da,
                       const PoseD* pb, const double* db, double* partial, int nblocks, cudaStream_t s);

// Reduced camera system S = blockdiag(H_ff + lambda I) - sum_n b_n b_n^T / (D_n + lambda)
// (solver.cpp:170-189, 375-392).  S is 6F x 6F row-major, full.
// Chunk plan for the dense (DMMA) Schur path: points sorted by visibility window, cut into
// chunks, one entry per 64x64 upper-triangle tile-block of each chunk's window Gram matrix.
struct SchurPlan {
  const int32_t* chunk_pts;  // internal point ids in window order (points with observations)
  int npts;
  const int32_t* chunk_of;   // npts: chunk of the p-th window-sorted point
  const int4* chunks;        // per chunk {begin, end, fmin, LD = roundup(6 W, 64)}
  const int64_t* chunk_off;  // per chunk offset (doubles) of its dense [points x LD] block
  double* dense;             // densified blocks b_n (scratch; valid while B is unchanged)
  double* wsort;             // npts: 1 / (D_n + lambda) of the window-sorted points (scratch)
  const int4* blocks;        // per work item {chunk, 0, 0, rb | cb << 16}
  int nblocks;
};
// key[t] = internal point of the first observation of tile t
void launch_tile_first_point(int ntiles, const int64_t* tile_q0, const int32_t* fm_point, int32_t* key, cudaStream_t s);
// dense_row[n] = chunk_off + (p - chunk begin) * LD - 6 fmin for the p-th window-sorted point n
void launch_dense_rows(const SchurPlan& plan, int64_t* dense_row, cudaStream_t s);
// Deterministic (64-bit fixed-point) accumulation; scale: 6F scratch, acc: 36F^2 scratch.
// plan == nullptr selects the per-point pair kernel.
// densify = false reuses plan->dense from the previous call with the same B.
void launch_schur(const ObsView& ov, const double* H21, const double* B, const double* D,
                  double lambda, double* S, double* scale, unsigned long long* acc, const SchurPlan* plan,
                  bool densify, cudaStream_t s);
// The two halves of launch_schur: the fixed-point accumulation of sum_n b_n b_n^T / (D_n + lambda)
// into acc (scale from H21), and S = blockdiag(H + lambda I) - acc / scale.  A point-sharded run sums
// acc over the ranks in between (exact: integer addition).
void launch_schur_acc(const ObsView& ov, const double* H21, const double* B, const double* D, double lambda,
                      double* scale, unsigned long long* acc, const SchurPlan* plan, bool densify, cudaStream_t s,
                      const double* scale_in = nullptr);  // scale_in: per-row fixed-point scales (else 2^30/sqrt(H_rr))
void launch_schur_final(const ObsView& ov, const double* H21, double lambda, const double* scale,
                        const unsigned long long* acc, double* S, cudaStream_t s);

// ---- rank exchange of point-sharded runs ----
// out[k] = sum (or max, for k in a max segment) over r = 0..world-1 of in[r * K + k], in rank order
// (bitwise identical on every rank).  Segments: [seg_end[i-1], seg_end[i]) with flag seg_max[i].
struct XPlan {
  int nseg;
  int seg_end[8];
  int seg_max[8];
};
void launch_xreduce(const double* in, int world, int K, const XPlan& plan, double* out, cudaStream_t s);
// rhs[i] = -g[i] + cf[i] (k_finalize's order)
void launch_rhs(int n, const double* g, const double* cf, double* rhs, cudaStream_t s);
// gauge = sum / n_total when enabled and positive-finite, else 1 (normalize_depth_gauge, solver.cpp:135-143)
void launch_gauge_from_sum(const double* sum, double n_total, int enabled, double* gauge, cudaStream_t s);

// In-place dense Cholesky (lower) of the n x n row-major S; *fail set on a
// non-positive / non-finite pivot (stands in for Eigen::LDLT::info()).
void launch_cholesky(double* S, int n, int* fail, cudaStream_t s);

// Fused factorization (one cooperative launch): lower Cholesky of S in place, X = L^-1
// (row-major lower), XT = X^T, Dinv = inverses of the 32x32 diagonal blocks; *fail set on a
// non-positive / non-finite pivot.  bar: 2 zero-initialised grid-barrier words (reusable).
void launch_chol_inv(double* S, int n, double* Dinv, double* X, double* XT, int* fail, unsigned int* bar,
                     cudaStream_t s);

// X = L^-1 (row-major lower) and XT = X^T, from the Cholesky factor in L (lower).
// Dinv: ceil(n/32) * 32 * 32 scratch.
void launch_tri_inverse(const double* L, int n, double* Dinv, double* X, double* XT, cudaStream_t s);

// x = L^-T L^-1 b = XT (X b) with the explicit inverse; y: n scratch.  *nonfinite set
// when x has a non-finite entry.
// Tiled dataflow Cholesky of the reduced system in place (factor.cu): lower L, Dinv (32 x 32 inverse
// diagonal tiles) and, with X / XT given, the explicit inverse L^-1 and its transpose.  flags:
// 2 * chol_tile_flags(n) ints, zero-initialised once; epoch strictly increasing per call.
void launch_chol_tiles(double* S, int n, double* Dinv, double* X, double* XT, int* flags, int epoch, int* fail,
                       cudaStream_t s);
int chol_tile_flags(int n);
void nccl_unique_id(void* out128);  // nccl_exchange.cu
void launch_trisolve(const double* X, const double* XT, int n, const double* b, double* y, double* x,
                     int* nonfinite, cudaStream_t s);

// Per-point values between internal and user point order (perm: internal -> user).
void launch_permute(int N, const int32_t* perm, const double* src, double* dst, bool to_user, cudaStream_t s);

// User indices of the points with D == 0 into out[0..count) (out holds N + 1 int32: the last
// slot is the counter); returns count (synchronizes s).
int64_t launch_zero_d(int N, const double* D, const int32_t* perm, int32_t* out, cudaStream_t s);

// Process-wide count of kernel launches issued by this library.
void count_launches(int64_t n);
int64_t launch_count();

}  // namespace pba_b200
