// Host engine behind the C ABI: owns the device state of one PBA problem and
// runs the reference's LM control flow (solver.cpp:481-654, 663-843) with all
// per-pixel / per-point / per-frame work on the GPU.  One 64-byte status copy
// crosses to the host per candidate evaluation.
#pragma once

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pba_gpu.h"
#include "kernels.hpp"

namespace pba_b200 {

struct PbaError : std::runtime_error {
  int code;
  PbaError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline double ms_since(std::chrono::steady_clock::time_point t0) {  // solver.cpp:16-18
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw PbaError(PBA_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device allocations are stream-ordered from the device's default memory pool, which is
// configured to retain freed memory (release threshold = max), behind an exact-size block
// cache: a released block is parked with an event recorded on its stream and handed to the
// next request of the same (rounded) size after that event (stream-ordered, no host wait).
// Repeated solves on same-shaped problems then never go back to the pool, whose large
// requests can otherwise stall on mapping new memory.
void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, size_t bytes, cudaStream_t s);
cudaStream_t alloc_stream();           // stream of the engine being constructed / used
// Host-side phase tracer (env PBA_TRACE=1): synchronizes s and prints the ms since the last mark.
void trace_mark(cudaStream_t s, const char* what);
void set_alloc_stream(cudaStream_t s);
void init_memory_pool();

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    s = alloc_stream();
    p = static_cast<T*>(dev_alloc(count * sizeof(T), s));
    n = count;
  }
  void release() {
    if (p) dev_free(p, n * sizeof(T), s);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

void sort_i32(int32_t* keys, int n, cudaStream_t s);  // engine_layout.cu

struct SolverState {
  pba_config cfg{};
  bool built = false;
  double lambda = 1e-6;
  int builds = 0;
  int factorizations = 0;
  int mcur = 0;  // index of the sticky residual mask in mask_[] (solver.hpp:162)
  // the build pass's tile partials and g_n records still hold IcSolver::run's initial pass (same
  // parameters, rows, residuals and mask); cleared by every later observation pass
  bool init_from_build = false;
  std::vector<std::string> warnings;  // frame warnings (solver.cpp:265-271)
  int64_t zero_d_count = 0;           // number of D_n == 0 points (:359-364)
  mutable std::vector<int32_t> zero_d;  // their user indices, downloaded and sorted on first request
  mutable bool zero_d_ready = false;
};

class Engine {
 public:
  // deferred: the target images may still be in flight when the constructor returns; the caller keeps
  // them valid until the first call that reads them returns (pba_gpu_create_deferred)
  explicit Engine(const pba_problem* p, bool deferred = false);
  ~Engine();

  // ---- C ABI operations (see include/pba_gpu.h) ----
  void set_params(const double* R, const double* t, const double* d);
  void get_params(double* R, double* t, double* d) const;
  void energy(double gamma, const uint8_t* mask, pba_energy_result* out, double* residuals, uint8_t* active);
  void ic_build(const pba_config* cfg);
  void ic_gradient(double* g);
  void ic_compute_step(double* dx);
  void ic_solve_step(const double* g, double* dx);
  void ic_factorize(double lambda);
  void ic_hessian(double* pp, double* dd, double* pd, double* lambda);
  void fc_build(double gamma, double* pp, double* dd, double* pd, double* g);
  void apply_update(int mode, const double* dx, double* R, double* t, double* d, int* invalid);
  double max_reproj_update(const double* R, const double* t, const double* d);
  void normalize_gauge();
  void begin(bool ic, const pba_config* cfg);
  bool iterate(pba_iter_stats* stats);  // returns true when the run is done
  void end(pba_report* rep);

  static void solve_schur_free(int F, int N, const int64_t* obs_ptr, const int32_t* obs_frame,
                               const double* pp, const double* dd, const double* pd, const double* g,
                               double lambda, double* dx);

  int64_t num_obs() const { return NO_; }
  int64_t device_bytes() const;
  cudaStream_t stream() const { return stream_; }
  void set_profiling(bool on);
  void kernel_times(int64_t* counts, double* total_ms);
  // IcSolver::warnings() (solver.hpp:130): the frame warnings, then one per zero-D point; the
  // per-point strings (tens of thousands at C4) are formatted once, on request
  int64_t warning_count() const { return static_cast<int64_t>(ic_.warnings.size()) + ic_.zero_d_count; }
  std::string warning(int64_t i) const;
  const std::string& warnings_text() const;

  std::string last_error;

  // point-sharded runs (pba_gpu_set_exchange)
  void set_exchange(int rank, int world, int64_t n_total, pba_exchange_fn fn, void* ctx);
  // in-library NCCL exchange (nccl_exchange.cu): a communicator from a ncclUniqueId, collectives on stream_
  void set_exchange_nccl(const void* id128, int rank, int world, int64_t n_total);

  // make this engine's stream the allocation stream of the calling thread (every C-ABI entry)
  void bind() const { set_alloc_stream(stream_); }

 private:
  // Declared first so it is destroyed last: device buffers free stream-ordered on it.
  struct StreamHolder {
    cudaStream_t s = nullptr;
    ~StreamHolder() {
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    }
  } sh_;
  // problem / layout
  int N_ = 0, F_ = 0, P_ = 0;
  int64_t NO_ = 0;
  PatternD pat_{};
  FrameD ref_{};
  std::vector<FrameD> frames_h_;
  std::vector<int32_t> perm_;    // internal point -> user point
  std::vector<int32_t> iperm_;   // user point -> internal point
  bool template_ok_ = true;
  std::vector<double> R_state_, t_state_;  // user order (host copy of the problem poses)
  ObsView ov_{};
  cudaStream_t stream_ = nullptr;

  DBuf<float> images_;
  DBuf<FrameD> frames_;
  DBuf<double2> anchor_, anchor_fm_;
  DBuf<double> tval_;             // template values N*P
  DBuf<double4> tgrad_;           // template records {tval, gx, gy, 0} N*P (IC passes)
  DBuf<int64_t> pm_ptr_, fm_ptr_, tile_q0_, tile_q1_;
  DBuf<int32_t> pm_frame_, pm2fm_, fm2pm_, fm_point_, tile_frame_, ftile_ptr_, tile_order_;
  DBuf<int32_t> uo2q_d_;         // caller obs -> frame-major obs q
  DBuf<int32_t> perm_d_;         // internal point -> user point (device copy)
  DBuf<int32_t> zero_idx_;       // scratch: compacted user indices (+1 counter slot)
  DBuf<double> perm_tmp_;        // scratch: per-point values in user order
  DBuf<PoseD> pose_state_, pose_cur_, pose_cand_, pose0_;
  DBuf<double> d_state_, d_cur_, d_cand_, d0_;
  DBuf<uint32_t> mask_[2];        // IC sticky mask / candidate active bits
  DBuf<uint32_t> scratch_bits_;
  DBuf<double> J_;                // 7 planes, IC frozen rows
  DBuf<double> Bic_, Dic_, Hic_;  // IC frozen BlockHessian (solver.hpp:163)
  DBuf<double> Bpm_;              // point-major copy of Bic_ for k_backsub
  DBuf<double> B_[2];             // frame-major pose-depth blocks (cur / cand)
  DBuf<double> D_[2];
  DBuf<double> H_[2];             // 21F
  DBuf<double> gn_[2], gf_[2], rhs_[2];
  DBuf<double2> rec_;
  DBuf<double> rec_g_;            // IC pass g_n terms (8 B per observation)
  DBuf<unsigned long long> gfix_;  // IC pass fixed-point g_n sums (N, zero between passes)
  DBuf<double> gscale_;            // per-point fixed-point scale S_n (set by the IC build)
  bool use_gfix_ = true;           // env PBA_IC_GFIX=0: per-observation records + point-major gather instead
  struct IcEvalArgs {              // the last IC pass (re-run without fixed point if its flag is raised)
    const PoseD* pose;
    const double* d;
    const uint32_t* mask_in;
    uint32_t* active_out;
    int buf;
    double lambda;
    const PoseD* pose_old;
    const double* d_old;
  } last_ic_eval_{};
  const double* schur_scale_in_ = nullptr;  // free Schur solve: host-bounded fixed-point row scales
  DBuf<double> scale_user_;
  std::vector<int64_t> ov_user_ptr_;   // the caller's observation list (point-major), kept by the free solve
  std::vector<int32_t> ov_user_frame_;
  DBuf<double> s_n_, dx_n_, xp_, g_tmp_;
  DBuf<double> r_out_;
  DBuf<double> partial_, partial_cf_, partial_bs_, partial_pt_, partial_mr_;
  DBuf<double> fscal_;            // per-frame scalar partials of k_finalize
  DBuf<unsigned int> ticket_;     // grid tickets {k_backsub, k_finalize}, k_chol_inv barrier {count, generation}
  DBuf<double> S_, schur_scale_, Linv_, LinvT_, Dinv_, ytmp_, gauge_;
  DBuf<unsigned long long> schur_acc_;
  bool chol_inv_ = false;          // env PBA_CHOL_INV=1: the round-1 grid-barrier factor + inverse kernel
  DBuf<int> chol_flags_;           // per-tile completion epochs of k_chol_tiles (factor, then inverse)
  int chol_epoch_ = 0;
  DBuf<int32_t> chunk_pts_, schur_chunk_of_;
  DBuf<int4> schur_blocks_, schur_chunks_;
  DBuf<int64_t> schur_chunk_off_;
  DBuf<double> schur_dense_, schur_wsort_;
  DBuf<int64_t> dense_row_;  // N: chunk-row slot base of each point (the fused dense write)
  const double* dense_B_ = nullptr;  // B whose blocks schur_dense_ holds (null = stale)
  int64_t schur_dense_elems_ = 0;
  SchurPlan schur_plan_{};
  DBuf<Status> status_;
  DBuf<int> flags_;
  Status* status_h_ = nullptr;    // pinned
  std::vector<FrameTab> tabs_;    // IC pass frame chunks (kernel parameters: frames, tiles, constant slot)
  DBuf<FrameRec> frame_recs_;     // IC pass frame records, built on the device per pass
  int64_t tab_min_obs_ = int64_t(1) << 20;  // frame tables from this many observations on (env PBA_TAB_MIN_OBS)
  cudaStream_t side_ = nullptr;   // second stream for the IC pass frame chunks
  cudaStream_t up_stream_ = nullptr;   // target-image upload (deferred handles: completes behind create)
  cudaEvent_t img_done_ = nullptr;
  bool images_pending_ = false;
  void ensure_images();
  cudaEvent_t fork_ = nullptr, join_ = nullptr;
  std::vector<int32_t> ftile_ptr_h_;  // host copy of ov_.ftile_ptr
  int* flags_h_ = nullptr;        // pinned

  SolverState ic_;
  mutable std::string wtext_;       // cache of warnings_text()
  mutable bool wtext_ok_ = false;

  // rank exchange of point-sharded runs (null fn = single process)
  struct Xch {
    int rank = 0, world = 1;
    int64_t n_total = 0;
    pba_exchange_fn fn = nullptr;
    void* ctx = nullptr;
  } xch_;
  std::shared_ptr<void> xch_owner_;  // state of an exchange the library owns (the NCCL communicator)
  struct XSeg {
    double* p;
    int n;
    bool max;
  };
  DBuf<double> xsend_, xrecv_, cf_, gauge_sum_;
  bool sharded() const { return xch_.fn != nullptr; }
  void xreduce(const std::vector<XSeg>& segs);          // sum / max over the ranks, in rank order
  void xsum_i64(unsigned long long* p, int64_t n);       // exact in-place integer sum
  void xcheck(bool ok, int code, const std::string& msg);  // the same error on every rank

  // run (stepping) state
  struct Run {
    bool active = false;
    bool ic = true;
    pba_config cfg{};
    std::chrono::steady_clock::time_point t_start;
    double wall_ms = 0.0;
    int iter = 0;
    int bad = 0;
    double energy = 0.0;
    int64_t initial_active = 0;
    int64_t num_active = 0;
    double lambda = 0.0;        // FC damping
    int fc_builds = 0, fc_factorizations = 0;
    int cur = 0;                // index of the current (accepted) double buffer
    double rhs_lambda = 0.0;    // damping baked into rhs_[cur]
    double gnorm2_n = 0.0;      // |g_n|^2 of the current gradient
    bool done = false;
    bool converged = false, diverged = false;
    int rejected = 0;
    int iterations = 0;
    std::string message;
    std::vector<pba_iter_stats> iters;
    std::vector<double> snapR, snapT, snapD;
  } run_;

  // profiling
  bool prof_ = false;
  std::vector<cudaEvent_t> ev_pool_;
  struct Pending { int kid; cudaEvent_t a, b; };
  std::vector<Pending> pending_;
  int64_t kcount_[PBA_K_COUNT] = {};
  double kms_[PBA_K_COUNT] = {};
  cudaEvent_t ev_begin(int kid);
  void ev_end(int kid, cudaEvent_t a);
  void drain_profile();

  // layout (engine_layout.cu)
  void build_layout(const pba_problem* p, const std::function<void()>& after_obs_upload);
  void mask_to_bits(const uint8_t* mask_user, uint32_t* bits_d);
  void bits_to_user(const uint32_t* bits_d, uint8_t* active_user);
  void rows_to_user(const double* src_fm, int w, double* dst_user);
  void rows_from_user(const double* src_user, int w, double* dst_fm);
  // helpers
  void check_template();  // every rank raises the same OutOfBounds in a sharded run
  void upload_poses(DBuf<PoseD>& dst, const double* R, const double* t);
  void upload_depths_user(DBuf<double>& dst, const double* d_user);
  void download_poses(const DBuf<PoseD>& src, double* R, double* t);
  void download_depths_user(const DBuf<double>& src, double* d_user);
  Status read_status();
  int read_flag(int i);
  void clear_flags();
  ObsArgs obs_args(double gamma) const;
  MaxUpdArgs maxupd_args(const PoseD* pose_old, const PoseD* pose_new, const double* d_old, const double* d_new) const;
  void finalize(const double* partial, const double* partial_cf, bool bs, bool pt, bool want_h, double* g_f,
                double* rhs, const double* g_f_in, double* H, bool status, int e_slot = 0);
  void ic_initial_from_build();  // the run's initial pass from the build pass's sums (no observation pass)
  // IC pieces
  void ic_eval(const PoseD* pose, const double* d, const uint32_t* mask_in, uint32_t* active_out, int buf,
               double lambda, const PoseD* pose_old, const double* d_old);
  void ic_rescale_rhs(int buf, double lambda);
  Status ic_read_status();
  void alloc_schur();
  void fuse_dense(ObsArgs& a);  // the pass also scatters B into the Schur chunk rows
  void build_frame_tabs(const PoseD* pose_d);
  int64_t zero_depth_points(const double* D);
  const std::vector<int32_t>& zero_d_list() const;
 public:
  int64_t warning_points(int32_t* out, int64_t cap) const;
 private:
  bool factor_reduced(const double* H, const double* B, const double* D, double lambda);
  void ic_factorize_loop(double lambda);
  void ic_refresh();
  void ic_solve_loop_and_download(double* dx);
  // FC pieces
  void alloc_fc();
  void fc_eval(double gamma, const PoseD* pose, const double* d, int buf, double lambda_next, const PoseD* pose_old,
               const double* d_old);
  void fc_rescale_rhs(int buf, double lambda);
  // shared
  void download_block_hessian(const DBuf<double>& H, const DBuf<double>& D, const DBuf<double>& B, double* pp,
                              double* dd, double* pd);
  void solve_block_hessian(const double* pp, const double* dd, const double* pd, const double* g, double lambda,
                           double* dx);
  void solve_xp(const double* rhs);  // trisolve with the factor in S_
  void backsub(bool ic, const double* B, const double* D, const double* g_n, double lambda, const double* d_cur,
               double* d_cand, double* dx_out);
  void record_iter(int iter, double energy, double max_upd, int64_t nact, bool accepted, pba_iter_stats* out);
  bool grad_is_zero(int buf);
  void commit_candidate();
  void gauge_candidate();
  bool iterate_ic(pba_iter_stats* st);
  bool iterate_fc(pba_iter_stats* st);
};

}  // namespace pba_b200
