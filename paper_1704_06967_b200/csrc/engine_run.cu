// Host engine, part 2: solve steps, FC pieces, sub-step APIs and the LM run loops.
// Every loop below restates /root/reference/proj/src/solver.cpp control flow
// (line numbers cited); numbers are produced by the kernels in kernels.cu.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "engine.hpp"

namespace pba_b200 {

namespace {

using Clock = std::chrono::steady_clock;

// IcSolver::solve_step refactors with lambda * 10 and recurses while the step is non-finite
// (solver.cpp:429-432).  With lambda = 0 (lambda0 = 0 and an unobservable depth, D_n + lambda = 0)
// the reference recurses until its stack overflows; here the retries are bounded like
// IcSolver::factorize's own attempts (solver.cpp:372, 60) and end in SingularHessian.
constexpr int kMaxNonfiniteRetries = 60;
[[noreturn]] void throw_nonfinite_exhausted() {
  throw PbaError(PBA_E_SINGULAR_HESSIAN, "SingularHessian: non-finite step after damping retries");
}

__global__ void k_depth_update(int N, int ic, const double* __restrict__ d, const double* __restrict__ d0,
                               const double* __restrict__ dx, double* __restrict__ out, int* __restrict__ nbad) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  // solver.cpp:553-560 (apply_ic_update with pc.d0 = d0_n) / :747-750
  const double v = ic ? ((d0[n] - dx[n]) / d0[n]) * d[n] : d[n] + dx[n];
  out[n] = v;
  if (v <= 0.0) atomicOr(nbad, 1);
}

__global__ void k_block_sum(const double* __restrict__ x, int n, double* __restrict__ partial) {
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += x[i];
  __shared__ double red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) v += red[w];
    partial[blockIdx.x] = v;
  }
}

void unpack21(const double* h21, double* full36) {
  int h = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      full36[6 * i + j] = h21[h];
      full36[6 * j + i] = h21[h];
      ++h;
    }
}

void need_built(bool built) {
  if (!built) throw PbaError(PBA_E_STATE, "IC solver not built (call pba_gpu_ic_build first)");
}

}  // namespace

void Engine::backsub(bool ic, const double* B, const double* D, const double* g_n, double lambda,
                     const double* d_cur, double* d_cand, double* dx_out) {
  BacksubArgs a{ov_, ic ? 1 : 0, xp_.p, B, D, g_n, lambda, d_cur, d0_.p, d_cand, dx_out, partial_bs_.p,
                (ic && B == Bic_.p && Bpm_.p) ? Bpm_.p : nullptr};
  a.xp_smem = 6 * static_cast<size_t>(F_) * sizeof(double) <= 48 * 1024 ? 1 : 0;
  a.ticket = ticket_.p;
  a.gauge_scale = gauge_.p;
  a.gauge_enabled = run_.cfg.normalize_depth_gauge ? 1 : 0;
  a.gauge_sum = sharded() ? gauge_sum_.p : nullptr;
  const auto e = ev_begin(PBA_K_REDUCE);
  if (!a.Bpm) {  // frame-major blocks: dots first (coalesced), then the point-major 8-byte gather
    launch_bdot(ov_, B, xp_.p, rec_g_.p, stream_);
    a.tq = rec_g_.p;
  }
  launch_backsub(a, stream_);
  if (sharded()) {  // the gauge mean is over every rank's points
    xreduce({{gauge_sum_.p, 1, false}});
    launch_gauge_from_sum(gauge_sum_.p, static_cast<double>(xch_.n_total), a.gauge_enabled, gauge_.p, stream_);
  }
  ev_end(PBA_K_REDUCE, e);
}

// ---- IcSolver::compute_step / solve_step mirrors (solver.cpp:404-434, 475-479) ----
void Engine::ic_solve_loop_and_download(double* dx) {
  double rhs_lambda = ic_.lambda;
  for (int retry = 0;; ++retry) {
    if (retry > kMaxNonfiniteRetries) throw_nonfinite_exhausted();
    if (rhs_lambda != ic_.lambda) {
      ic_rescale_rhs(0, ic_.lambda);
      rhs_lambda = ic_.lambda;
    }
    clear_flags();
    solve_xp(rhs_[0].p);
    backsub(true, Bic_.p, Dic_.p, gn_[0].p, ic_.lambda, d0_.p, d_cand_.p, dx_n_.p);
    finalize(nullptr, nullptr, true, false, false, nullptr, nullptr, nullptr, nullptr, true);
    const Status s = read_status();
    if (!flags_h_[1] && s.nonfinite == 0) break;
    ic_factorize_loop(ic_.lambda * 10.0);  // solver.cpp:429-432
  }
  if (F_ > 0) ck(cudaMemcpy(dx, xp_.p, 6 * F_ * sizeof(double), cudaMemcpyDeviceToHost), "xp");
  download_depths_user(dx_n_, dx + 6 * F_);
}

void Engine::ic_compute_step(double* dx) {
  need_built(ic_.built);
  ic_eval(pose0_.p, d0_.p, mask_[ic_.mcur].p, scratch_bits_.p, 0, ic_.lambda, nullptr, nullptr);
  (void)ic_read_status();
  ic_solve_loop_and_download(dx);
}

void Engine::ic_solve_step(const double* g, double* dx) {
  need_built(ic_.built);
  if (F_ > 0) ck(cudaMemcpy(gf_[0].p, g, 6 * F_ * sizeof(double), cudaMemcpyHostToDevice), "g_f");
  upload_depths_user(gn_[0], g + 6 * F_);
  ic_rescale_rhs(0, ic_.lambda);
  ic_solve_loop_and_download(dx);
}

void Engine::ic_hessian(double* pp, double* dd, double* pd, double* lambda) {
  need_built(ic_.built);
  download_block_hessian(Hic_, Dic_, Bic_, pp, dd, pd);
  if (lambda) *lambda = ic_.lambda;
}

void Engine::download_block_hessian(const DBuf<double>& H, const DBuf<double>& D, const DBuf<double>& B, double* pp,
                                    double* dd, double* pd) {
  if (pp) {
    std::vector<double> h(21 * static_cast<size_t>(F_));
    if (F_ > 0) ck(cudaMemcpy(h.data(), H.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost), "H");
    for (int f = 0; f < F_; ++f) unpack21(&h[21 * f], pp + 36 * f);
  }
  if (dd) download_depths_user(D, dd);
  if (pd) rows_to_user(B.p, 6, pd);
}

// refresh_ic_hessian (solver.cpp:505-531): H from the frozen rows with fresh weights
void Engine::ic_refresh() {
  ic_.init_from_build = false;  // the pass overwrites the tile partials
  ObsArgs a = obs_args(ic_.cfg.gamma);
  a.pose_eval = pose_cur_.p;
  a.d_eval = d_cur_.p;
  a.mask_in = mask_[ic_.mcur].p;
  a.active_out = scratch_bits_.p;
  a.Jm = J_.p;
  a.B_out = Bic_.p;
  fuse_dense(a);
  auto e = ev_begin(PBA_K_IC_BUILD);
  launch_obs(OBS_REFRESH, a, stream_);
  ev_end(PBA_K_IC_BUILD, e);
  PointArgs pa{ov_, PT_DONLY, rec_.p, nullptr, Dic_.p, 0.0, nullptr, partial_pt_.p};
  e = ev_begin(PBA_K_REDUCE);
  launch_point(pa, stream_);
  ev_end(PBA_K_REDUCE, e);
  finalize(partial_.p, nullptr, false, false, true, nullptr, nullptr, nullptr, Hic_.p, false);
  launch_b_to_pm(ov_, Bic_.p, Bpm_.p, stream_);
}

// ---- FC pieces -------------------------------------------------------------------
void Engine::alloc_fc() {
  const size_t nO = std::max<int64_t>(NO_, 1);
  for (int b = 0; b < 2; ++b) {
    B_[b].alloc(6 * nO);
    D_[b].alloc(std::max(N_, 1));
    H_[b].alloc(21 * std::max(F_, 1));
  }
  alloc_schur();
}

// Residual pass + FC J^T W J / J^T W r build at (pose, d) (solver.cpp:63-103, 688-724)
// and the Schur rhs term with lambda_next.
void Engine::fc_eval(double gamma, const PoseD* pose, const double* d, int buf, double lambda_next,
                     const PoseD* pose_old, const double* d_old) {
  ic_.init_from_build = false;  // the pass overwrites the tile partials
  ObsArgs a = obs_args(gamma);
  a.pose_eval = pose;
  a.pose_old = pose_old;
  a.d_eval = d;
  a.d_old = d_old;
  a.mask_in = nullptr;
  a.active_out = scratch_bits_.p;
  a.B_out = B_[buf].p;
  fuse_dense(a);
  auto e = ev_begin(PBA_K_OBS_PASS);
  launch_obs(OBS_FC, a, stream_);
  ev_end(PBA_K_OBS_PASS, e);
  PointArgs pa{ov_, PT_FCH, rec_.p, gn_[buf].p, D_[buf].p, lambda_next, s_n_.p, partial_pt_.p};
  e = ev_begin(PBA_K_REDUCE);
  launch_point(pa, stream_);
  const MaxUpdArgs mu = maxupd_args(pose_old, pose, d_old, d);
  launch_cf(ov_, B_[buf].p, s_n_.p, partial_cf_.p, stream_, pose_old ? &mu : nullptr);
  ev_end(PBA_K_REDUCE, e);
  finalize(partial_.p, partial_cf_.p, pose_old != nullptr, true, true, gf_[buf].p, rhs_[buf].p, nullptr, H_[buf].p,
           true);
}

void Engine::fc_rescale_rhs(int buf, double lambda) {
  PointArgs pa{ov_, PT_RESCALE, rec_.p, gn_[buf].p, D_[buf].p, lambda, s_n_.p, partial_pt_.p};
  const auto e = ev_begin(PBA_K_REDUCE);
  launch_point(pa, stream_);
  launch_cf(ov_, B_[buf].p, s_n_.p, partial_cf_.p, stream_);
  ev_end(PBA_K_REDUCE, e);
  finalize(nullptr, partial_cf_.p, false, false, false, nullptr, rhs_[buf].p, gf_[buf].p, nullptr, false);
}

void Engine::fc_build(double gamma, double* pp, double* dd, double* pd, double* g) {
  check_template();
  ensure_images();
  alloc_fc();
  fc_eval(gamma, pose_state_.p, d_state_.p, 0, 1.0, nullptr, nullptr);
  (void)read_status();
  download_block_hessian(H_[0], D_[0], B_[0], pp, dd, pd);
  if (g) {
    if (F_ > 0) ck(cudaMemcpy(g, gf_[0].p, 6 * F_ * sizeof(double), cudaMemcpyDeviceToHost), "g_f");
    download_depths_user(gn_[0], g + 6 * F_);
  }
}

// ---- sub-step APIs ----------------------------------------------------------------
void Engine::apply_update(int mode, const double* dx, double* R, double* t, double* d, int* invalid) {
  const bool ic = mode == 0;
  if (ic) need_built(ic_.built);
  if (F_ > 0) ck(cudaMemcpy(xp_.p, dx, 6 * F_ * sizeof(double), cudaMemcpyHostToDevice), "xp");
  upload_depths_user(dx_n_, dx + 6 * F_);
  clear_flags();
  launch_pose_update(ic ? 1 : 0, F_, pose_state_.p, pose0_.p, xp_.p, pose_cand_.p, stream_);
  if (N_ > 0)
    k_depth_update<<<(N_ + 255) / 256, 256, 0, stream_>>>(N_, ic ? 1 : 0, d_state_.p, d0_.p, dx_n_.p, d_cand_.p,
                                                           flags_.p + 2);
  if (N_ > 0) count_launches(1);
  const int bad = read_flag(2);
  download_poses(pose_cand_, R, t);
  download_depths_user(d_cand_, d);
  if (invalid) *invalid = bad ? 1 : 0;
}

double Engine::max_reproj_update(const double* R, const double* t, const double* d) {
  check_template();
  upload_poses(pose_cand_, R, t);
  upload_depths_user(d_cand_, d);
  const int nb = static_cast<int>(std::min<int64_t>(1024, std::max<int64_t>(1, (NO_ + 255) / 256)));
  launch_max_reproj(ov_, frames_.p, ref_, anchor_.p, pat_.dx[0], pat_.dy[0], pose_state_.p, d_state_.p,
                    pose_cand_.p, d_cand_.p, partial_mr_.p, nb, stream_);
  std::vector<double> part(nb);
  ck(cudaMemcpyAsync(part.data(), partial_mr_.p, nb * sizeof(double), cudaMemcpyDeviceToHost, stream_), "mr");
  ck(cudaStreamSynchronize(stream_), "sync");
  ck(cudaGetLastError(), "kernel");
  double m = 0.0;
  for (double v : part) m = std::max(m, v);  // final max over per-block maxima
  return NO_ > 0 ? m : 0.0;
}

// normalize_depth_gauge (solver.cpp:135-143) on the problem parameters
void Engine::normalize_gauge() {
  const int nb = std::max(1, std::min(1024, (N_ + 255) / 256));
  if (N_ > 0) {
    k_block_sum<<<nb, 256, 0, stream_>>>(d_state_.p, N_, partial_mr_.p);
    count_launches(1);
  }
  std::vector<double> part(nb, 0.0);
  ck(cudaMemcpyAsync(part.data(), partial_mr_.p, nb * sizeof(double), cudaMemcpyDeviceToHost, stream_), "sum");
  ck(cudaStreamSynchronize(stream_), "sync");
  double mean = 0.0;
  for (double v : part) mean += v;
  mean /= static_cast<double>(N_);
  if (mean <= 0.0 || !std::isfinite(mean)) return;
  launch_commit(N_, F_, d_state_.p, pose_state_.p, mean, mean, d_state_.p, pose_state_.p, stream_);
  download_poses(pose_state_, R_state_.data(), t_state_.data());
}

// ---- free solve_normal_equations_schur (solver.cpp:165-213) --------------------------
void Engine::solve_block_hessian(const double* pp, const double* dd, const double* pd, const double* g,
                                 double lambda, double* dx) {
  alloc_fc();
  std::vector<double> h21(21 * static_cast<size_t>(F_));
  for (int f = 0; f < F_; ++f) {
    int h = 0;
    for (int i = 0; i < 6; ++i)
      for (int j = i; j < 6; ++j) h21[21 * f + h++] = pp[36 * f + 6 * i + j];
  }
  if (F_ > 0) ck(cudaMemcpy(H_[0].p, h21.data(), h21.size() * sizeof(double), cudaMemcpyHostToDevice), "H");
  // The fixed-point Schur accumulator needs a bound on every partial sum.  Built passes get it from
  // the PSD block Hessian (Cauchy-Schwarz: sum_n |B_ni B_nj| / D_n <= sqrt(H_ii H_jj)); caller
  // blocks may be anything, so the row scales come from m_r = max(H_rr, sum_n B_nr^2 / |D_n + lambda|)
  // (the same inequality with |D_n + lambda|), and D_n + lambda = 0 is the reference's
  // non-finite outcome (solver.cpp:177-211: the 1/D terms are inf/NaN).
  {
    std::vector<double> m(6 * static_cast<size_t>(F_), 0.0);
    for (int f = 0; f < F_; ++f)
      for (int i = 0; i < 6; ++i) m[6 * f + i] = std::max(pp[36 * f + 7 * i], 0.0);
    const int64_t* op = ov_user_ptr_.data();
    for (int n = 0; n < N_; ++n) {
      const double Dl = dd[n] + lambda;
      bool any = false;
      for (int64_t o = op[n]; o < op[n + 1]; ++o)
        for (int i = 0; i < 6; ++i) any |= pd[6 * o + i] != 0.0;
      if (Dl == 0.0 || !std::isfinite(Dl))
        throw PbaError(PBA_E_SINGULAR_HESSIAN, any ? "SingularHessian: non-finite pose solution"
                                                   : "SingularHessian: non-finite depth solution");
      const double w = 1.0 / std::fabs(Dl);
      for (int64_t o = op[n]; o < op[n + 1]; ++o) {
        const int f = ov_user_frame_[o];
        for (int i = 0; i < 6; ++i) m[6 * f + i] += pd[6 * o + i] * pd[6 * o + i] * w;
      }
    }
    for (double& v : m) {
      if (!std::isfinite(v)) throw PbaError(PBA_E_SINGULAR_HESSIAN, "SingularHessian: non-finite pose solution");
      v = v > 0.0 ? 1073741824.0 / std::sqrt(v) : 1073741824.0;
    }
    scale_user_.alloc(std::max<size_t>(m.size(), 1));
    if (!m.empty()) ck(cudaMemcpy(scale_user_.p, m.data(), m.size() * sizeof(double), cudaMemcpyHostToDevice), "scale");
  }
  upload_depths_user(D_[0], dd);
  rows_from_user(pd, 6, B_[0].p);
  dense_B_ = nullptr;
  if (F_ > 0) ck(cudaMemcpy(gf_[0].p, g, 6 * F_ * sizeof(double), cudaMemcpyHostToDevice), "g_f");
  upload_depths_user(gn_[0], g + 6 * F_);
  schur_scale_in_ = scale_user_.p;
  const bool fok = factor_reduced(H_[0].p, B_[0].p, D_[0].p, lambda);
  schur_scale_in_ = nullptr;
  if (!fok) throw PbaError(PBA_E_SINGULAR_HESSIAN, "SingularHessian: Schur-reduced factorization failed");
  fc_rescale_rhs(0, lambda);
  clear_flags();
  solve_xp(rhs_[0].p);
  if (read_flag(1)) throw PbaError(PBA_E_SINGULAR_HESSIAN, "SingularHessian: non-finite pose solution");
  backsub(false, B_[0].p, D_[0].p, gn_[0].p, lambda, d_state_.p, d_cand_.p, dx_n_.p);
  finalize(nullptr, nullptr, true, false, false, nullptr, nullptr, nullptr, nullptr, true);
  const Status s = read_status();
  if (s.nonfinite > 0) throw PbaError(PBA_E_SINGULAR_HESSIAN, "SingularHessian: non-finite depth solution");
  if (F_ > 0) ck(cudaMemcpy(dx, xp_.p, 6 * F_ * sizeof(double), cudaMemcpyDeviceToHost), "xp");
  download_depths_user(dx_n_, dx + 6 * F_);
}

void Engine::solve_schur_free(int F, int N, const int64_t* obs_ptr, const int32_t* obs_frame, const double* pp,
                              const double* dd, const double* pd, const double* g, double lambda, double* dx) {
  // A problem shell carrying only the observation structure (images are never read).
  static const float dummy[16] = {0};
  std::vector<pba_image> tg(F, pba_image{4, 4, 1, 1, 0, 0, dummy});
  std::vector<double> R(9 * static_cast<size_t>(F), 0.0), t(3 * static_cast<size_t>(F), 0.0);
  for (int f = 0; f < F; ++f) R[9 * f] = R[9 * f + 4] = R[9 * f + 8] = 1.0;
  std::vector<double> anc(2 * static_cast<size_t>(N), 0.0), d(N, 1.0);
  const int32_t pat[2] = {0, 0};
  pba_problem p{};
  p.ref = pba_image{4, 4, 1, 1, 0, 0, dummy};
  p.num_frames = F;
  p.targets = tg.data();
  p.pose_R = R.data();
  p.pose_t = t.data();
  p.num_points = N;
  p.anchors_px = anc.data();
  p.inv_depths = d.data();
  p.pattern_size = 1;
  p.pattern = pat;
  p.obs_ptr = obs_ptr;
  p.obs_frame = obs_frame;
  Engine e(&p);
  e.ov_user_ptr_.resize(static_cast<size_t>(N) + 1);
  for (int n = 0; n <= N; ++n) e.ov_user_ptr_[n] = obs_ptr ? obs_ptr[n] : static_cast<int64_t>(n) * F;
  e.ov_user_frame_.resize(static_cast<size_t>(e.ov_user_ptr_[N]));
  for (int64_t o = 0; o < e.ov_user_ptr_[N]; ++o) e.ov_user_frame_[o] = obs_frame ? obs_frame[o] : static_cast<int32_t>(o % F);
  e.solve_block_hessian(pp, dd, pd, g, lambda, dx);
}

// =====================================================================================
// LM run loops: IcSolver::run (solver.cpp:481-654), FcSolver::run (solver.cpp:663-843)
// =====================================================================================
void Engine::begin(bool ic, const pba_config* cfg) {
  run_ = Run{};
  run_.ic = ic;
  run_.t_start = Clock::now();
  if (ic) {
    if (cfg || !ic_.built) ic_build(cfg);  // ic_solve == fresh IcSolver(state, cfg).run()
    run_.cfg = ic_.cfg;
    if (F_ > 0) ck(cudaMemcpyAsync(pose_cur_.p, pose0_.p, F_ * sizeof(PoseD), cudaMemcpyDeviceToDevice, stream_), "p");
    if (N_ > 0) ck(cudaMemcpyAsync(d_cur_.p, d0_.p, N_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "d");
    // :487-495 initial pass, sticky mask &= active
    Status s{};
    if (ic_.init_from_build) {  // the build pass already evaluated it (ic_initial_from_build)
      ic_initial_from_build();
      s = read_status();
      ic_.init_from_build = false;  // gn_[0] / rhs_[0] now belong to the run
    } else {
      ic_eval(pose_cur_.p, d_cur_.p, mask_[ic_.mcur].p, mask_[1 - ic_.mcur].p, 0, ic_.lambda, nullptr, nullptr);
      s = ic_read_status();
      ic_.mcur = 1 - ic_.mcur;
    }
    if (s.num_active == 0) throw PbaError(PBA_E_EMPTY_PROBLEM, "no in-bounds residuals");
    run_.energy = s.energy;
    run_.initial_active = run_.num_active = static_cast<int64_t>(s.num_active);
    run_.rhs_lambda = ic_.lambda;
    run_.gnorm2_n = s.gnorm2_n;
  } else {
    if (cfg) {
      run_.cfg = *cfg;
    } else {
      pba_config_default(&run_.cfg);
    }
    check_template();
    ensure_images();
    alloc_fc();
    if (F_ > 0) ck(cudaMemcpyAsync(pose_cur_.p, pose_state_.p, F_ * sizeof(PoseD), cudaMemcpyDeviceToDevice, stream_), "p");
    if (N_ > 0) ck(cudaMemcpyAsync(d_cur_.p, d_state_.p, N_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "d");
    run_.lambda = run_.cfg.lambda0;  // :679
    // :674 initial residual pass, fused with the iteration-1 Hessian build (:688-724)
    fc_eval(run_.cfg.gamma, pose_cur_.p, d_cur_.p, 0, run_.lambda, nullptr, nullptr);
    const Status s = read_status();
    if (s.num_active == 0) throw PbaError(PBA_E_EMPTY_PROBLEM, "no in-bounds residuals");  // :675
    run_.energy = s.energy;
    run_.initial_active = run_.num_active = static_cast<int64_t>(s.num_active);
    run_.rhs_lambda = run_.lambda;
    run_.gnorm2_n = s.gnorm2_n;
  }
  run_.cur = 0;
  run_.wall_ms = ms_since(run_.t_start);
  run_.active = true;
}

bool Engine::iterate(pba_iter_stats* st) {
  if (!run_.active) throw PbaError(PBA_E_STATE, "no active run (call pba_gpu_ic_begin / pba_gpu_fc_begin)");
  if (run_.done) return true;
  return run_.ic ? iterate_ic(st) : iterate_fc(st);
}

void Engine::record_iter(int iter, double energy, double max_upd, int64_t nact, bool accepted, pba_iter_stats* out) {
  pba_iter_stats s{};
  s.iter = iter;
  s.energy = energy;
  s.max_update_px = max_upd;
  s.wall_ms = run_.wall_ms;
  s.hessian_builds = run_.ic ? ic_.builds : run_.fc_builds;
  s.hessian_factorizations = run_.ic ? ic_.factorizations : run_.fc_factorizations;
  s.num_active = nact;
  s.accepted = accepted ? 1 : 0;
  run_.iters.push_back(s);
  if (out) *out = s;
  if (run_.cfg.record_snapshots) {
    const size_t i = run_.snapR.size() / std::max<size_t>(9 * F_, 1);
    (void)i;
    std::vector<double> R(9 * static_cast<size_t>(F_)), t(3 * static_cast<size_t>(F_)), d(N_);
    download_poses(pose_cur_, R.data(), t.data());
    download_depths_user(d_cur_, d.data());
    run_.snapR.insert(run_.snapR.end(), R.begin(), R.end());
    run_.snapT.insert(run_.snapT.end(), t.begin(), t.end());
    run_.snapD.insert(run_.snapD.end(), d.begin(), d.end());
  }
}

bool Engine::grad_is_zero(int buf) {
  if (run_.gnorm2_n != 0.0) return false;
  std::vector<double> g(6 * static_cast<size_t>(F_));
  if (F_ > 0) ck(cudaMemcpy(g.data(), gf_[buf].p, g.size() * sizeof(double), cudaMemcpyDeviceToHost), "g_f");
  for (double v : g)
    if (v != 0.0) return false;
  return true;
}

// normalize_depth_gauge of the candidate (solver.cpp:135-143), on the device, before the
// candidate is evaluated (see k_gauge_mean); accepting is then a plain copy.
void Engine::gauge_candidate() {
  launch_gauge(N_, F_, gauge_.p, d_cand_.p, pose_cand_.p, stream_);  // scale formed by k_backsub
}

void Engine::commit_candidate() {  // solver.cpp:611-620, 803-809
  launch_commit(N_, F_, d_cand_.p, pose_cand_.p, 1.0, 1.0, d_cur_.p, pose_cur_.p, stream_);
}

bool Engine::iterate_ic(pba_iter_stats* st) {
  Run& R = run_;
  const int iter = R.iter + 1;
  if (iter > R.cfg.max_iters) {
    R.done = true;
    return true;
  }
  R.iter = iter;
  const auto t_iter = Clock::now();
  const int b0 = R.cur, b1 = 1 - R.cur;
  if (R.cfg.refresh_ic_hessian && iter > 1) {  // :505-531
    ic_refresh();
    ++ic_.builds;
    ic_factorize_loop(ic_.lambda);
    ic_rescale_rhs(b0, ic_.lambda);
    R.rhs_lambda = ic_.lambda;
  }
  bool accepted = false;
  Status s{};
  int nonfinite_retries = 0;
  while (!accepted) {  // :538-606
    if (R.rhs_lambda != ic_.lambda) {
      ic_rescale_rhs(b0, ic_.lambda);
      R.rhs_lambda = ic_.lambda;
    }
    clear_flags();
    solve_xp(rhs_[b0].p);                                                   // solve_step
    launch_pose_update(1, F_, pose_cur_.p, pose0_.p, xp_.p, pose_cand_.p, stream_);  // :544-552
    backsub(true, Bic_.p, Dic_.p, gn_[b0].p, ic_.lambda, d_cur_.p, d_cand_.p, nullptr);  // :418-428, :553-560
    gauge_candidate();                                                      // :618-620 (gauge-invariant pass)
    ic_eval(pose_cand_.p, d_cand_.p, mask_[ic_.mcur].p, mask_[1 - ic_.mcur].p, b1, ic_.lambda, pose_cur_.p,
            d_cur_.p);                                                      // :561 + next g
    s = ic_read_status();
    if (flags_h_[1] || s.nonfinite > 0) {  // :429-432
      if (++nonfinite_retries > kMaxNonfiniteRetries) throw_nonfinite_exhausted();
      ic_factorize_loop(ic_.lambda * 10.0);
      continue;
    }
    const bool valid = s.invalid == 0 && s.num_active > 0;
    if (valid && s.energy <= R.energy * (1.0 + 1e-12) + 1e-15) {  // :566
      accepted = true;
      R.bad = 0;
    } else {
      if (valid && s.max_upd < R.cfg.threshold_px) {  // :573-595
        R.converged = true;
        R.message = "converged: sub-threshold step rejected";
        R.wall_ms += ms_since(t_iter);
        record_iter(iter, R.energy, s.max_upd, R.num_active, false, st);
        R.iterations = iter;
        R.done = true;
        return true;
      }
      ++R.bad;  // :596-604
      ++R.rejected;
      if (R.bad >= R.cfg.max_bad_steps) {
        R.diverged = true;
        R.message = "Diverged: " + std::to_string(R.bad) + " consecutive rejected damped steps";
        R.done = true;
        return true;
      }
      ic_factorize_loop(ic_.lambda * 10.0);
    }
  }
  const double max_upd = s.max_upd;  // :609
  const bool zero_grad = max_upd < R.cfg.threshold_px ? grad_is_zero(b0) : false;
  commit_candidate();                 // :611-620
  ic_.mcur = 1 - ic_.mcur;            // mask_ &= cand_pass.active (:613-615)
  R.energy = s.energy;
  R.num_active = static_cast<int64_t>(s.num_active);
  R.cur = b1;
  R.rhs_lambda = ic_.lambda;
  R.gnorm2_n = s.gnorm2_n;
  R.wall_ms += ms_since(t_iter);
  record_iter(iter, R.energy, max_upd, R.num_active, true, st);
  R.iterations = iter;
  if (max_upd < R.cfg.threshold_px) {  // :637-643
    R.converged = true;
    if (zero_grad) R.message = "no-progress convergence: zero gradient";
    R.done = true;
    return true;
  }
  return false;
}

bool Engine::iterate_fc(pba_iter_stats* st) {
  Run& R = run_;
  const int iter = R.iter + 1;
  if (iter > R.cfg.max_iters) {
    R.done = true;
    return true;
  }
  R.iter = iter;
  const auto t_iter = Clock::now();
  const int b0 = R.cur, b1 = 1 - R.cur;
  ++R.fc_builds;  // :724 (the build itself was fused into the previous accepted pass)
  bool accepted = false;
  Status s{};
  double lam_next = R.lambda;
  while (!accepted) {  // :730-791
    ++R.fc_factorizations;
    bool ok = factor_reduced(H_[b0].p, B_[b0].p, D_[b0].p, R.lambda);
    lam_next = std::max(R.lambda / 10.0, R.cfg.lambda0);
    if (ok) {
      if (R.rhs_lambda != R.lambda) {
        fc_rescale_rhs(b0, R.lambda);
        R.rhs_lambda = R.lambda;
      }
      clear_flags();
      solve_xp(rhs_[b0].p);
      launch_pose_update(0, F_, pose_cur_.p, pose0_.p, xp_.p, pose_cand_.p, stream_);  // :744-746
      backsub(false, B_[b0].p, D_[b0].p, gn_[b0].p, R.lambda, d_cur_.p, d_cand_.p, nullptr);  // :747-750
      gauge_candidate();  // :807-809: H for the next iteration is built at the normalized candidate
      fc_eval(R.cfg.gamma, pose_cand_.p, d_cand_.p, b1, lam_next, pose_cur_.p, d_cur_.p);     // :752 + next H
      s = read_status();
      if (flags_h_[1] || s.nonfinite > 0) ok = false;  // non-finite solution (:195-211)
    }
    if (!ok) {  // :735-739
      R.lambda *= 10.0;
      ++R.rejected;
      if (++R.bad >= R.cfg.max_bad_steps) break;
      continue;
    }
    const bool valid = s.invalid == 0 && s.num_active > 0;
    if (valid && s.energy <= R.energy * (1.0 + 1e-12) + 1e-15) {  // :756-759
      accepted = true;
      R.bad = 0;
      R.lambda = lam_next;
    } else {
      if (valid && s.max_upd < R.cfg.threshold_px) {  // :764-786
        R.converged = true;
        R.message = "converged: sub-threshold step rejected";
        R.wall_ms += ms_since(t_iter);
        record_iter(iter, R.energy, s.max_upd, R.num_active, false, st);
        R.iterations = iter;
        break;
      }
      R.lambda *= 10.0;  // :787-789
      ++R.rejected;
      if (++R.bad >= R.cfg.max_bad_steps) break;
    }
  }
  if (!accepted) {  // :792-798
    if (!R.converged) {
      R.diverged = true;
      R.message = "Diverged: " + std::to_string(R.bad) + " consecutive rejected damped steps";
    }
    R.done = true;
    return true;
  }
  const double max_upd = s.max_upd;  // :800-801
  const bool zero_grad = max_upd < R.cfg.threshold_px ? grad_is_zero(b0) : false;
  commit_candidate();
  R.energy = s.energy;
  R.num_active = static_cast<int64_t>(s.num_active);
  R.cur = b1;
  R.rhs_lambda = lam_next;
  R.gnorm2_n = s.gnorm2_n;
  R.wall_ms += ms_since(t_iter);
  record_iter(iter, R.energy, max_upd, R.num_active, true, st);
  R.iterations = iter;
  if (max_upd < R.cfg.threshold_px) {  // :826-832
    R.converged = true;
    if (zero_grad) R.message = "no-progress convergence: zero gradient";
    R.done = true;
    return true;
  }
  return false;
}

void Engine::end(pba_report* rep) {
  if (!run_.active) throw PbaError(PBA_E_STATE, "no active run");
  run_.active = false;
  if (!rep) return;
  const Run& R = run_;
  rep->converged = R.converged;
  rep->diverged = R.diverged;
  rep->iterations = R.iterations;
  rep->hessian_builds = R.ic ? ic_.builds : R.fc_builds;
  rep->hessian_factorizations = R.ic ? ic_.factorizations : R.fc_factorizations;
  rep->rejected_steps = R.rejected;
  rep->final_energy = R.energy;
  rep->total_wall_ms = R.wall_ms;
  rep->masked_residuals = R.initial_active - R.num_active;
  if (rep->final_R || rep->final_t) download_poses(pose_cur_, rep->final_R, rep->final_t);
  if (rep->final_inv_depths) download_depths_user(d_cur_, rep->final_inv_depths);
  const int n = std::min<int>(static_cast<int>(R.iters.size()), std::max(rep->iters_capacity, 0));
  rep->num_iters = n;
  for (int i = 0; i < n; ++i) {
    if (rep->iters) rep->iters[i] = R.iters[i];
    if (R.cfg.record_snapshots) {
      if (rep->snap_R) std::memcpy(rep->snap_R + 9 * static_cast<size_t>(F_) * i, &R.snapR[9 * static_cast<size_t>(F_) * i], 9 * F_ * sizeof(double));
      if (rep->snap_t) std::memcpy(rep->snap_t + 3 * static_cast<size_t>(F_) * i, &R.snapT[3 * static_cast<size_t>(F_) * i], 3 * F_ * sizeof(double));
      if (rep->snap_d) std::memcpy(rep->snap_d + static_cast<size_t>(N_) * i, &R.snapD[static_cast<size_t>(N_) * i], N_ * sizeof(double));
    }
  }
  std::snprintf(rep->message, sizeof(rep->message), "%s", R.message.c_str());
}

}  // namespace pba_b200
