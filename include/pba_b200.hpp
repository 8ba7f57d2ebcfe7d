// pba_b200.hpp — header-only C++ mirror of the reference solver API
// (/root/reference/proj/include/pba/solver.hpp:18-197, errors.hpp:9-40) over the C ABI
// of pba_gpu.h.  Same class / function names, argument meaning and exception classes,
// without Eigen: poses are std::array<double, 9> (row-major R) + std::array<double, 3>.
// Link with paper_1704_06967_b200/lib/libpba_gpu.so.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pba_gpu.h"

namespace pba_b200 {

// ---- errors.hpp:9-40 ----
struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct DegenerateDepth : Error { using Error::Error; };
struct InvalidDepth : Error { using Error::Error; };
struct OutOfBounds : Error { using Error::Error; };
struct EmptyProblem : Error { using Error::Error; };
struct SpecInfeasible : Error { using Error::Error; };

inline void throw_status(int rc, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (rc) {
    case PBA_OK: return;
    case PBA_E_EMPTY_PROBLEM: throw EmptyProblem(m);
    case PBA_E_OUT_OF_BOUNDS: throw OutOfBounds(m);
    case PBA_E_INVALID_DEPTH: throw InvalidDepth(m);
    case PBA_E_DEGENERATE_DEPTH: throw DegenerateDepth(m);
    case PBA_E_SPEC_INFEASIBLE: throw SpecInfeasible(m);
    default: throw Error(m);  // includes "SingularHessian: ..." (solver.cpp:192,401)
  }
}

// ---- data model (solver.hpp:18-54, image.hpp:14-80) ----
struct Intrinsics { double fx{1.0}, fy{1.0}, cx{0.0}, cy{0.0}; };
struct Image {
  int width{0}, height{0};
  Intrinsics K{};
  std::vector<float> data;  // row-major fp32
};
struct Pose {
  std::array<double, 9> R{1, 0, 0, 0, 1, 0, 0, 0, 1};
  std::array<double, 3> t{0, 0, 0};
};
struct HuberLoss { double gamma{0.03}; };
struct ProblemState {
  Image ref;
  std::vector<Image> targets;
  std::vector<Pose> poses;
  std::vector<std::array<double, 2>> anchors_px;
  std::vector<double> inv_depths;
  std::vector<std::array<int32_t, 2>> pattern{{0, 0}, {-1, -1}, {0, -1}, {1, -1}, {-1, 0},
                                              {1, 0},  {-1, 1},  {0, 1},  {1, 1}};  // square(1)
  std::vector<int64_t> obs_ptr;     // extension: visibility list (empty = dense)
  std::vector<int32_t> obs_frame;
  int num_frames() const { return static_cast<int>(targets.size()); }
  int num_points() const { return static_cast<int>(anchors_px.size()); }
};
struct SolverConfig {
  double gamma{0.03};
  double threshold_px{5e-3};
  int max_iters{200};
  double lambda0{1e-6};
  int max_bad_steps{8};
  bool normalize_depth_gauge{true};
  bool refresh_ic_hessian{false};
  bool record_snapshots{false};
  pba_config c() const {
    return pba_config{gamma, threshold_px, max_iters, lambda0, max_bad_steps, normalize_depth_gauge ? 1 : 0,
                      refresh_ic_hessian ? 1 : 0, record_snapshots ? 1 : 0};
  }
};
struct BlockHessian {
  int F{0}, N{0};
  std::vector<std::array<double, 36>> pose_pose;
  std::vector<double> depth_depth;
  std::vector<std::array<double, 6>> pose_depth;  // observation order (dense: n*F + f)
  double lambda{0.0};
};
struct IterationStats {
  int iter{0};
  double energy{0.0}, max_update_px{0.0}, wall_ms{0.0};
  int hessian_builds{0}, hessian_factorizations{0};
  std::vector<Pose> poses;
  std::vector<double> inv_depths;
};
struct SolveReport {
  std::vector<IterationStats> iters;
  bool converged{false}, diverged{false};
  int iterations{0}, hessian_builds{0}, hessian_factorizations{0}, rejected_steps{0};
  double final_energy{0.0}, total_wall_ms{0.0};
  int64_t masked_residuals{0};
  std::vector<Pose> final_poses;
  std::vector<double> final_inv_depths;
  std::vector<std::string> warnings;
  std::string message;
};
struct EnergyResult {
  double energy{0.0};
  std::vector<double> residuals;
  std::vector<uint8_t> active;
  int64_t num_active{0}, num_out_of_bounds{0};
};

namespace detail {
// every warning in one call (pba_gpu_warnings_text): large problems can carry one per point
inline std::vector<std::string> all_warnings(const pba_handle* h) {
  std::vector<std::string> w;
  if (pba_gpu_warning_count(h) == 0) return w;
  const int64_t n = pba_gpu_warnings_text(h, nullptr, 0);
  std::string buf(static_cast<size_t>(n) + 1, '\0');
  pba_gpu_warnings_text(h, buf.data(), n + 1);
  buf.resize(static_cast<size_t>(n));
  size_t a = 0;
  while (a <= buf.size()) {
    const size_t b = buf.find('\n', a);
    w.emplace_back(buf.substr(a, b == std::string::npos ? std::string::npos : b - a));
    if (b == std::string::npos) break;
    a = b + 1;
  }
  return w;
}
struct Handle {
  pba_handle* h{nullptr};
  int F{0}, N{0}, P{0};
  int64_t NO{0};
  explicit Handle(const ProblemState& st) {
    std::vector<pba_image> tg;
    for (const Image& im : st.targets)
      tg.push_back(pba_image{im.width, im.height, im.K.fx, im.K.fy, im.K.cx, im.K.cy, im.data.data()});
    std::vector<double> R, t, an;
    for (const Pose& p : st.poses) {
      R.insert(R.end(), p.R.begin(), p.R.end());
      t.insert(t.end(), p.t.begin(), p.t.end());
    }
    for (const auto& a : st.anchors_px) an.insert(an.end(), a.begin(), a.end());
    std::vector<int32_t> pat;
    for (const auto& o : st.pattern) pat.insert(pat.end(), o.begin(), o.end());
    pba_problem p{};
    p.ref = pba_image{st.ref.width, st.ref.height, st.ref.K.fx, st.ref.K.fy, st.ref.K.cx, st.ref.K.cy,
                      st.ref.data.data()};
    p.num_frames = st.num_frames();
    p.targets = tg.data();
    p.pose_R = R.data();
    p.pose_t = t.data();
    p.num_points = st.num_points();
    p.anchors_px = an.data();
    p.inv_depths = st.inv_depths.data();
    p.pattern_size = static_cast<int32_t>(st.pattern.size());
    p.pattern = pat.data();
    if (!st.obs_ptr.empty()) {
      p.obs_ptr = st.obs_ptr.data();
      p.obs_frame = st.obs_frame.data();
    }
    throw_status(pba_gpu_create(&p, &h), pba_gpu_last_error(nullptr));
    F = st.num_frames();
    N = st.num_points();
    P = static_cast<int>(st.pattern.size());
    NO = pba_gpu_num_observations(h);
  }
  ~Handle() { pba_gpu_destroy(h); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  void check(int rc) const { throw_status(rc, pba_gpu_last_error(h)); }

  SolveReport report(bool ic, const pba_config* cfg, int capacity, bool snaps) {
    std::vector<double> R(9 * F), t(3 * F), d(N);
    std::vector<pba_iter_stats> its(capacity > 0 ? capacity : 1);
    std::vector<double> sR, sT, sD;
    pba_report rep{};
    rep.final_R = R.data();
    rep.final_t = t.data();
    rep.final_inv_depths = d.data();
    rep.iters = its.data();
    rep.iters_capacity = capacity;
    if (snaps) {
      sR.resize(static_cast<size_t>(capacity) * 9 * F);
      sT.resize(static_cast<size_t>(capacity) * 3 * F);
      sD.resize(static_cast<size_t>(capacity) * N);
      rep.snap_R = sR.data();
      rep.snap_t = sT.data();
      rep.snap_d = sD.data();
    }
    check(ic ? pba_gpu_ic_run(h, cfg, &rep) : pba_gpu_fc_run(h, cfg, &rep));
    SolveReport out;
    out.converged = rep.converged;
    out.diverged = rep.diverged;
    out.iterations = rep.iterations;
    out.hessian_builds = rep.hessian_builds;
    out.hessian_factorizations = rep.hessian_factorizations;
    out.rejected_steps = rep.rejected_steps;
    out.final_energy = rep.final_energy;
    out.total_wall_ms = rep.total_wall_ms;
    out.masked_residuals = rep.masked_residuals;
    out.message = rep.message;
    auto poses_at = [&](const double* Rp, const double* tp) {
      std::vector<Pose> v(F);
      for (int f = 0; f < F; ++f) {
        for (int i = 0; i < 9; ++i) v[f].R[i] = Rp[9 * f + i];
        for (int i = 0; i < 3; ++i) v[f].t[i] = tp[3 * f + i];
      }
      return v;
    };
    out.final_poses = poses_at(R.data(), t.data());
    out.final_inv_depths = d;
    for (int i = 0; i < rep.num_iters; ++i) {
      IterationStats s;
      s.iter = its[i].iter;
      s.energy = its[i].energy;
      s.max_update_px = its[i].max_update_px;
      s.wall_ms = its[i].wall_ms;
      s.hessian_builds = its[i].hessian_builds;
      s.hessian_factorizations = its[i].hessian_factorizations;
      if (snaps) {
        s.poses = poses_at(&sR[static_cast<size_t>(i) * 9 * F], &sT[static_cast<size_t>(i) * 3 * F]);
        s.inv_depths.assign(sD.begin() + static_cast<size_t>(i) * N, sD.begin() + static_cast<size_t>(i + 1) * N);
      }
      out.iters.push_back(std::move(s));
    }
    out.warnings = all_warnings(h);
    return out;
  }
};
}  // namespace detail

// energy_eval (solver.hpp:110-111)
inline EnergyResult energy_eval(const ProblemState& state, const HuberLoss& huber,
                                const std::vector<uint8_t>* mask = nullptr) {
  detail::Handle h(state);
  EnergyResult r;
  r.residuals.resize(static_cast<size_t>(h.NO) * h.P);
  r.active.resize(r.residuals.size());
  pba_energy_result e{};
  h.check(pba_gpu_energy(h.h, huber.gamma, mask ? mask->data() : nullptr, &e, r.residuals.data(), r.active.data()));
  r.energy = e.energy;
  r.num_active = e.num_active;
  r.num_out_of_bounds = e.num_out_of_bounds;
  return r;
}

// IcSolver (solver.hpp:115-169)
class IcSolver {
 public:
  explicit IcSolver(const ProblemState& state, SolverConfig config = {})
      : h_(std::make_unique<detail::Handle>(state)), cfg_(config) {}
  void build() {
    if (built_) return;
    const pba_config c = cfg_.c();
    h_->check(pba_gpu_ic_build(h_->h, &c));
    built_ = true;
  }
  std::vector<double> compute_step() {
    build();
    std::vector<double> dx(6 * h_->F + h_->N);
    h_->check(pba_gpu_ic_compute_step(h_->h, dx.data()));
    return dx;
  }
  std::vector<double> gradient() {
    build();
    std::vector<double> g(6 * h_->F + h_->N);
    h_->check(pba_gpu_ic_gradient(h_->h, g.data()));
    return g;
  }
  SolveReport run() {
    build();
    return h_->report(true, nullptr, cfg_.max_iters > 0 ? cfg_.max_iters : 1, cfg_.record_snapshots);
  }
  BlockHessian hessian() const {
    BlockHessian H;
    H.F = h_->F;
    H.N = h_->N;
    H.pose_pose.resize(H.F);
    H.depth_depth.resize(H.N);
    H.pose_depth.resize(static_cast<size_t>(h_->NO));
    h_->check(pba_gpu_ic_hessian(h_->h, H.pose_pose.empty() ? nullptr : H.pose_pose[0].data(), H.depth_depth.data(),
                                 H.pose_depth.empty() ? nullptr : H.pose_depth[0].data(), &H.lambda));
    return H;
  }
  std::vector<std::string> warnings() const { return detail::all_warnings(h_->h); }

 private:
  std::unique_ptr<detail::Handle> h_;
  SolverConfig cfg_;
  bool built_{false};
};

// FcSolver (solver.hpp:172-182)
class FcSolver {
 public:
  explicit FcSolver(const ProblemState& state, SolverConfig config = {})
      : h_(std::make_unique<detail::Handle>(state)), cfg_(config) {}
  SolveReport run() {
    const pba_config c = cfg_.c();
    return h_->report(false, &c, cfg_.max_iters > 0 ? cfg_.max_iters : 1, cfg_.record_snapshots);
  }

 private:
  std::unique_ptr<detail::Handle> h_;
  SolverConfig cfg_;
};

// ic_solve / fc_solve (solver.cpp:845-851): the drop-in for the CLI seam pba.cpp:74-77
inline SolveReport ic_solve(const ProblemState& state, const SolverConfig& config) {
  detail::Handle h(state);
  const pba_config c = config.c();
  return h.report(true, &c, config.max_iters > 0 ? config.max_iters : 1, config.record_snapshots);
}
inline SolveReport fc_solve(const ProblemState& state, const SolverConfig& config) {
  return FcSolver(state, config).run();
}

// solve_normal_equations_schur (solver.hpp:190-192)
inline std::vector<double> solve_normal_equations_schur(const BlockHessian& H, const std::vector<double>& g,
                                                        double lambda, const std::vector<int64_t>* obs_ptr = nullptr,
                                                        const std::vector<int32_t>* obs_frame = nullptr) {
  std::vector<double> dx(6 * H.F + H.N);
  const int rc = pba_gpu_solve_normal_equations_schur(
      H.F, H.N, obs_ptr ? obs_ptr->data() : nullptr, obs_frame ? obs_frame->data() : nullptr,
      H.pose_pose.empty() ? nullptr : H.pose_pose[0].data(), H.depth_depth.data(),
      H.pose_depth.empty() ? nullptr : H.pose_depth[0].data(), g.data(), lambda, dx.data());
  throw_status(rc, pba_gpu_last_error(nullptr));
  return dx;
}

// ---- joint multi-host window with per-frame affine brightness (pba_gpu_mh_*; no reference
//      counterpart: the model is stated in oracle/multihost.cpp) ----
struct MultiHostProblem {
  std::vector<Image> images;               // K frames, each with its intrinsics; frame 0 held
  std::vector<Pose> poses;                 // K: X_i = R_i X_w + t_i
  std::vector<double> affine_a, affine_b;  // K or empty (= 0)
  std::vector<int32_t> host;               // N
  std::vector<std::array<double, 2>> anchors_px;
  std::vector<double> inv_depths;
  std::vector<std::array<int32_t, 2>> pattern{{0, 0}, {-1, -1}, {0, -1}, {1, -1}, {-1, 0},
                                              {1, 0},  {-1, 1},  {0, 1},  {1, 1}};
  std::vector<int64_t> obs_ptr;            // CSR of target frames (empty = every other frame)
  std::vector<int32_t> obs_frame;
  bool optimize_affine{true};
};
struct MultiHostReport : SolveReport {
  std::vector<double> final_a, final_b;
};

inline MultiHostReport mh_fc_solve(const MultiHostProblem& p, const SolverConfig& config) {
  const int K = static_cast<int>(p.images.size()), N = static_cast<int>(p.anchors_px.size());
  std::vector<pba_image> im(K);
  std::vector<double> R(9 * static_cast<size_t>(K)), t(3 * static_cast<size_t>(K)), an(2 * static_cast<size_t>(N));
  std::vector<int32_t> pat;
  for (int f = 0; f < K; ++f) {
    const Image& g = p.images[f];
    im[f] = pba_image{g.width, g.height, g.K.fx, g.K.fy, g.K.cx, g.K.cy, g.data.data()};
    for (int i = 0; i < 9; ++i) R[9 * f + i] = p.poses[f].R[i];
    for (int i = 0; i < 3; ++i) t[3 * f + i] = p.poses[f].t[i];
  }
  for (int n = 0; n < N; ++n) {
    an[2 * n] = p.anchors_px[n][0];
    an[2 * n + 1] = p.anchors_px[n][1];
  }
  for (const auto& o : p.pattern) {
    pat.push_back(o[0]);
    pat.push_back(o[1]);
  }
  pba_mh_problem q{};
  q.num_frames = K;
  q.images = im.data();
  q.pose_R = R.data();
  q.pose_t = t.data();
  q.affine_a = p.affine_a.empty() ? nullptr : p.affine_a.data();
  q.affine_b = p.affine_b.empty() ? nullptr : p.affine_b.data();
  q.num_points = N;
  q.host = p.host.data();
  q.anchors_px = an.data();
  q.inv_depths = p.inv_depths.data();
  q.pattern_size = static_cast<int32_t>(p.pattern.size());
  q.pattern = pat.data();
  q.obs_ptr = p.obs_ptr.empty() ? nullptr : p.obs_ptr.data();
  q.obs_frame = p.obs_frame.empty() ? nullptr : p.obs_frame.data();
  q.optimize_affine = p.optimize_affine ? 1 : 0;
  pba_mh_handle* h = nullptr;
  throw_status(pba_gpu_mh_create(&q, &h), pba_gpu_mh_last_error(nullptr));
  std::unique_ptr<pba_mh_handle, void (*)(pba_mh_handle*)> guard(h, pba_gpu_mh_destroy);
  const int cap = config.max_iters > 0 ? config.max_iters : 1;
  MultiHostReport out;
  std::vector<double> Rf(9 * static_cast<size_t>(K)), tf(3 * static_cast<size_t>(K));
  out.final_inv_depths.resize(N);
  out.final_a.resize(K);
  out.final_b.resize(K);
  std::vector<pba_iter_stats> its(cap);
  pba_report rep{};
  rep.final_R = Rf.data();
  rep.final_t = tf.data();
  rep.final_inv_depths = out.final_inv_depths.data();
  rep.iters = its.data();
  rep.iters_capacity = cap;
  const pba_config c = config.c();
  throw_status(pba_gpu_mh_fc_run(h, &c, &rep, out.final_a.data(), out.final_b.data()), pba_gpu_mh_last_error(h));
  out.converged = rep.converged;
  out.diverged = rep.diverged;
  out.iterations = rep.iterations;
  out.hessian_builds = rep.hessian_builds;
  out.hessian_factorizations = rep.hessian_factorizations;
  out.rejected_steps = rep.rejected_steps;
  out.final_energy = rep.final_energy;
  out.total_wall_ms = rep.total_wall_ms;
  out.masked_residuals = rep.masked_residuals;
  out.message = rep.message;
  for (int f = 0; f < K; ++f) {
    Pose q2;
    for (int i = 0; i < 9; ++i) q2.R[i] = Rf[9 * f + i];
    for (int i = 0; i < 3; ++i) q2.t[i] = tf[3 * f + i];
    out.final_poses.push_back(q2);
  }
  for (int i = 0; i < rep.num_iters; ++i) {
    IterationStats st;
    st.iter = its[i].iter;
    st.energy = its[i].energy;
    st.max_update_px = its[i].max_update_px;
    st.wall_ms = its[i].wall_ms;
    st.hessian_builds = its[i].hessian_builds;
    st.hessian_factorizations = its[i].hessian_factorizations;
    out.iters.push_back(st);
  }
  return out;
}

}  // namespace pba_b200
