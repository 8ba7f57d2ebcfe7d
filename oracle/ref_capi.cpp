// C API over the UNMODIFIED reference (/root/reference/proj/src/*.cpp compiled against
// oracle/ref_shim) — TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile's `ref` target into
// oracle/_ref/libpba_ref.so; never linked by the product.
//
// Mirrors oracle/pba_oracle_c.h (and hence include/pba_gpu.h) call for call, prefix pba_ref_, so the
// parity tests can drive the reference, the restated oracle and the GPU library through the same
// Python Handle.  Every call goes to the reference's own public API (solver.hpp:107-197,
// synth.hpp:62-80, geometry.hpp:50-128); IcSolver's private factorize / solve_step are reached
// through the reference's own test hook `friend class SolverTestAccess` (solver.hpp:136).
//
// The reference stores the dense N x F x P problem (solver.hpp:101), so a problem with an observation
// list is accepted only when the list is the dense one (every point in every frame).
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../include/pba_gpu.h"
#include "pba/errors.hpp"
#include "pba/geometry.hpp"
#include "pba/image.hpp"
#include "pba/solver.hpp"
#include "pba/synth.hpp"
#include "pba_oracle_c.h"  // pba_oracle_scene_spec

namespace pba {
// The reference's test-access hook (solver.hpp:136).
class SolverTestAccess {
 public:
  static void factorize(IcSolver& s, double lambda) { s.factorize(lambda); }
  static Eigen::VectorXd solve_step(IcSolver& s, const Eigen::VectorXd& g) { return s.solve_step(g); }
  static const std::vector<Pose>& pose0(const IcSolver& s) { return s.pose0_; }
  static const std::vector<double>& d0(const IcSolver& s) { return s.d0_; }
  static double lambda(const IcSolver& s) { return s.lambda_; }
};
}  // namespace pba

using namespace pba;

struct pba_ref_handle {
  ProblemState st;
  std::unique_ptr<IcSolver> ic;
  std::string last_error;
};

namespace {

template <typename Fn>
int guarded(pba_ref_handle* h, Fn&& fn) {
  try {
    fn();
    return PBA_OK;
  } catch (const EmptyProblem& e) {
    if (h) h->last_error = e.what();
    return PBA_E_EMPTY_PROBLEM;
  } catch (const OutOfBounds& e) {
    if (h) h->last_error = e.what();
    return PBA_E_OUT_OF_BOUNDS;
  } catch (const InvalidDepth& e) {
    if (h) h->last_error = e.what();
    return PBA_E_INVALID_DEPTH;
  } catch (const DegenerateDepth& e) {
    if (h) h->last_error = e.what();
    return PBA_E_DEGENERATE_DEPTH;
  } catch (const SpecInfeasible& e) {
    if (h) h->last_error = e.what();
    return PBA_E_SPEC_INFEASIBLE;
  } catch (const Error& e) {
    if (h) h->last_error = e.what();
    const std::string w = e.what();
    return w.rfind("SingularHessian", 0) == 0 ? PBA_E_SINGULAR_HESSIAN : PBA_E_ARG;
  } catch (const std::exception& e) {
    if (h) h->last_error = e.what();
    return PBA_E_ARG;
  }
}

Image to_image(const pba_image& d) {
  Image img(d.width, d.height, Intrinsics{d.fx, d.fy, d.cx, d.cy});
  for (int v = 0; v < d.height; ++v)
    for (int u = 0; u < d.width; ++u) img.at(u, v) = static_cast<double>(d.data[static_cast<size_t>(v) * d.width + u]);
  return img;
}

Pose to_pose(const double* R, const double* t) {
  Pose p;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p.R(i, j) = R[3 * i + j];
  p.t = Vec3(t[0], t[1], t[2]);
  return p;
}

void from_pose(const Pose& p, double* R, double* t) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[3 * i + j] = p.R(i, j);
  for (int i = 0; i < 3; ++i) t[i] = p.t(i);
}

SolverConfig to_config(const pba_config* c) {
  SolverConfig s;
  if (!c) return s;
  s.gamma = c->gamma;
  s.threshold_px = c->threshold_px;
  s.max_iters = c->max_iters;
  s.lambda0 = c->lambda0;
  s.max_bad_steps = c->max_bad_steps;
  s.normalize_depth_gauge = c->normalize_depth_gauge != 0;
  s.refresh_ic_hessian = c->refresh_ic_hessian != 0;
  s.record_snapshots = c->record_snapshots != 0;
  return s;
}

// SolveReport -> pba_report.  The reference's IterationStats has no accepted flag: an iteration is a
// rejection-terminated one only when it is the last and the run stopped on
// "converged: sub-threshold step rejected" (solver.cpp:573-595); num_active is not recorded (-1).
void fill_report(const SolveReport& r, int F, int N, pba_report* out) {
  out->converged = r.converged;
  out->diverged = r.diverged;
  out->iterations = r.iterations;
  out->hessian_builds = r.hessian_builds;
  out->hessian_factorizations = r.hessian_factorizations;
  out->rejected_steps = r.rejected_steps;
  out->final_energy = r.final_energy;
  out->total_wall_ms = r.total_wall_ms;
  out->masked_residuals = r.masked_residuals;
  if (out->final_R && out->final_t)
    for (int f = 0; f < F; ++f) from_pose(r.final_poses[f], out->final_R + 9 * f, out->final_t + 3 * f);
  if (out->final_inv_depths)
    for (int n = 0; n < N; ++n) out->final_inv_depths[n] = r.final_inv_depths[n];
  const bool last_rejected = r.message == "converged: sub-threshold step rejected";
  out->num_iters = 0;
  for (size_t k = 0; k < r.iters.size(); ++k) {
    const IterationStats& it = r.iters[k];
    if (out->num_iters >= out->iters_capacity) break;
    const int i = out->num_iters++;
    if (out->iters) {
      pba_iter_stats& s = out->iters[i];
      s.iter = it.iter;
      s.energy = it.energy;
      s.max_update_px = it.max_update_px;
      s.wall_ms = it.wall_ms;
      s.hessian_builds = it.hessian_builds;
      s.hessian_factorizations = it.hessian_factorizations;
      s.num_active = -1;
      s.accepted = (last_rejected && k + 1 == r.iters.size()) ? 0 : 1;
    }
    if (!it.poses.empty() && out->snap_R && out->snap_t)
      for (int f = 0; f < F; ++f)
        from_pose(it.poses[f], out->snap_R + (static_cast<size_t>(i) * F + f) * 9,
                  out->snap_t + (static_cast<size_t>(i) * F + f) * 3);
    if (!it.inv_depths.empty() && out->snap_d)
      for (int n = 0; n < N; ++n) out->snap_d[static_cast<size_t>(i) * N + n] = it.inv_depths[n];
  }
  std::snprintf(out->message, sizeof(out->message), "%s", r.message.c_str());
}

bool is_dense_list(int F, int N, const int64_t* ptr, const int32_t* frame) {
  if (!ptr) return true;
  for (int n = 0; n <= N; ++n)
    if (ptr[n] != static_cast<int64_t>(n) * F) return false;
  for (int n = 0; n < N; ++n)
    for (int f = 0; f < F; ++f)
      if (frame[static_cast<size_t>(n) * F + f] != f) return false;
  return true;
}

// BlockHessian from the observation layout (unobserved (n, f) blocks are exact zeros, which the
// reference's Schur loops skip: solver.cpp:181, 185).
BlockHessian block_hessian(int F, int N, const int64_t* ptr, const int32_t* frame, const double* pp,
                           const double* dd, const double* pd) {
  BlockHessian H;
  H.F = F;
  H.N = N;
  H.pose_pose.assign(F, Mat66::Zero());
  H.depth_depth.assign(N, 0.0);
  H.pose_depth.assign(static_cast<size_t>(N) * F, Eigen::Matrix<double, 6, 1>::Zero());
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) H.pose_pose[f](i, j) = pp[36 * f + 6 * i + j];
  for (int n = 0; n < N; ++n) H.depth_depth[n] = dd[n];
  for (int n = 0; n < N; ++n) {
    const int64_t a = ptr ? ptr[n] : static_cast<int64_t>(n) * F;
    const int64_t b = ptr ? ptr[n + 1] : static_cast<int64_t>(n + 1) * F;
    for (int64_t o = a; o < b; ++o) {
      const int f = ptr ? frame[o] : static_cast<int>(o - a);
      for (int i = 0; i < 6; ++i) H.pose_depth[static_cast<size_t>(n) * F + f](i) = pd[6 * o + i];
    }
  }
  return H;
}

}  // namespace

extern "C" {

int pba_ref_create(const pba_problem* p, pba_ref_handle** out) {
  *out = nullptr;
  auto h = std::make_unique<pba_ref_handle>();
  const int rc = guarded(h.get(), [&] {
    if (!is_dense_list(p->num_frames, p->num_points, p->obs_ptr, p->obs_frame))
      throw Error("the reference stores the dense N x F x P problem (solver.hpp:101); observation lists "
                  "other than the dense one are not expressible");
    ProblemState& st = h->st;
    st.ref = to_image(p->ref);
    for (int f = 0; f < p->num_frames; ++f) {
      st.targets.push_back(to_image(p->targets[f]));
      st.poses.push_back(to_pose(p->pose_R + 9 * f, p->pose_t + 3 * f));
    }
    for (int n = 0; n < p->num_points; ++n) {
      st.anchors_px.emplace_back(p->anchors_px[2 * n], p->anchors_px[2 * n + 1]);
      st.inv_depths.push_back(p->inv_depths[n]);
    }
    st.patch.offsets.clear();
    for (int k = 0; k < p->pattern_size; ++k) st.patch.offsets.emplace_back(p->pattern[2 * k], p->pattern[2 * k + 1]);
  });
  if (rc == PBA_OK) *out = h.release();
  return rc;
}

void pba_ref_destroy(pba_ref_handle* h) { delete h; }
const char* pba_ref_last_error(const pba_ref_handle* h) { return h ? h->last_error.c_str() : ""; }
int64_t pba_ref_num_observations(const pba_ref_handle* h) {
  return static_cast<int64_t>(h->st.num_points()) * h->st.num_frames();
}

int pba_ref_set_params(pba_ref_handle* h, const double* R, const double* t, const double* d) {
  return guarded(h, [&] {
    for (int f = 0; f < h->st.num_frames(); ++f) h->st.poses[f] = to_pose(R + 9 * f, t + 3 * f);
    for (int n = 0; n < h->st.num_points(); ++n) h->st.inv_depths[n] = d[n];
    h->ic.reset();
  });
}

int pba_ref_get_params(pba_ref_handle* h, double* R, double* t, double* d) {
  return guarded(h, [&] {
    for (int f = 0; f < h->st.num_frames(); ++f) from_pose(h->st.poses[f], R + 9 * f, t + 3 * f);
    for (int n = 0; n < h->st.num_points(); ++n) d[n] = h->st.inv_depths[n];
  });
}

int pba_ref_energy(pba_ref_handle* h, double gamma, const uint8_t* mask, pba_energy_result* out,
                   double* residuals, uint8_t* active) {
  return guarded(h, [&] {
    std::vector<uint8_t> m;
    const size_t n = static_cast<size_t>(h->st.num_points()) * h->st.num_frames() * h->st.patch.offsets.size();
    if (mask) m.assign(mask, mask + n);
    const EnergyResult e = energy_eval(h->st, HuberLoss{gamma}, mask ? &m : nullptr);
    out->energy = e.energy;
    out->num_active = e.num_active;
    out->num_out_of_bounds = e.num_out_of_bounds;
    if (residuals) std::memcpy(residuals, e.residuals.data(), n * sizeof(double));
    if (active) std::memcpy(active, e.active.data(), n);
  });
}

int pba_ref_ic_build(pba_ref_handle* h, const pba_config* cfg) {
  return guarded(h, [&] {
    h->ic = std::make_unique<IcSolver>(h->st, to_config(cfg));
    h->ic->build();
  });
}

static IcSolver& built(pba_ref_handle* h) {
  if (!h->ic) throw Error("IcSolver::build has not been called");
  return *h->ic;
}

int pba_ref_ic_gradient(pba_ref_handle* h, double* g) {
  return guarded(h, [&] {
    const Eigen::VectorXd v = built(h).gradient();
    for (Eigen::Index i = 0; i < v.size(); ++i) g[i] = v(i);
  });
}

int pba_ref_ic_compute_step(pba_ref_handle* h, double* dx) {
  return guarded(h, [&] {
    const Eigen::VectorXd v = built(h).compute_step();
    for (Eigen::Index i = 0; i < v.size(); ++i) dx[i] = v(i);
  });
}

int pba_ref_ic_solve_step(pba_ref_handle* h, const double* g, double* dx) {
  return guarded(h, [&] {
    IcSolver& s = built(h);
    const int dim = 6 * h->st.num_frames() + h->st.num_points();
    Eigen::VectorXd gv(dim);
    for (int i = 0; i < dim; ++i) gv(i) = g[i];
    const Eigen::VectorXd v = SolverTestAccess::solve_step(s, gv);
    for (int i = 0; i < dim; ++i) dx[i] = v(i);
  });
}

int pba_ref_ic_factorize(pba_ref_handle* h, double lambda) {
  return guarded(h, [&] { SolverTestAccess::factorize(built(h), lambda); });
}

int pba_ref_ic_hessian(pba_ref_handle* h, double* pp, double* dd, double* pd, double* lambda) {
  return guarded(h, [&] {
    const BlockHessian& H = built(h).hessian();
    for (int f = 0; f < H.F; ++f)
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) pp[36 * f + 6 * i + j] = H.pose_pose[f](i, j);
    for (int n = 0; n < H.N; ++n) dd[n] = H.depth_depth[n];
    for (size_t b = 0; b < H.pose_depth.size(); ++b)
      for (int i = 0; i < 6; ++i) pd[6 * b + i] = H.pose_depth[b](i);
    if (lambda) *lambda = H.lambda;
  });
}

int pba_ref_warning_count(const pba_ref_handle* h) {
  return h->ic ? static_cast<int>(h->ic->warnings().size()) : 0;
}

int pba_ref_warning(const pba_ref_handle* h, int i, char* buf, int len) {
  if (!h->ic || i < 0 || i >= static_cast<int>(h->ic->warnings().size())) return PBA_E_ARG;
  std::snprintf(buf, static_cast<size_t>(len), "%s", h->ic->warnings()[i].c_str());
  return PBA_OK;
}

int64_t pba_ref_warnings_text(const pba_ref_handle* h, char* buf, int64_t len) {
  std::string all;
  if (h->ic)
    for (const std::string& w : h->ic->warnings()) {
      if (!all.empty()) all += '\n';
      all += w;
    }
  if (buf && len > 0) {
    const size_t n = std::min<size_t>(all.size(), static_cast<size_t>(len - 1));
    std::memcpy(buf, all.data(), n);
    buf[n] = 0;
  }
  return static_cast<int64_t>(all.size());
}

int pba_ref_ic_run(pba_ref_handle* h, const pba_config* cfg, pba_report* rep) {
  return guarded(h, [&] {
    const SolveReport r = ic_solve(h->st, to_config(cfg));
    fill_report(r, h->st.num_frames(), h->st.num_points(), rep);
  });
}

int pba_ref_fc_run(pba_ref_handle* h, const pba_config* cfg, pba_report* rep) {
  return guarded(h, [&] {
    const SolveReport r = fc_solve(h->st, to_config(cfg));
    fill_report(r, h->st.num_frames(), h->st.num_points(), rep);
  });
}

static int free_solve(bool dense, int32_t F, int32_t N, const int64_t* ptr, const int32_t* frame, const double* pp,
                      const double* dd, const double* pd, const double* g, double lambda, double* dx) {
  return guarded(nullptr, [&] {
    const BlockHessian H = block_hessian(F, N, ptr, frame, pp, dd, pd);
    Eigen::VectorXd gv(6 * F + N);
    for (int i = 0; i < 6 * F + N; ++i) gv(i) = g[i];
    const Eigen::VectorXd v = dense ? solve_normal_equations_dense(H, gv, lambda)
                                    : solve_normal_equations_schur(H, gv, lambda);
    for (int i = 0; i < 6 * F + N; ++i) dx[i] = v(i);
  });
}

int pba_ref_solve_normal_equations_schur(int32_t F, int32_t N, const int64_t* ptr, const int32_t* frame,
                                         const double* pp, const double* dd, const double* pd, const double* g,
                                         double lambda, double* dx) {
  return free_solve(false, F, N, ptr, frame, pp, dd, pd, g, lambda, dx);
}

int pba_ref_solve_normal_equations_dense(int32_t F, int32_t N, const int64_t* ptr, const int32_t* frame,
                                         const double* pp, const double* dd, const double* pd, const double* g,
                                         double lambda, double* dx) {
  return free_solve(true, F, N, ptr, frame, pp, dd, pd, g, lambda, dx);
}

// Candidate update by the reference's geometry (solver.cpp:544-560 IC with the build's p0 and
// d0 = 1 for poses; solver.cpp:744-750 FC), without touching the problem parameters.
int pba_ref_apply_update(pba_ref_handle* h, int mode, const double* dx, double* R_out, double* t_out,
                         double* d_out, int* invalid) {
  return guarded(h, [&] {
    const int F = h->st.num_frames(), N = h->st.num_points();
    *invalid = 0;
    try {
      for (int f = 0; f < F; ++f) {
        Vec6 d6;
        for (int i = 0; i < 6; ++i) d6(i) = dx[6 * f + i];
        Pose next;
        if (mode == 0) {
          const IcSolver& s = built(h);
          ProxyConstants pc;
          pc.R0 = SolverTestAccess::pose0(s)[f].R;
          pc.t0 = SolverTestAccess::pose0(s)[f].t;
          pc.d0 = 1.0;
          Vec7 dp = Vec7::Zero();
          dp.head<6>() = d6;
          next = apply_ic_update(h->st.poses[f], 1.0, pc, dp).first;
        } else {
          next = pose_boxplus(h->st.poses[f], d6);
        }
        from_pose(next, R_out + 9 * f, t_out + 3 * f);
      }
      for (int n = 0; n < N; ++n) {
        const double dd = dx[6 * F + n];
        if (mode == 0) {
          ProxyConstants pc;
          pc.d0 = SolverTestAccess::d0(built(h))[n];
          Vec7 dp = Vec7::Zero();
          dp(6) = dd;
          d_out[n] = apply_ic_update(Pose{}, h->st.inv_depths[n], pc, dp).second;
        } else {
          d_out[n] = h->st.inv_depths[n] + dd;
          if (d_out[n] <= 0.0) *invalid = 1;
        }
      }
    } catch (const InvalidDepth&) {
      *invalid = 1;
    }
  });
}

// ---- reference scene generator (synth.hpp:14-80) ------------------------------------------------
void pba_ref_scene_spec_default(pba_oracle_scene_spec* s) {
  const SceneSpec d;
  s->width = d.width;
  s->height = d.height;
  s->fx = d.intrinsics.fx;
  s->fy = d.intrinsics.fy;
  s->cx = d.intrinsics.cx;
  s->cy = d.intrinsics.cy;
  s->octaves = d.texture.octaves;
  s->base_wavelength_px = d.texture.base_wavelength_px;
  s->lo = d.texture.lo;
  s->hi = d.texture.hi;
  s->geometry_kind = d.geometry.kind == GeometrySpec::Kind::Plane ? 0 : 1;
  s->base_depth = d.geometry.base_depth;
  s->amplitude = d.geometry.amplitude;
  s->wavelength_px = d.geometry.wavelength_px;
  s->trajectory_kind = d.trajectory.kind == TrajectorySpec::Kind::Orbit ? 0 : 1;
  s->frames = d.trajectory.frames;
  s->span_deg = d.trajectory.span_deg;
  for (int i = 0; i < 3; ++i) s->extent[i] = d.trajectory.extent(i);
  s->num_points = d.num_points;
  s->patch_radius = d.patch_radius;
  s->seed = d.seed;
  s->supersample = d.supersample;
}

int pba_ref_render_sequence(const pba_oracle_scene_spec* s, double* ref, double* targets, double* R, double* t,
                            double* anchors, double* inv_depths, char* err, int errlen) {
  pba_ref_handle tmp;
  const int rc = guarded(&tmp, [&] {
    SceneSpec spec;
    spec.width = s->width;
    spec.height = s->height;
    spec.intrinsics = Intrinsics{s->fx, s->fy, s->cx, s->cy};
    spec.texture.octaves = s->octaves;
    spec.texture.base_wavelength_px = s->base_wavelength_px;
    spec.texture.lo = s->lo;
    spec.texture.hi = s->hi;
    spec.geometry.kind = s->geometry_kind == 0 ? GeometrySpec::Kind::Plane : GeometrySpec::Kind::Heightfield;
    spec.geometry.base_depth = s->base_depth;
    spec.geometry.amplitude = s->amplitude;
    spec.geometry.wavelength_px = s->wavelength_px;
    spec.trajectory.kind = s->trajectory_kind == 0 ? TrajectorySpec::Kind::Orbit : TrajectorySpec::Kind::Dolly;
    spec.trajectory.frames = s->frames;
    spec.trajectory.span_deg = s->span_deg;
    spec.trajectory.extent = Vec3(s->extent[0], s->extent[1], s->extent[2]);
    spec.num_points = s->num_points;
    spec.patch_radius = s->patch_radius;
    spec.seed = s->seed;
    spec.supersample = s->supersample;
    const RenderedScene sc = render_sequence(spec);
    const size_t WH = static_cast<size_t>(spec.width) * spec.height;
    for (int v = 0; v < spec.height; ++v)
      for (int u = 0; u < spec.width; ++u) ref[static_cast<size_t>(v) * spec.width + u] = sc.ref.at(u, v);
    for (int f = 0; f < spec.trajectory.frames; ++f) {
      for (int v = 0; v < spec.height; ++v)
        for (int u = 0; u < spec.width; ++u)
          targets[f * WH + static_cast<size_t>(v) * spec.width + u] = sc.targets[f].at(u, v);
      from_pose(sc.poses[f], R + 9 * f, t + 3 * f);
    }
    for (int n = 0; n < spec.num_points; ++n) {
      anchors[2 * n] = sc.anchors_px[n].x();
      anchors[2 * n + 1] = sc.anchors_px[n].y();
      inv_depths[n] = sc.inv_depths[n];
    }
  });
  if (rc != PBA_OK && err && errlen > 0) std::snprintf(err, static_cast<size_t>(errlen), "%s", tmp.last_error.c_str());
  return rc;
}

int pba_ref_perturb_parameters(int32_t F, double* R, double* t, int32_t N, double* d, double sigma, uint64_t seed) {
  return guarded(nullptr, [&] {
    std::vector<Pose> poses;
    for (int f = 0; f < F; ++f) poses.push_back(to_pose(R + 9 * f, t + 3 * f));
    std::vector<double> depths(d, d + N);
    perturb_parameters(poses, depths, sigma, seed);
    for (int f = 0; f < F; ++f) from_pose(poses[f], R + 9 * f, t + 3 * f);
    for (int n = 0; n < N; ++n) d[n] = depths[n];
  });
}

}  // extern "C"
