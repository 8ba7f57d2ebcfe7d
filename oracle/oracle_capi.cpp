// CPU ORACLE C API — TEST INFRASTRUCTURE ONLY (see pba_oracle.hpp).
// Exposes the oracle through the same calls as include/pba_gpu.h.
#include <cstdlib>
#include <cstring>
#include <memory>

#include "pba_oracle.hpp"
#include "pba_oracle_c.h"

using namespace oracle;

struct pba_oracle_handle {
  ProblemState st;
  std::unique_ptr<IcSolver> ic;
  std::string last_error;
};

namespace {

template <typename Fn>
int guarded(pba_oracle_handle* h, Fn&& fn) {
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
  const size_t n = static_cast<size_t>(d.width) * d.height;
  for (size_t i = 0; i < n; ++i) img.data()[i] = static_cast<double>(d.data[i]);
  return img;
}

Pose to_pose(const double* R, const double* t) {
  Pose p;
  for (int i = 0; i < 9; ++i) p.R.a[i] = R[i];
  p.t = Vec3(t[0], t[1], t[2]);
  return p;
}

void from_pose(const Pose& p, double* R, double* t) {
  for (int i = 0; i < 9; ++i) R[i] = p.R.a[i];
  t[0] = p.t.x;
  t[1] = p.t.y;
  t[2] = p.t.z;
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
  for (int f = 0; f < F; ++f)
    if (out->final_R && out->final_t) from_pose(r.final_poses[f], out->final_R + 9 * f, out->final_t + 3 * f);
  if (out->final_inv_depths)
    for (int n = 0; n < N; ++n) out->final_inv_depths[n] = r.final_inv_depths[n];
  out->num_iters = 0;
  for (const auto& it : r.iters) {
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
      s.num_active = it.num_active;
      s.accepted = it.accepted ? 1 : 0;
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

BlockHessian to_hessian(int F, int N, const int64_t* obs_ptr, const int32_t* obs_frame,
                        const double* pp, const double* dd, const double* pd) {
  BlockHessian H;
  H.F = F;
  H.N = N;
  H.obs_ptr.resize(static_cast<size_t>(N) + 1);
  if (obs_ptr) {
    for (int n = 0; n <= N; ++n) H.obs_ptr[n] = obs_ptr[n];
    H.obs_frame.assign(obs_frame, obs_frame + H.obs_ptr[N]);
  } else {
    for (int n = 0; n <= N; ++n) H.obs_ptr[n] = static_cast<int64_t>(n) * F;
    H.obs_frame.resize(static_cast<size_t>(N) * F);
    for (int n = 0; n < N; ++n)
      for (int f = 0; f < F; ++f) H.obs_frame[static_cast<size_t>(n) * F + f] = f;
  }
  H.pose_pose.resize(F);
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < 36; ++i) H.pose_pose[f][i] = pp[36 * f + i];
  H.depth_depth.assign(dd, dd + N);
  const int64_t NO = H.obs_ptr[N];
  H.pose_depth.resize(static_cast<size_t>(NO));
  for (int64_t o = 0; o < NO; ++o)
    for (int i = 0; i < 6; ++i) H.pose_depth[o][i] = pd[6 * o + i];
  return H;
}

void export_hessian(const BlockHessian& H, double* pp, double* dd, double* pd, double* lambda) {
  if (pp)
    for (int f = 0; f < H.F; ++f)
      for (int i = 0; i < 36; ++i) pp[36 * f + i] = H.pose_pose[f][i];
  if (dd)
    for (int n = 0; n < H.N; ++n) dd[n] = H.depth_depth[n];
  if (pd)
    for (size_t o = 0; o < H.pose_depth.size(); ++o)
      for (int i = 0; i < 6; ++i) pd[6 * o + i] = H.pose_depth[o][i];
  if (lambda) *lambda = H.lambda;
}

}  // namespace

extern "C" {

int pba_oracle_create(const pba_problem* p, pba_oracle_handle** out) {
  if (!p || !out) return PBA_E_ARG;
  auto h = std::make_unique<pba_oracle_handle>();
  const int rc = guarded(h.get(), [&] {
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
    for (int k = 0; k < p->pattern_size; ++k) st.patch.offsets.push_back({p->pattern[2 * k], p->pattern[2 * k + 1]});
    if (p->obs_ptr) {
      st.obs_ptr.assign(p->obs_ptr, p->obs_ptr + p->num_points + 1);
      st.obs_frame.assign(p->obs_frame, p->obs_frame + st.obs_ptr.back());
    }
  });
  if (rc != PBA_OK) return rc;
  *out = h.release();
  return PBA_OK;
}

void pba_oracle_destroy(pba_oracle_handle* h) { delete h; }

const char* pba_oracle_last_error(const pba_oracle_handle* h) { return h ? h->last_error.c_str() : ""; }

int64_t pba_oracle_num_observations(const pba_oracle_handle* h) {
  return h->st.obs_ptr.empty() ? static_cast<int64_t>(h->st.num_points()) * h->st.num_frames()
                               : h->st.obs_ptr.back();
}

int pba_oracle_set_params(pba_oracle_handle* h, const double* R, const double* t, const double* d) {
  for (int f = 0; f < h->st.num_frames(); ++f) h->st.poses[f] = to_pose(R + 9 * f, t + 3 * f);
  for (int n = 0; n < h->st.num_points(); ++n) h->st.inv_depths[n] = d[n];
  return PBA_OK;
}

int pba_oracle_get_params(pba_oracle_handle* h, double* R, double* t, double* d) {
  for (int f = 0; f < h->st.num_frames(); ++f) from_pose(h->st.poses[f], R + 9 * f, t + 3 * f);
  for (int n = 0; n < h->st.num_points(); ++n) d[n] = h->st.inv_depths[n];
  return PBA_OK;
}

int pba_oracle_energy(pba_oracle_handle* h, double gamma, const uint8_t* mask,
                      pba_energy_result* out, double* residuals, uint8_t* active) {
  return guarded(h, [&] {
    std::vector<uint8_t> m;
    const size_t sz = static_cast<size_t>(pba_oracle_num_observations(h)) * h->st.patch.offsets.size();
    if (mask) m.assign(mask, mask + sz);
    const EnergyResult r = energy_eval(h->st, HuberLoss{gamma}, mask ? &m : nullptr);
    if (out) {
      out->energy = r.energy;
      out->num_active = r.num_active;
      out->num_out_of_bounds = r.num_out_of_bounds;
    }
    if (residuals) std::memcpy(residuals, r.residuals.data(), sz * sizeof(double));
    if (active) std::memcpy(active, r.active.data(), sz);
  });
}

int pba_oracle_ic_build(pba_oracle_handle* h, const pba_config* cfg) {
  return guarded(h, [&] {
    h->ic = std::make_unique<IcSolver>(h->st, to_config(cfg));
    h->ic->build();
  });
}

static int need_ic(pba_oracle_handle* h) {
  if (!h->ic) {
    h->last_error = "IC solver not built";
    return PBA_E_STATE;
  }
  return PBA_OK;
}

int pba_oracle_ic_gradient(pba_oracle_handle* h, double* g) {
  if (int rc = need_ic(h)) return rc;
  return guarded(h, [&] {
    const auto v = h->ic->gradient();
    std::memcpy(g, v.data(), v.size() * sizeof(double));
  });
}

int pba_oracle_ic_compute_step(pba_oracle_handle* h, double* dx) {
  if (int rc = need_ic(h)) return rc;
  return guarded(h, [&] {
    const auto v = h->ic->compute_step();
    std::memcpy(dx, v.data(), v.size() * sizeof(double));
  });
}

int pba_oracle_ic_solve_step(pba_oracle_handle* h, const double* g, double* dx) {
  if (int rc = need_ic(h)) return rc;
  return guarded(h, [&] {
    const size_t n = static_cast<size_t>(6) * h->st.num_frames() + h->st.num_points();
    const auto v = h->ic->solve_step(std::vector<double>(g, g + n));
    std::memcpy(dx, v.data(), v.size() * sizeof(double));
  });
}

int pba_oracle_ic_factorize(pba_oracle_handle* h, double lambda) {
  if (int rc = need_ic(h)) return rc;
  return guarded(h, [&] { h->ic->factorize(lambda); });
}

int pba_oracle_ic_hessian(pba_oracle_handle* h, double* pp, double* dd, double* pd, double* lambda) {
  if (int rc = need_ic(h)) return rc;
  export_hessian(h->ic->hessian(), pp, dd, pd, lambda);
  return PBA_OK;
}

int pba_oracle_warning_count(const pba_oracle_handle* h) {
  return h->ic ? static_cast<int>(h->ic->warnings().size()) : 0;
}

int64_t pba_oracle_warnings_text(const pba_oracle_handle* h, char* buf, int64_t len) {
  std::string all;
  if (h->ic)
    for (const auto& w : h->ic->warnings()) {
      if (!all.empty()) all += '\n';
      all += w;
    }
  if (buf && len > 0) {
    const size_t n = std::min<size_t>(all.size(), static_cast<size_t>(len - 1));
    std::memcpy(buf, all.data(), n);
    buf[n] = '\0';
  }
  return static_cast<int64_t>(all.size());
}
// mirror of pba_gpu_warning_points: the trailing "point <n>: ..." warnings as indices
int64_t pba_oracle_warning_points(const pba_oracle_handle* h, int32_t* idx, int64_t cap) {
  if (!h->ic) return 0;
  const auto& w = h->ic->warnings();
  size_t i = w.size();
  while (i > 0 && w[i - 1].rfind("point ", 0) == 0) --i;
  const int64_t n = static_cast<int64_t>(w.size() - i);
  for (int64_t j = 0; j < n && idx && j < cap; ++j) idx[j] = std::atoi(w[i + j].c_str() + 6);
  return n;
}
int pba_oracle_warning(const pba_oracle_handle* h, int i, char* buf, int len) {
  if (!h->ic || i < 0 || i >= static_cast<int>(h->ic->warnings().size())) return PBA_E_ARG;
  std::snprintf(buf, len, "%s", h->ic->warnings()[i].c_str());
  return PBA_OK;
}

int pba_oracle_ic_run(pba_oracle_handle* h, const pba_config* cfg, pba_report* rep) {
  return guarded(h, [&] {
    h->ic = std::make_unique<IcSolver>(h->st, to_config(cfg));
    const SolveReport r = h->ic->run();
    fill_report(r, h->st.num_frames(), h->st.num_points(), rep);
  });
}

int pba_oracle_fc_build(pba_oracle_handle* h, double gamma, double* pp, double* dd, double* pd,
                        double* g) {
  return guarded(h, [&] {
    SolverConfig c;
    c.gamma = gamma;
    FcSolver fc(h->st, c);
    BlockHessian H;
    std::vector<double> gv;
    fc.build_once(H, gv);
    export_hessian(H, pp, dd, pd, nullptr);
    if (g) std::memcpy(g, gv.data(), gv.size() * sizeof(double));
  });
}

int pba_oracle_fc_run(pba_oracle_handle* h, const pba_config* cfg, pba_report* rep) {
  return guarded(h, [&] {
    const SolveReport r = FcSolver(h->st, to_config(cfg)).run();
    fill_report(r, h->st.num_frames(), h->st.num_points(), rep);
  });
}

int pba_oracle_solve_normal_equations_schur(int32_t F, int32_t N, const int64_t* obs_ptr,
                                            const int32_t* obs_frame, const double* pp,
                                            const double* dd, const double* pd, const double* g,
                                            double lambda, double* dx) {
  return guarded(nullptr, [&] {
    const BlockHessian H = to_hessian(F, N, obs_ptr, obs_frame, pp, dd, pd);
    const auto v = solve_normal_equations_schur(H, std::vector<double>(g, g + 6 * F + N), lambda);
    std::memcpy(dx, v.data(), v.size() * sizeof(double));
  });
}

int pba_oracle_solve_normal_equations_dense(int32_t F, int32_t N, const int64_t* obs_ptr,
                                            const int32_t* obs_frame, const double* pp,
                                            const double* dd, const double* pd, const double* g,
                                            double lambda, double* dx) {
  return guarded(nullptr, [&] {
    const BlockHessian H = to_hessian(F, N, obs_ptr, obs_frame, pp, dd, pd);
    const auto v = solve_normal_equations_dense(H, std::vector<double>(g, g + 6 * F + N), lambda);
    std::memcpy(dx, v.data(), v.size() * sizeof(double));
  });
}

int pba_oracle_apply_update(pba_oracle_handle* h, int mode, const double* dx, double* R_out,
                            double* t_out, double* d_out, int* invalid) {
  const int F = h->st.num_frames();
  const int N = h->st.num_points();
  if (mode == 0 && need_ic(h) != PBA_OK) return PBA_E_STATE;
  return guarded(h, [&] {
    bool valid = true;
    for (int f = 0; f < F; ++f) {
      Pose next;
      if (mode == 0) {  // solver.cpp:544-552
        ProxyConstants pc;
        pc.R0 = h->ic->pose0()[f].R;
        pc.t0 = h->ic->pose0()[f].t;
        pc.d0 = 1.0;
        Vec7 dp{};
        for (int i = 0; i < 6; ++i) dp[i] = dx[6 * f + i];
        next = apply_ic_update(h->st.poses[f], 1.0, pc, dp).first;
      } else {  // solver.cpp:744-746
        Vec6 d6;
        for (int i = 0; i < 6; ++i) d6[i] = dx[6 * f + i];
        next = pose_boxplus(h->st.poses[f], d6);
      }
      from_pose(next, R_out + 9 * f, t_out + 3 * f);
    }
    for (int n = 0; n < N; ++n) {
      double d;
      if (mode == 0) {  // solver.cpp:553-560
        d = ((h->ic->d0()[n] - dx[6 * F + n]) / h->ic->d0()[n]) * h->st.inv_depths[n];
      } else {  // solver.cpp:747-750
        d = h->st.inv_depths[n] + dx[6 * F + n];
      }
      if (d <= 0.0) valid = false;
      d_out[n] = d;
    }
    *invalid = valid ? 0 : 1;
  });
}

int pba_oracle_max_reproj_update(pba_oracle_handle* h, const double* R, const double* t,
                                 const double* d, double* px) {
  return guarded(h, [&] {
    const TemplateData tpl = build_template(h->st);
    const ObsList obs = ObsList::from(h->st);
    std::vector<Pose> np(h->st.num_frames());
    for (int f = 0; f < h->st.num_frames(); ++f) np[f] = to_pose(R + 9 * f, t + 3 * f);
    std::vector<double> nd(d, d + h->st.num_points());
    *px = max_reprojection_update_px(h->st, obs, tpl, h->st.poses, h->st.inv_depths, np, nd);
  });
}

int pba_oracle_normalize_gauge(pba_oracle_handle* h) {
  normalize_depth_gauge(h->st.poses, h->st.inv_depths);
  return PBA_OK;
}

void pba_oracle_scene_spec_default(pba_oracle_scene_spec* s) {
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
  s->extent[0] = d.trajectory.extent.x;
  s->extent[1] = d.trajectory.extent.y;
  s->extent[2] = d.trajectory.extent.z;
  s->num_points = d.num_points;
  s->patch_radius = d.patch_radius;
  s->seed = d.seed;
  s->supersample = d.supersample;
}

int pba_oracle_render_sequence(const pba_oracle_scene_spec* s, double* ref, double* targets,
                               double* R, double* t, double* anchors, double* inv_depths,
                               char* err, int errlen) {
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
  pba_oracle_handle tmp;
  const int rc = guarded(&tmp, [&] {
    const RenderedScene sc = render_sequence(spec);
    const size_t px = static_cast<size_t>(spec.width) * spec.height;
    std::memcpy(ref, sc.ref.data().data(), px * sizeof(double));
    for (int f = 0; f < spec.trajectory.frames; ++f) {
      std::memcpy(targets + px * f, sc.targets[f].data().data(), px * sizeof(double));
      from_pose(sc.poses[f], R + 9 * f, t + 3 * f);
    }
    for (int n = 0; n < spec.num_points; ++n) {
      anchors[2 * n] = sc.anchors_px[n].x;
      anchors[2 * n + 1] = sc.anchors_px[n].y;
      inv_depths[n] = sc.inv_depths[n];
    }
  });
  if (rc != PBA_OK && err && errlen > 0) std::snprintf(err, errlen, "%s", tmp.last_error.c_str());
  return rc;
}

int pba_oracle_perturb_parameters(int32_t F, double* R, double* t, int32_t N, double* d,
                                  double sigma, uint64_t seed) {
  std::vector<Pose> poses(F);
  for (int f = 0; f < F; ++f) poses[f] = to_pose(R + 9 * f, t + 3 * f);
  std::vector<double> depths(d, d + N);
  perturb_parameters(poses, depths, sigma, seed);
  for (int f = 0; f < F; ++f) from_pose(poses[f], R + 9 * f, t + 3 * f);
  for (int n = 0; n < N; ++n) d[n] = depths[n];
  return PBA_OK;
}

}  // extern "C"

// ---- joint multi-host window (multihost.cpp) ---------------------------------------
struct pba_oracle_mh_handle {
  MhProblem p;
  std::string last_error;
};

namespace {
template <typename Fn>
int guarded_mh(pba_oracle_mh_handle* h, Fn&& fn) {
  pba_oracle_handle tmp;  // carries the error text of the shared exception mapping
  const int rc = guarded(&tmp, fn);
  if (h && rc != PBA_OK) h->last_error = tmp.last_error;
  return rc;
}
}  // namespace

extern "C" {

int pba_oracle_mh_create(const pba_mh_problem* q, pba_oracle_mh_handle** out) {
  if (!q || !out) return PBA_E_ARG;
  auto h = std::make_unique<pba_oracle_mh_handle>();
  const int rc = guarded_mh(h.get(), [&] {
    const int K = q->num_frames, N = q->num_points, P = q->pattern_size;
    if (K < 2 || N < 0 || P < 1) throw Error("bad multi-host problem sizes");
    MhProblem& p = h->p;
    for (int f = 0; f < K; ++f) {
      p.images.push_back(to_image(q->images[f]));
      p.poses.push_back(to_pose(q->pose_R + 9 * f, q->pose_t + 3 * f));
    }
    if (q->affine_a) p.affine_a.assign(q->affine_a, q->affine_a + K);
    if (q->affine_b) p.affine_b.assign(q->affine_b, q->affine_b + K);
    for (int n = 0; n < N; ++n) {
      p.host.push_back(q->host[n]);
      p.anchors_px.emplace_back(q->anchors_px[2 * n], q->anchors_px[2 * n + 1]);
      p.inv_depths.push_back(q->inv_depths[n]);
    }
    p.patch.offsets.clear();
    for (int k = 0; k < P; ++k) p.patch.offsets.push_back({q->pattern[2 * k], q->pattern[2 * k + 1]});
    if (q->obs_ptr) {
      p.obs_ptr.assign(q->obs_ptr, q->obs_ptr + N + 1);
      p.obs_frame.assign(q->obs_frame, q->obs_frame + q->obs_ptr[N]);
    }
    p.optimize_affine = q->optimize_affine != 0;
  });
  if (rc != PBA_OK) return rc;
  *out = h.release();
  return PBA_OK;
}

void pba_oracle_mh_destroy(pba_oracle_mh_handle* h) { delete h; }

const char* pba_oracle_mh_last_error(const pba_oracle_mh_handle* h) { return h ? h->last_error.c_str() : ""; }

int pba_oracle_mh_energy(pba_oracle_mh_handle* h, double gamma, pba_energy_result* out) {
  if (!h) return PBA_E_ARG;
  return guarded_mh(h, [&] {
    const MhEnergy e = mh_energy(h->p, HuberLoss{gamma});
    if (out) {
      out->energy = e.energy;
      out->num_active = e.num_active;
      out->num_out_of_bounds = e.num_oob;
    }
  });
}

int pba_oracle_mh_fc_run(pba_oracle_mh_handle* h, const pba_config* cfg, pba_report* rep, double* a_out,
                         double* b_out) {
  if (!h) return PBA_E_ARG;
  return guarded_mh(h, [&] {
    const MhReport r = mh_fc_solve(h->p, to_config(cfg));
    const int K = static_cast<int>(h->p.images.size());
    if (rep) fill_report(r.base, K, static_cast<int>(h->p.anchors_px.size()), rep);
    for (int f = 0; f < K; ++f) {
      if (a_out) a_out[f] = r.final_a[f];
      if (b_out) b_out[f] = r.final_b[f];
    }
  });
}

}  // extern "C"
