// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see pba_oracle.hpp).
//
// Joint multi-host window with per-frame affine brightness, forwards compositional
// (SURVEY.md §8f row 1).  The reference has no such solver: this is OUR statement of the
// model, built from the reference's single-host pieces, and it is what the GPU path of
// include/pba_gpu.h `pba_gpu_mh_*` is checked against.  It reduces to the reference's
// FcSolver::run (solver.cpp:663-843) when every point is hosted in frame 0 (identity) and the
// affine parameters are held (the reduction is a test, tests/test_multihost.py).
//
// Model.  Frames i = 0..K-1 with poses T_i (X_i = R_i X_w + t_i; T_0 = identity, fixed) and
// affine brightness (a_i, b_i) (frame 0: held at its values).  Point n is hosted in frame h(n)
// at an anchor pixel with inverse depth d_n; its template pixel k has the host ray x~_k and the
// template value tpl_k = I_h(anchor + offset_k) (build_template, solver.cpp:33-53).  In a
// target frame t != h:
//   T_th = T_t T_h^-1:  R_th = R_t R_h^T,  t_th = t_t - R_th t_h
//   warp x_t = pi(R_th x~ + d t_th) (project_warp, geometry.cpp:107-127) in t's intrinsics
//   r = e^(a_t - a_h) (tpl - b_h) + b_t - I_t(x_t)          (a = b = 0: the reference's r)
// Parameters per frame i >= 1: (omega, dt) with pose_boxplus (R <- exp(omega) R, t <- t + dt,
// geometry.cpp:93-98) and, when optimised, (da, db); per point d <- d + dd.
// Jacobian of one pixel: the reference's FC row w.r.t. the relative pose increment
// (fc_warp_jacobian, geometry.cpp:129-139; row = -(grad^T J_img), solver.cpp:706-709),
// chained to the absolute increments:
//   omega_th = omega_t - R_th omega_h,   dt_th = dt_t - R_th dt_h + [u]x omega_th,  u = R_th t_h
//   => J_omega_t = J_w + J_t [u]x,  J_dt_t = J_t,  J_omega_h = -J_omega_t R_th,  J_dt_h = -J_t R_th
//   J_a_t = alpha (tpl - b_h), J_b_t = 1, J_a_h = -alpha (tpl - b_h), J_b_h = -alpha,
//   alpha = e^(a_t - a_h).
// Normal equations: dense frame block H_FF (Q (K-1) square, Q = 6 or 8) with the host-target
// cross blocks, per-point D_n and b_n; Levenberg damping (H + lambda I) and the reduced system
// S = H_FF + lambda I - sum_n b_n b_n^T / (D_n + lambda) (solver.cpp:165-213 generalised).
// LM control, gauge (mean inverse depth, all translations) and the max reprojection update are
// the reference's FC rules (solver.cpp:685-843, :105-143).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>

#include "pba_oracle.hpp"

namespace oracle {

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) { return std::chrono::duration<double, std::milli>(Clock::now() - t0).count(); }
bool in_margin(const Image& img, const Vec2& px) {  // solver.cpp:22-25
  return px.x >= 1.0 && px.x <= img.width() - 3 && px.y >= 1.0 && px.y <= img.height() - 3;
}

Pose relative(const Pose& Tt, const Pose& Th) {  // T_t T_h^-1
  Pose r;
  r.R = Tt.R * Th.R.transpose();
  r.t = Tt.t - r.R * Th.t;
  return r;
}

struct MhTemplate {
  std::vector<Vec2> norm;  // host-normalized template rays, N*P
  std::vector<double> val;
};

MhTemplate mh_template(const MhProblem& p) {  // build_template (solver.cpp:33-53) in each host
  const int N = static_cast<int>(p.anchors_px.size());
  const int P = static_cast<int>(p.patch.offsets.size());
  MhTemplate t;
  t.norm.resize(static_cast<size_t>(N) * P);
  t.val.resize(t.norm.size());
  for (int n = 0; n < N; ++n) {
    const Image& img = p.images[p.host[n]];
    for (int k = 0; k < P; ++k) {
      const Vec2 px = p.anchors_px[n] + Vec2(p.patch.offsets[k][0], p.patch.offsets[k][1]);
      if (!in_margin(img, px)) throw OutOfBounds("template patch pixel outside its host image");
      t.norm[static_cast<size_t>(n) * P + k] = img.intrinsics().to_normalized(px);
      t.val[static_cast<size_t>(n) * P + k] = img.sample_px_unchecked(px);
    }
  }
  return t;
}

struct MhObs {
  std::vector<int64_t> ptr;
  std::vector<int32_t> frame;
};

MhObs mh_obs(const MhProblem& p) {
  const int N = static_cast<int>(p.anchors_px.size());
  const int K = static_cast<int>(p.images.size());
  MhObs o;
  if (!p.obs_ptr.empty()) {
    o.ptr = p.obs_ptr;
    o.frame = p.obs_frame;
    for (int n = 0; n < N; ++n)
      for (int64_t q = o.ptr[n]; q < o.ptr[n + 1]; ++q)
        if (o.frame[q] == p.host[n] || o.frame[q] < 0 || o.frame[q] >= K) throw Error("bad multi-host observation");
    return o;
  }
  o.ptr.assign(static_cast<size_t>(N) + 1, 0);
  for (int n = 0; n < N; ++n) {
    for (int f = 0; f < K; ++f)
      if (f != p.host[n]) o.frame.push_back(f);
    o.ptr[n + 1] = static_cast<int64_t>(o.frame.size());
  }
  return o;
}

struct MhState {
  std::vector<Pose> poses;
  std::vector<double> a, b, d;
};

struct MhPass {
  double energy{0.0};
  int64_t num_active{0}, num_oob{0};
  std::vector<double> r;
  std::vector<uint8_t> active;
};

MhPass mh_residuals(const MhProblem& p, const MhObs& obs, const MhTemplate& tpl, const MhState& s,
                    const HuberLoss& huber) {
  const int N = static_cast<int>(p.anchors_px.size());
  const int P = static_cast<int>(p.patch.offsets.size());
  MhPass out;
  out.r.assign(obs.frame.size() * P, 0.0);
  out.active.assign(out.r.size(), 0);
  for (int n = 0; n < N; ++n) {
    const int h = p.host[n];
    for (int64_t o = obs.ptr[n]; o < obs.ptr[n + 1]; ++o) {
      const int t = obs.frame[o];
      const Pose Tth = relative(s.poses[t], s.poses[h]);
      const double alpha = std::exp(s.a[t] - s.a[h]);
      const Image& img = p.images[t];
      for (int k = 0; k < P; ++k) {
        const size_t idx = static_cast<size_t>(o) * P + k;
        Vec2 w;
        try {
          w = project_warp(tpl.norm[static_cast<size_t>(n) * P + k], Tth, s.d[n]);
        } catch (const DegenerateDepth&) {
          ++out.num_oob;
          continue;
        }
        const Vec2 px = img.intrinsics().to_pixel(w);
        if (!in_margin(img, px)) {
          ++out.num_oob;
          continue;
        }
        const double r = alpha * (tpl.val[static_cast<size_t>(n) * P + k] - s.b[h]) + s.b[t] - img.sample_px_unchecked(px);
        out.r[idx] = r;
        out.active[idx] = 1;
        out.energy += huber.loss(r);
        ++out.num_active;
      }
    }
  }
  return out;
}

// block index of frame i >= 1 in the frame parameter vector (frame 0 is held)
inline int fblk(int f, int Q) { return (f - 1) * Q; }

struct MhSystem {
  int nF{0}, N{0}, Q{6};
  std::vector<double> H;   // nF x nF (frame parameters)
  std::vector<double> B;   // N x nF (b_n rows)
  std::vector<double> D;   // N
  std::vector<double> g;   // nF + N
};

MhSystem mh_build(const MhProblem& p, const MhObs& obs, const MhTemplate& tpl, const MhState& s,
                  const HuberLoss& huber, const MhPass& pass) {
  const int K = static_cast<int>(p.images.size());
  const int N = static_cast<int>(p.anchors_px.size());
  const int P = static_cast<int>(p.patch.offsets.size());
  MhSystem S;
  S.Q = p.optimize_affine ? 8 : 6;
  S.nF = S.Q * (K - 1);
  S.N = N;
  S.H.assign(static_cast<size_t>(S.nF) * S.nF, 0.0);
  S.B.assign(static_cast<size_t>(N) * S.nF, 0.0);
  S.D.assign(N, 0.0);
  S.g.assign(static_cast<size_t>(S.nF) + N, 0.0);
  const int Q = S.Q;
  std::vector<int> col(2 * Q);
  std::vector<double> row(2 * Q);
  for (int n = 0; n < N; ++n) {
    const int h = p.host[n];
    for (int64_t o = obs.ptr[n]; o < obs.ptr[n + 1]; ++o) {
      const int t = obs.frame[o];
      const Pose Tth = relative(s.poses[t], s.poses[h]);
      const Vec3 u = Tth.R * s.poses[h].t;
      const double alpha = std::exp(s.a[t] - s.a[h]);
      for (int k = 0; k < P; ++k) {
        const size_t idx = static_cast<size_t>(o) * P + k;
        if (!pass.active[idx]) continue;
        const Vec2& x = tpl.norm[static_cast<size_t>(n) * P + k];
        double rel[7];
        try {  // solver.cpp:706-709 at the relative pose
          const Vec2 w = project_warp(x, Tth, s.d[n]);
          const Vec2 grad = image_gradient(p.images[t], w);
          const WarpJacobian wj = fc_warp_jacobian(x, Tth, s.d[n]);
          for (int c = 0; c < 7; ++c) rel[c] = -(grad.x * wj.image[0][c] + grad.y * wj.image[1][c]);
        } catch (const Error&) {
          continue;
        }
        // chain to the absolute increments of t and h
        double Jwt[3], Jtt[3], Jwh[3], Jth[3];
        for (int j = 0; j < 3; ++j) {  // J_w + J_t [u]x  ([u]x = skew(u), row vector times matrix)
          double v = rel[j];
          for (int i = 0; i < 3; ++i) v += rel[3 + i] * skew(u)(i, j);
          Jwt[j] = v;
          Jtt[j] = rel[3 + j];
        }
        for (int j = 0; j < 3; ++j) {
          double vw = 0.0, vt = 0.0;
          for (int i = 0; i < 3; ++i) {
            vw += Jwt[i] * Tth.R(i, j);
            vt += Jtt[i] * Tth.R(i, j);
          }
          Jwh[j] = -vw;
          Jth[j] = -vt;
        }
        const double ja = alpha * (tpl.val[static_cast<size_t>(n) * P + k] - s.b[h]);
        int m = 0;
        auto put = [&](int f, const double* jw, const double* jt, double a_, double b_) {
          if (f == 0) return;
          const int c0 = fblk(f, Q);
          for (int i = 0; i < 3; ++i) { col[m] = c0 + i; row[m++] = jw[i]; }
          for (int i = 0; i < 3; ++i) { col[m] = c0 + 3 + i; row[m++] = jt[i]; }
          if (Q == 8) {
            col[m] = c0 + 6; row[m++] = a_;
            col[m] = c0 + 7; row[m++] = b_;
          }
        };
        put(t, Jwt, Jtt, ja, 1.0);
        put(h, Jwh, Jth, -ja, -alpha);
        const double wgt = huber.weight(pass.r[idx]);
        const double wr = wgt * pass.r[idx];
        const double jd = rel[6];
        for (int i = 0; i < m; ++i) {
          for (int j = 0; j < m; ++j) S.H[static_cast<size_t>(col[i]) * S.nF + col[j]] += wgt * row[i] * row[j];
          S.B[static_cast<size_t>(n) * S.nF + col[i]] += wgt * row[i] * jd;
          S.g[col[i]] += row[i] * wr;
        }
        S.D[n] += wgt * jd * jd;
        S.g[static_cast<size_t>(S.nF) + n] += jd * wr;
      }
    }
  }
  return S;
}

// S = H_FF + lambda I - sum_n b_n b_n^T / (D_n + lambda); xp = S^-1 (-g_F + sum_n b_n g_n / (D_n + lambda));
// dx_n = (-g_n - b_n . xp) / (D_n + lambda)  (solver.cpp:165-213 with the dense frame block)
std::vector<double> mh_solve(const MhSystem& S, double lambda) {
  const int nF = S.nF, N = S.N;
  std::vector<double> A = S.H;
  for (int i = 0; i < nF; ++i) A[static_cast<size_t>(i) * nF + i] += lambda;
  std::vector<double> rhs(nF);
  for (int i = 0; i < nF; ++i) rhs[i] = -S.g[i];
  for (int n = 0; n < N; ++n) {
    const double Dl = S.D[n] + lambda;
    const double* b = &S.B[static_cast<size_t>(n) * nF];
    const double gd = S.g[static_cast<size_t>(nF) + n];
    for (int i = 0; i < nF; ++i) {
      if (b[i] == 0.0) continue;
      rhs[i] += b[i] * (gd / Dl);
      for (int j = 0; j < nF; ++j) A[static_cast<size_t>(i) * nF + j] -= b[i] * b[j] / Dl;
    }
  }
  DenseCholesky chol;
  if (!chol.compute(A, nF)) throw Error("SingularHessian: multi-host reduced factorization failed");
  const std::vector<double> xp = chol.solve(rhs);
  std::vector<double> dx(static_cast<size_t>(nF) + N);
  for (int i = 0; i < nF; ++i) {
    if (!std::isfinite(xp[i])) throw Error("SingularHessian: non-finite pose solution");
    dx[i] = xp[i];
  }
  for (int n = 0; n < N; ++n) {
    const double* b = &S.B[static_cast<size_t>(n) * nF];
    double acc = -S.g[static_cast<size_t>(nF) + n];
    for (int i = 0; i < nF; ++i) acc -= b[i] * xp[i];
    dx[static_cast<size_t>(nF) + n] = acc / (S.D[n] + lambda);
    if (!std::isfinite(dx[static_cast<size_t>(nF) + n])) throw Error("SingularHessian: non-finite depth solution");
  }
  return dx;
}

double mh_max_update(const MhProblem& p, const MhObs& obs, const MhTemplate& tpl, const MhState& s0,
                     const MhState& s1) {  // solver.cpp:105-131 over every (n, target)
  const int N = static_cast<int>(p.anchors_px.size());
  const int P = static_cast<int>(p.patch.offsets.size());
  double mx = 0.0;
  for (int n = 0; n < N; ++n) {
    const int h = p.host[n];
    const Vec2& x = tpl.norm[static_cast<size_t>(n) * P];
    for (int64_t o = obs.ptr[n]; o < obs.ptr[n + 1]; ++o) {
      const int t = obs.frame[o];
      try {
        const Vec2 a = p.images[t].intrinsics().to_pixel(project_warp(x, relative(s0.poses[t], s0.poses[h]), s0.d[n]));
        const Vec2 b = p.images[t].intrinsics().to_pixel(project_warp(x, relative(s1.poses[t], s1.poses[h]), s1.d[n]));
        mx = std::max(mx, (a - b).norm());
      } catch (const DegenerateDepth&) {
        mx = std::numeric_limits<double>::infinity();
      }
    }
  }
  return mx;
}

void mh_gauge(MhState& s) {  // normalize_depth_gauge (solver.cpp:135-143) over every frame
  double mean = 0.0;
  for (double d : s.d) mean += d;
  mean /= static_cast<double>(s.d.size());
  if (mean <= 0.0 || !std::isfinite(mean)) return;
  for (double& d : s.d) d /= mean;
  for (Pose& q : s.poses) q.t = q.t * mean;
}

MhState initial_state(const MhProblem& p) {
  MhState s;
  s.poses = p.poses;
  const size_t K = p.images.size();
  s.a = p.affine_a.empty() ? std::vector<double>(K, 0.0) : p.affine_a;
  s.b = p.affine_b.empty() ? std::vector<double>(K, 0.0) : p.affine_b;
  s.d = p.inv_depths;
  return s;
}

void validate(const MhProblem& p) {
  const int K = static_cast<int>(p.images.size());
  if (K < 2) throw Error("multi-host window needs at least 2 frames");
  if (p.poses.size() != p.images.size()) throw Error("one pose per frame");
  if (p.host.size() != p.anchors_px.size() || p.inv_depths.size() != p.anchors_px.size())
    throw Error("host / anchors / inverse depths size mismatch");
  for (int h : p.host)
    if (h < 0 || h >= K) throw Error("host frame out of range");
}

}  // namespace

MhEnergy mh_energy(const MhProblem& p, const HuberLoss& huber) {
  validate(p);
  const MhTemplate tpl = mh_template(p);
  const MhObs obs = mh_obs(p);
  const MhPass pass = mh_residuals(p, obs, tpl, initial_state(p), huber);
  if (pass.num_active == 0) throw EmptyProblem();
  return {pass.energy, pass.num_active, pass.num_oob};
}

MhReport mh_fc_solve(const MhProblem& p, const SolverConfig& config) {
  validate(p);
  const HuberLoss huber{config.gamma};
  const auto t_start = Clock::now();
  const MhTemplate tpl = mh_template(p);
  const MhObs obs = mh_obs(p);
  const int K = static_cast<int>(p.images.size());
  const int N = static_cast<int>(p.anchors_px.size());
  const int Q = p.optimize_affine ? 8 : 6;

  MhReport report;
  MhState s = initial_state(p);
  MhPass pass = mh_residuals(p, obs, tpl, s, huber);
  if (pass.num_active == 0) throw EmptyProblem();  // :675
  const int64_t initial_active = pass.num_active;
  double energy = pass.energy;
  double lambda = config.lambda0;  // :679
  double wall_ms = ms_since(t_start);
  int bad = 0, builds = 0, factorizations = 0;

  auto record = [&](int iter, double e, double mu, int64_t nact, bool acc) {
    IterationStats st;
    st.iter = iter;
    st.energy = e;
    st.max_update_px = mu;
    st.wall_ms = wall_ms;
    st.hessian_builds = builds;
    st.hessian_factorizations = factorizations;
    st.num_active = nact;
    st.accepted = acc;
    if (config.record_snapshots) {
      st.poses = s.poses;
      st.inv_depths = s.d;
    }
    report.base.iters.push_back(std::move(st));
    report.base.iterations = iter;
  };

  for (int iter = 1; iter <= config.max_iters; ++iter) {  // FcSolver::run, solver.cpp:685-843
    const auto t_iter = Clock::now();
    const MhSystem S = mh_build(p, obs, tpl, s, huber, pass);
    ++builds;
    bool accepted = false;
    MhState cand;
    MhPass cand_pass;
    while (!accepted) {
      std::vector<double> dx;
      try {  // :732-740
        ++factorizations;
        dx = mh_solve(S, lambda);
      } catch (const Error&) {
        lambda *= 10.0;
        ++report.base.rejected_steps;
        if (++bad >= config.max_bad_steps) break;
        continue;
      }
      cand = s;
      bool valid = true;
      for (int f = 1; f < K; ++f) {  // :744-746 (+ affine)
        const int c0 = fblk(f, Q);
        Vec6 d6;
        for (int i = 0; i < 6; ++i) d6[i] = dx[c0 + i];
        cand.poses[f] = pose_boxplus(s.poses[f], d6);
        if (Q == 8) {
          cand.a[f] = s.a[f] + dx[c0 + 6];
          cand.b[f] = s.b[f] + dx[c0 + 7];
        }
      }
      for (int n = 0; n < N; ++n) {  // :747-750
        cand.d[n] = s.d[n] + dx[static_cast<size_t>(Q) * (K - 1) + n];
        if (cand.d[n] <= 0.0) valid = false;
      }
      if (valid) {
        cand_pass = mh_residuals(p, obs, tpl, cand, huber);
        valid = cand_pass.num_active > 0;
      }
      if (valid && cand_pass.energy <= energy * (1.0 + 1e-12) + 1e-15) {  // :756-759
        accepted = true;
        bad = 0;
        lambda = std::max(lambda / 10.0, config.lambda0);
      } else {
        if (valid) {  // :764-786
          const double mu = mh_max_update(p, obs, tpl, s, cand);
          if (mu < config.threshold_px) {
            report.base.converged = true;
            report.base.message = "converged: sub-threshold step rejected";
            wall_ms += ms_since(t_iter);
            record(iter, energy, mu, pass.num_active, false);
            break;
          }
        }
        lambda *= 10.0;
        ++report.base.rejected_steps;
        if (++bad >= config.max_bad_steps) break;
      }
    }
    if (!accepted) {  // :792-798
      if (report.base.converged) break;
      report.base.diverged = true;
      report.base.message = "Diverged: " + std::to_string(bad) + " consecutive rejected damped steps";
      break;
    }
    const double mu = mh_max_update(p, obs, tpl, s, cand);
    bool zero_grad = true;
    for (double v : S.g)
      if (v != 0.0) zero_grad = false;
    s = std::move(cand);
    energy = cand_pass.energy;
    pass = std::move(cand_pass);
    if (config.normalize_depth_gauge) mh_gauge(s);
    wall_ms += ms_since(t_iter);
    record(iter, energy, mu, pass.num_active, true);
    if (mu < config.threshold_px) {
      report.base.converged = true;
      if (zero_grad) report.base.message = "no-progress convergence: zero gradient";
      break;
    }
  }
  report.base.hessian_builds = builds;
  report.base.hessian_factorizations = factorizations;
  report.base.final_energy = energy;
  report.base.total_wall_ms = wall_ms;
  report.base.final_poses = s.poses;
  report.base.final_inv_depths = s.d;
  report.base.masked_residuals = initial_active - pass.num_active;
  report.final_a = s.a;
  report.final_b = s.b;
  return report;
}

}  // namespace oracle
