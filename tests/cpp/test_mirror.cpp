// C++ parity tests through include/pba_b200.hpp (the reference-shaped C++ mirror over the
// C ABI), written like the reference's doctest cases (test_solver.cpp).  Scenes come from
// the CPU oracle's restated synth.cpp; expected values from the oracle (TEST INFRASTRUCTURE).
#include <cmath>
#include <cstdio>
#include <string>

#include "../../include/pba_b200.hpp"
#include "../../oracle/pba_oracle.hpp"

static int g_fail = 0;
#define CHECK(c)                                                                    \
  do {                                                                              \
    if (!(c)) {                                                                     \
      ++g_fail;                                                                     \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);            \
    }                                                                               \
  } while (0)

static oracle::SceneSpec small_spec(int frames, int points) {  // test_solver.cpp:14-23
  oracle::SceneSpec s;
  s.width = 160;
  s.height = 120;
  s.intrinsics = {130.0, 130.0, 79.5, 59.5};
  s.num_points = points;
  s.trajectory.frames = frames;
  s.trajectory.span_deg = 6.0;
  return s;
}

// Same inputs for both sides: fp32-rounded images.
struct Pair {
  oracle::ProblemState o;
  pba_b200::ProblemState g;
};
static Pair make_pair(const oracle::RenderedScene& sc, int radius, double sigma, uint64_t seed) {
  Pair p;
  p.o.ref = sc.ref;
  p.o.targets = sc.targets;
  p.o.poses = sc.poses;
  p.o.anchors_px = sc.anchors_px;
  p.o.inv_depths = sc.inv_depths;
  p.o.patch = oracle::PatchPattern::square(radius);
  oracle::perturb_parameters(p.o.poses, p.o.inv_depths, sigma, seed);
  auto cvt = [](oracle::Image& im) {
    pba_b200::Image g;
    g.width = im.width();
    g.height = im.height();
    g.K = {im.intrinsics().fx, im.intrinsics().fy, im.intrinsics().cx, im.intrinsics().cy};
    g.data.resize(im.data().size());
    for (size_t i = 0; i < g.data.size(); ++i) {
      g.data[i] = static_cast<float>(im.data()[i]);
      im.data()[i] = static_cast<double>(g.data[i]);
    }
    return g;
  };
  p.g.ref = cvt(p.o.ref);
  for (auto& t : p.o.targets) p.g.targets.push_back(cvt(t));
  for (const auto& ps : p.o.poses) {
    pba_b200::Pose q;
    for (int i = 0; i < 9; ++i) q.R[i] = ps.R.a[i];
    q.t = {ps.t.x, ps.t.y, ps.t.z};
    p.g.poses.push_back(q);
  }
  for (const auto& a : p.o.anchors_px) p.g.anchors_px.push_back({a.x, a.y});
  p.g.inv_depths = p.o.inv_depths;
  p.g.pattern.clear();
  for (const auto& o : p.o.patch.offsets) p.g.pattern.push_back({o[0], o[1]});
  return p;
}

static void energy_matches() {
  auto pr = make_pair(oracle::render_sequence(small_spec(2, 3)), 1, 2e-3, 5);
  const auto eo = oracle::energy_eval(pr.o, oracle::HuberLoss{0.03});
  const auto eg = pba_b200::energy_eval(pr.g, pba_b200::HuberLoss{0.03});
  CHECK(eg.num_active == eo.num_active);
  CHECK(std::abs(eg.energy - eo.energy) <= 1e-5 * eo.energy);
}

static void empty_problem_throws() {  // test_solver.cpp:103-108
  auto pr = make_pair(oracle::render_sequence(small_spec(2, 3)), 1, 0.0, 1);
  for (auto& p : pr.g.poses) p.t = {50.0, 0.0, 0.0};
  bool thrown = false;
  try {
    pba_b200::energy_eval(pr.g, pba_b200::HuberLoss{0.03});
  } catch (const pba_b200::EmptyProblem&) {
    thrown = true;
  }
  CHECK(thrown);
}

static void ic_step_matches_oracle() {  // test_solver.cpp:163-206 (vs the pinned oracle)
  auto pr = make_pair(oracle::render_sequence(small_spec(2, 3)), 0, 1e-3, 7);
  oracle::IcSolver so(pr.o, oracle::SolverConfig{});
  so.build();
  const auto dxo = so.compute_step();
  pba_b200::IcSolver sg(pr.g, pba_b200::SolverConfig{});
  sg.build();
  const auto dxg = sg.compute_step();
  // compare after removing the scale-gauge direction (0, t0, -d0)
  const int F = pr.o.num_frames(), N = pr.o.num_points();
  std::vector<double> v(6 * F + N, 0.0);
  for (int f = 0; f < F; ++f) {
    v[6 * f + 3] = pr.o.poses[f].t.x;
    v[6 * f + 4] = pr.o.poses[f].t.y;
    v[6 * f + 5] = pr.o.poses[f].t.z;
  }
  for (int n = 0; n < N; ++n) v[6 * F + n] = -pr.o.inv_depths[n];
  double vv = 0, ag = 0, ao = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    vv += v[i] * v[i];
    ag += dxg[i] * v[i];
    ao += dxo[i] * v[i];
  }
  double num = 0, den = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    const double a = dxg[i] - ag / vv * v[i], b = dxo[i] - ao / vv * v[i];
    num += (a - b) * (a - b);
    den += b * b;
  }
  CHECK(std::sqrt(num) <= 1e-4 * std::sqrt(den));
}

static void noisy_start_counters() {  // test_solver.cpp:225-249
  auto pr = make_pair(oracle::render_sequence(small_spec(3, 10)), 1, 1e-3, 8);
  pba_b200::SolverConfig cfg;
  cfg.record_snapshots = true;
  const auto fc = pba_b200::fc_solve(pr.g, cfg);
  const auto ic = pba_b200::ic_solve(pr.g, cfg);
  CHECK(fc.converged);
  CHECK(ic.converged);
  CHECK(ic.hessian_builds == 1);
  for (size_t i = 1; i < fc.iters.size(); ++i) CHECK(fc.iters[i].energy <= fc.iters[i - 1].energy * (1 + 1e-12) + 1e-15);
  for (size_t i = 1; i < ic.iters.size(); ++i) CHECK(ic.iters[i].energy <= ic.iters[i - 1].energy * (1 + 1e-12) + 1e-15);
  for (const auto& it : fc.iters) CHECK(it.hessian_builds == it.iter);
  CHECK(std::abs(fc.final_energy - ic.final_energy) <= 0.01 * std::max(fc.final_energy, ic.final_energy));
  const auto ico = oracle::ic_solve(pr.o, oracle::SolverConfig{});
  CHECK(ico.iterations == ic.iterations);
}

static void zero_translation_warning() {  // test_solver.cpp:266-278
  auto pr = make_pair(oracle::render_sequence(small_spec(2, 3)), 1, 0.0, 1);
  pr.g.targets = {pr.g.ref};
  pr.g.poses = {pba_b200::Pose{}};
  pba_b200::IcSolver s(pr.g, pba_b200::SolverConfig{});
  s.build();
  const auto w = s.warnings();
  CHECK(!w.empty() && w.front().find("zero initial translation") != std::string::npos);
  for (double dd : s.hessian().depth_depth) CHECK(dd == 0.0);
}

static void joint_window_reduces_to_fc() {  // the joint window of a single-host problem = fc_solve
  auto pr = make_pair(oracle::render_sequence(small_spec(3, 10)), 1, 1e-3, 8);
  pba_b200::MultiHostProblem w;
  w.images.push_back(pr.g.ref);
  w.poses.push_back(pba_b200::Pose{});
  for (size_t f = 0; f < pr.g.targets.size(); ++f) {
    w.images.push_back(pr.g.targets[f]);
    w.poses.push_back(pr.g.poses[f]);
  }
  w.host.assign(pr.g.anchors_px.size(), 0);
  w.anchors_px = pr.g.anchors_px;
  w.inv_depths = pr.g.inv_depths;
  w.pattern = pr.g.pattern;
  w.optimize_affine = false;
  pba_b200::SolverConfig cfg;
  cfg.max_iters = 10;
  const auto r = pba_b200::mh_fc_solve(w, cfg);
  oracle::SolverConfig oc;
  oc.max_iters = 10;
  const auto ref = oracle::fc_solve(pr.o, oc);
  CHECK(r.iterations == ref.iterations);
  CHECK(r.converged == ref.converged);
  CHECK(std::abs(r.final_energy - ref.final_energy) <= 1e-5 * ref.final_energy);
  CHECK(r.final_poses.size() == pr.g.poses.size() + 1 && r.final_a.size() == w.images.size());
  for (size_t n = 0; n < ref.final_inv_depths.size(); ++n)
    CHECK(std::abs(r.final_inv_depths[n] - ref.final_inv_depths[n]) <= 1e-4 * std::abs(ref.final_inv_depths[n]));
}

int main() {
  struct {
    const char* name;
    void (*fn)();
  } cases[] = {{"energy_eval matches the oracle", energy_matches},
               {"energy_eval throws when nothing is in bounds", empty_problem_throws},
               {"one IC step equals the oracle (gauge removed)", ic_step_matches_oracle},
               {"noisy start: both converge, counters correct", noisy_start_counters},
               {"zero initial translation warning", zero_translation_warning},
               {"joint multi-host window of a single-host problem = fc_solve", joint_window_reduces_to_fc}};
  int failed = 0;
  for (auto& c : cases) {
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    const bool ok = g_fail == before;
    failed += ok ? 0 : 1;
    std::printf("%s  %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  return failed ? 1 : 0;
}
