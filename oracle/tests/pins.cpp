// CPU ORACLE PINS — TEST INFRASTRUCTURE ONLY.
//
// The reference has no golden vectors on disk; every pin is a
// runtime known-answer / property test.  This binary restates those tests
// (same names, seeds, sizes and tolerances) against the oracle so the oracle is
// pinned before it is used to judge the GPU path.  Sources:
//   /root/reference/proj/tests/test_geometry.cpp, test_image.cpp,
//   test_solver.cpp, test_synth.cpp, acceptance.cpp (criteria 1,2,4-9).
// Usage: pins [substring-filter]   — prints PASS/FAIL per case, exit 1 on failure.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "../pba_oracle.hpp"

using namespace oracle;

// ---- mini test framework -----------------------------------------------------
static int g_fail_checks = 0;
static std::string g_case;
#define CHECK(cond)                                                                   \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      ++g_fail_checks;                                                                \
      std::printf("  CHECK failed [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, T)          \
  do {                                    \
    bool thrown_ = false;                 \
    try {                                 \
      (void)(expr);                       \
    } catch (const T&) {                  \
      thrown_ = true;                     \
    } catch (...) {                       \
    }                                     \
    CHECK(thrown_ && #T);                 \
  } while (0)
static bool approx(double a, double b, double eps = 1e-5) {  // doctest::Approx default scale
  return std::abs(a - b) < eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}

struct Case {
  const char* name;
  std::function<void()> fn;
};
static std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name) \
  static void CAT(tc_, __LINE__)(); \
  static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
  static void CAT(tc_, __LINE__)()

// ---- helpers (tests/helpers.hpp) -----------------------------------------------
static std::mt19937_64 make_rng(uint64_t s) { return std::mt19937_64(s); }
static double uniform(std::mt19937_64& r, double lo, double hi) {
  return std::uniform_real_distribution<double>(lo, hi)(r);
}
static Vec3 random_vec3(std::mt19937_64& r, double s) {
  const double a = uniform(r, -s, s), b = uniform(r, -s, s), c = uniform(r, -s, s);
  return Vec3(a, b, c);
}
static Pose random_pose(std::mt19937_64& r, double rs, double ts) {
  Pose p;
  p.R = so3_exp(random_vec3(r, rs));
  p.t = random_vec3(r, ts);
  return p;
}
static Mat3 mat_exp_taylor(const Mat3& A) {  // helpers.hpp:35-43 (3x3)
  Mat3 sum = Mat3::Identity(), term = Mat3::Identity();
  for (int k = 1; k <= 20; ++k) {
    term = (term * A) * (1.0 / k);
    sum = sum + term;
  }
  return sum;
}
static double naive_energy(const ProblemState& st, double gamma) {  // helpers.hpp:63-91
  double total = 0.0;
  const auto& K = st.ref.intrinsics();
  for (size_t n = 0; n < st.anchors_px.size(); ++n)
    for (size_t f = 0; f < st.targets.size(); ++f)
      for (const auto& off : st.patch.offsets) {
        const Vec2 px = st.anchors_px[n] + Vec2(off[0], off[1]);
        const Vec2 x = K.to_normalized(px);
        if (!st.ref.in_bounds_px(px)) continue;
        Vec2 warped;
        try {
          warped = project_warp(x, st.poses[f], st.inv_depths[n]);
        } catch (const DegenerateDepth&) {
          continue;
        }
        const Vec2 wpx = st.targets[f].intrinsics().to_pixel(warped);
        if (wpx.x < 1.0 || wpx.x > st.targets[f].width() - 3 || wpx.y < 1.0 ||
            wpx.y > st.targets[f].height() - 3)
          continue;
        const double r = st.ref.sample_px_unchecked(px) - st.targets[f].sample_px_unchecked(wpx);
        const double a = std::abs(r);
        total += a <= gamma ? 0.5 * r * r : gamma * (a - 0.5 * gamma);
      }
  return total;
}
template <typename Fn>
static double golden_section_min(const Fn& f, double a, double b, double tol) {  // helpers.hpp:95-111
  const double phi = (std::sqrt(5.0) - 1.0) / 2.0;
  double c = b - phi * (b - a), d = a + phi * (b - a);
  while (b - a > tol) {
    if (f(c) < f(d)) {
      b = d;
      d = c;
      c = b - phi * (b - a);
    } else {
      a = c;
      c = d;
      d = a + phi * (b - a);
    }
  }
  return 0.5 * (a + b);
}
static Vec7 rand_dir7(std::mt19937_64& r) {
  Vec7 d;
  double s = 0;
  for (int c = 0; c < 7; ++c) {
    d[c] = uniform(r, -1.0, 1.0);
    s += d[c] * d[c];
  }
  s = std::sqrt(s);
  for (double& v : d) v /= s;
  return d;
}
static Vec7 scale7(const Vec7& d, double e) {
  Vec7 o;
  for (int i = 0; i < 7; ++i) o[i] = d[i] * e;
  return o;
}
static double jac_maxabs(const double J[2][7]) {
  double m = 0;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 7; ++c) m = std::max(m, std::abs(J[r][c]));
  return m;
}

static SceneSpec small_spec(int frames = 2, int points = 6) {  // test_solver.cpp:14-23
  SceneSpec s;
  s.width = 160;
  s.height = 120;
  s.intrinsics = {130.0, 130.0, 79.5, 59.5};
  s.num_points = points;
  s.trajectory.frames = frames;
  s.trajectory.span_deg = 6.0;
  return s;
}
static ProblemState make_state(const RenderedScene& sc, int patch_radius = 1) {  // :25-34
  ProblemState st;
  st.ref = sc.ref;
  st.targets = sc.targets;
  st.poses = sc.poses;
  st.anchors_px = sc.anchors_px;
  st.inv_depths = sc.inv_depths;
  st.patch = PatchPattern::square(patch_radius);
  return st;
}
static double vnorm(const std::vector<double>& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

// ============================ geometry (test_geometry.cpp) ============================
TEST_CASE("skew matrix reproduces the cross product") {  // :12-20
  auto rng = make_rng(11);
  for (int i = 0; i < 50; ++i) {
    const Vec3 a = random_vec3(rng, 2.0), b = random_vec3(rng, 2.0);
    CHECK(approx((skew(a) * b - a.cross(b)).norm(), 0.0));
    CHECK((skew(a) + skew(a).transpose()).norm() == 0.0);
  }
}
TEST_CASE("so3_exp basics") {  // :22-28
  CHECK((so3_exp(Vec3(0, 0, 0)) - Mat3::Identity()).norm() == 0.0);
  const Mat3 R = so3_exp(Vec3(0, 0, M_PI / 2));
  CHECK((R * Vec3(1, 0, 0) - Vec3(0, 1, 0)).norm() < 1e-12);
}
TEST_CASE("so3_exp matches a truncated Taylor series") {  // :30-40
  auto rng = make_rng(12);
  for (int i = 0; i < 200; ++i) {
    const Vec3 w = random_vec3(rng, 0.5);
    const Mat3 R = so3_exp(w);
    CHECK((R - mat_exp_taylor(skew(w))).norm() < 1e-10);
    CHECK((R.transpose() * R - Mat3::Identity()).norm() < 1e-12);
  }
}
TEST_CASE("boxplus is the identity at zero and composes as documented") {  // :77-90 (pose part)
  auto rng = make_rng(16);
  const Pose pose = random_pose(rng, 0.8, 0.5);
  const Pose same = pose_boxplus(pose, Vec6{});
  CHECK((same.R - pose.R).norm() == 0.0);
  CHECK((same.t - pose.t).norm() == 0.0);
  const Vec6 delta{0.1, -0.2, 0.05, 0.3, 0.0, -0.1};
  const Pose moved = pose_boxplus(pose, delta);
  CHECK((moved.R - so3_exp(Vec3(0.1, -0.2, 0.05)) * pose.R).norm() < 1e-14);
  CHECK((moved.t - (pose.t + Vec3(0.3, 0.0, -0.1))).norm() == 0.0);
}
TEST_CASE("project arithmetic and scale invariance") {  // :100-107
  CHECK((project(Vec3(2, 4, 2)) - Vec2(1, 2)).norm() == 0.0);
  CHECK((project(Vec3(0.3, -0.7, 1)) - Vec2(0.3, -0.7)).norm() == 0.0);
  const Vec3 v(0.4, -1.1, 2.3);
  CHECK((project(3.7 * v) - project(v)).norm() < 1e-15);
  CHECK_THROWS_AS(project(Vec3(1, 1, 0)), DegenerateDepth);
  CHECK_THROWS_AS(project(Vec3(1, 1, 1e-13)), DegenerateDepth);
}
TEST_CASE("project_jacobian matches finite differences") {  // :109-122
  auto rng = make_rng(17);
  for (int i = 0; i < 100; ++i) {
    Vec3 v = random_vec3(rng, 1.0);
    v.z = uniform(rng, 0.5, 3.0);
    double J[2][3];
    project_jacobian(v, J);
    double err = 0;
    for (int c = 0; c < 3; ++c) {
      Vec3 hi = v, lo = v;
      hi[c] += 1e-6;
      lo[c] -= 1e-6;
      const Vec2 fd = (project(hi) - project(lo)) * (1.0 / 2e-6);
      err += (fd.x - J[0][c]) * (fd.x - J[0][c]) + (fd.y - J[1][c]) * (fd.y - J[1][c]);
    }
    CHECK(std::sqrt(err) < 1e-8);
  }
}
TEST_CASE("project_warp identities") {  // :124-138
  auto rng = make_rng(18);
  for (int i = 0; i < 50; ++i) {
    const Vec2 x(uniform(rng, -0.5, 0.5), uniform(rng, -0.5, 0.5));
    const double d = uniform(rng, 0.2, 3.0);
    CHECK((project_warp(x, Pose{}, d) - x).norm() == 0.0);
    Pose pose;
    const double tau = uniform(rng, -0.2, 0.5);
    pose.t = Vec3(0, 0, tau);
    CHECK((project_warp(x, pose, d) - x * (1.0 / (1.0 + d * tau))).norm() < 1e-15);
  }
}
TEST_CASE("project_warp equals independent 3D composition") {  // :140-150
  auto rng = make_rng(19);
  for (int i = 0; i < 200; ++i) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    const Pose pose = random_pose(rng, 0.5, 0.3);
    const double d = uniform(rng, 0.3, 2.5);
    const Vec3 v = pose.R * homogeneous(x) + d * pose.t;
    if (v.z < 0.1) continue;
    CHECK((project_warp(x, pose, d) - project(v)).norm() < 1e-15);
  }
}
TEST_CASE("fc_warp_jacobian: zero depth column at identity pose") {  // :152-161
  auto rng = make_rng(20);
  for (int i = 0; i < 200; ++i) {
    const Vec2 x(uniform(rng, -0.5, 0.5), uniform(rng, -0.5, 0.5));
    const double d = uniform(rng, 0.1, 5.0);
    const auto J = fc_warp_jacobian(x, Pose{}, d);
    CHECK(J.image[0][6] == 0.0);
    CHECK(J.image[1][6] == 0.0);
  }
}
TEST_CASE("fc_warp_jacobian matches finite differences") {  // :163-191
  auto rng = make_rng(21);
  int checked = 0;
  while (checked < 200) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    const Pose pose = random_pose(rng, 0.4, 0.3);
    const double d = uniform(rng, 0.3, 2.5);
    if ((pose.R * homogeneous(x) + d * pose.t).z < 0.2) continue;
    ++checked;
    const auto J = fc_warp_jacobian(x, pose, d);
    double fd[2][7];
    const double h = 1e-6;
    for (int c = 0; c < 6; ++c) {
      Vec6 delta{};
      delta[c] = h;
      const Vec2 hi = project_warp(x, pose_boxplus(pose, delta), d);
      delta[c] = -h;
      const Vec2 lo = project_warp(x, pose_boxplus(pose, delta), d);
      fd[0][c] = (hi.x - lo.x) / (2 * h);
      fd[1][c] = (hi.y - lo.y) / (2 * h);
    }
    const Vec2 dh = project_warp(x, pose, d + h) - project_warp(x, pose, d - h);
    fd[0][6] = dh.x / (2 * h);
    fd[1][6] = dh.y / (2 * h);
    double m = 0;
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 7; ++c) m = std::max(m, std::abs(J.image[r][c] - fd[r][c]));
    CHECK(m / std::max(1.0, jac_maxabs(J.image)) < 1e-5);
  }
}
TEST_CASE("fc_warp_jacobian translation-x column at identity") {  // :193-203
  auto rng = make_rng(22);
  for (int i = 0; i < 50; ++i) {
    const Vec2 x(uniform(rng, -0.5, 0.5), uniform(rng, -0.5, 0.5));
    const double d = uniform(rng, 0.2, 3.0);
    const auto J = fc_warp_jacobian(x, Pose{}, d);
    CHECK(approx(J.image[0][3], d, 1e-12));
    CHECK(approx(J.image[1][3], 0.0));
  }
}
TEST_CASE("make_proxy_constants identity and hand example") {  // :205-220
  const auto pc_id = make_proxy_constants(Vec2(0.2, -0.1), Pose{}, 1.0);
  CHECK(approx(pc_id.zbar0, 1.0));
  CHECK((pc_id.M - Mat3::Identity()).norm() < 1e-15);
  Pose pose0;
  pose0.t = Vec3(0, 0, 0.5);
  const auto pc = make_proxy_constants(Vec2(0, 0), pose0, 1.0);
  CHECK(approx(pc.zbar0, 1.5));
  CHECK(approx(pc.M(0, 0), 1.5));
  CHECK(approx(pc.M(1, 1), 1.5));
  CHECK((Vec3(pc.M(0, 2), pc.M(1, 2), pc.M(2, 2)) - Vec3(0, 0, 1.0)).norm() < 1e-15);
}
TEST_CASE("make_proxy_constants algebraic invariant") {  // :222-240
  auto rng = make_rng(23);
  for (int i = 0; i < 100; ++i) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    const Pose pose0 = random_pose(rng, 0.4, 0.3);
    const double d0 = uniform(rng, 0.3, 2.5);
    const Vec3 v = pose0.R * homogeneous(x) + d0 * pose0.t;
    if (v.z < 0.2) continue;
    const auto pc = make_proxy_constants(x, pose0, d0);
    Mat3 Z = pc.zbar0 * Mat3::Identity();
    Z(0, 2) -= pc.t0.x;
    Z(1, 2) -= pc.t0.y;
    Z(2, 2) -= pc.t0.z;
    CHECK((pc.M - pc.R0.transpose() * Z).norm() < 1e-14);
    CHECK(approx(pc.zbar0, v.z / d0, 1e-12));
  }
}
TEST_CASE("proxy warp identity: phi(x; 0) = x") {  // :242-253
  auto rng = make_rng(24);
  for (int i = 0; i < 200; ++i) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    const Pose pose0 = random_pose(rng, 0.4, 0.3);
    const double d0 = uniform(rng, 0.3, 2.5);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.2) continue;
    const auto pc = make_proxy_constants(x, pose0, d0);
    CHECK((proxy_warp_grad_form(x, pc, Vec7{}) - x).norm() < 1e-12);
    CHECK((proxy_warp_update_form(x, pc, Vec7{}) - x).norm() < 1e-12);
  }
}
TEST_CASE("invert_warp undoes the initial warp") {  // :255-266
  auto rng = make_rng(25);
  for (int i = 0; i < 200; ++i) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    const Pose pose0 = random_pose(rng, 0.4, 0.3);
    const double d0 = uniform(rng, 0.3, 2.5);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.2) continue;
    const auto pc = make_proxy_constants(x, pose0, d0);
    CHECK((invert_warp(project_warp(x, pose0, d0), pc) - x).norm() < 1e-10);
  }
}
TEST_CASE("proxy warp forms agree as dp -> 0, with O(dp) discrepancy") {  // :268-294
  auto rng = make_rng(26);
  for (int i = 0; i < 100; ++i) {
    const Vec2 x(uniform(rng, -0.3, 0.3), uniform(rng, -0.3, 0.3));
    const Pose pose0 = random_pose(rng, 0.3, 0.3);
    const double d0 = uniform(rng, 0.5, 2.0);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.3) continue;
    const auto pc = make_proxy_constants(x, pose0, d0);
    const Vec7 dir = rand_dir7(rng);
    auto gap = [&](double e) {
      const Vec7 dp = scale7(dir, e);
      return (proxy_warp_grad_form(x, pc, dp) - proxy_warp_update_form(x, pc, dp)).norm();
    };
    const double g3 = gap(1e-3), g5 = gap(1e-5);
    CHECK(g3 < 10.0 * 1e-3);
    CHECK(g5 < 10.0 * 1e-5);
    if (g5 > 1e-12) CHECK(approx(g3 / g5, 100.0, 0.05));
  }
}
TEST_CASE("proxy warp update form rejects non-positive updated depth") {  // :296-301
  const auto pc = make_proxy_constants(Vec2(0, 0), Pose{}, 0.5);
  Vec7 dp{};
  dp[6] = -0.6;
  CHECK_THROWS_AS(proxy_warp_update_form(Vec2(0, 0), pc, dp), InvalidDepth);
}
TEST_CASE("first-order inverse: quadratic shrinkage of phi compose phi^-1") {  // :303-346
  auto rng = make_rng(27);
  int configs = 0;
  while (configs < 30) {
    const Vec2 x(uniform(rng, -0.3, 0.3), uniform(rng, -0.3, 0.3));
    Pose pose0 = random_pose(rng, 0.3, 0.3);
    if (pose0.t.norm() < 0.1) pose0.t = pose0.t * (0.15 / pose0.t.norm());
    const double d0 = uniform(rng, 0.5, 2.0);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.3) continue;
    ++configs;
    const auto pc = make_proxy_constants(x, pose0, d0);
    const Vec7 dir = rand_dir7(rng);
    std::vector<double> le, lr;
    for (double eps : {1e-2, 1e-3, 1e-4}) {
      const Vec7 dp = scale7(dir, eps);
      const Vec2 y = proxy_warp_update_form(x, pc, dp);
      const double err = (proxy_warp_update_form(y, pc, scale7(dp, -1.0)) - x).norm();
      if (err == 0.0) break;
      le.push_back(std::log10(eps));
      lr.push_back(std::log10(err));
    }
    if (lr.size() < 3) continue;
    double mx = 0, my = 0;
    for (int k = 0; k < 3; ++k) {
      mx += le[k] / 3;
      my += lr[k] / 3;
    }
    double num = 0, den = 0;
    for (int k = 0; k < 3; ++k) {
      num += (le[k] - mx) * (lr[k] - my);
      den += (le[k] - mx) * (le[k] - mx);
    }
    CHECK(approx(num / den, 2.0, 0.05));
  }
}
TEST_CASE("ic_jacobian_row: depth column zero iff t0 is zero") {  // :348-359
  auto rng = make_rng(28);
  for (int i = 0; i < 100; ++i) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    const Pose pose0 = random_pose(rng, 0.4, 0.0);
    const double d0 = uniform(rng, 0.3, 2.5);
    const auto J = ic_jacobian_row(x, make_proxy_constants(x, pose0, d0));
    CHECK(J.image[0][6] == 0.0);
    CHECK(J.image[1][6] == 0.0);
  }
}
TEST_CASE("ic_jacobian_row matches finite differences of the grad form") {  // :361-389
  auto rng = make_rng(29);
  int checked = 0;
  while (checked < 200) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    Pose pose0 = random_pose(rng, 0.4, 0.3);
    if (pose0.t.norm() < 0.1) pose0.t = pose0.t * (0.3 / std::max(pose0.t.norm(), 1e-9));
    const double d0 = uniform(rng, 0.3, 2.5);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.2) continue;
    ++checked;
    const auto pc = make_proxy_constants(x, pose0, d0);
    const auto J = ic_jacobian_row(x, pc);
    CHECK(std::hypot(J.image[0][6], J.image[1][6]) > 0.0);
    double m = 0;
    for (int c = 0; c < 7; ++c) {
      Vec7 dp{};
      dp[c] = 1e-6;
      const Vec2 hi = proxy_warp_grad_form(x, pc, dp);
      dp[c] = -1e-6;
      const Vec2 lo = proxy_warp_grad_form(x, pc, dp);
      m = std::max(m, std::abs((hi.x - lo.x) / 2e-6 - J.image[0][c]));
      m = std::max(m, std::abs((hi.y - lo.y) / 2e-6 - J.image[1][c]));
    }
    CHECK(m / std::max(1.0, jac_maxabs(J.image)) < 1e-5);
  }
}
TEST_CASE("apply_ic_update identities and pure depth update") {  // :391-412
  auto rng = make_rng(30);
  const Pose pose_k = random_pose(rng, 0.4, 0.3);
  const Pose p0 = random_pose(rng, 0.3, 0.3);
  const auto pc = make_proxy_constants(Vec2(0.1, 0.2), p0, 1.2);
  const auto same = apply_ic_update(pose_k, 0.8, pc, Vec7{});
  CHECK((same.first.R - pose_k.R).norm() < 1e-15);
  CHECK((same.first.t - pose_k.t).norm() < 1e-15);
  CHECK(approx(same.second, 0.8));
  Vec7 dp{};
  dp[6] = 0.3;
  const auto two = apply_ic_update(pose_k, 0.8, pc, dp);
  CHECK((two.first.R - pose_k.R).norm() < 1e-15);
  CHECK((two.first.t - pose_k.t).norm() < 1e-15);
  CHECK(approx(two.second, (pc.d0 - 0.3) / pc.d0 * 0.8));
  dp[6] = pc.d0 + 0.1;
  CHECK_THROWS_AS(apply_ic_update(pose_k, 0.8, pc, dp), InvalidDepth);
}
TEST_CASE("apply_ic_update composition is first-order accurate") {  // :414-448
  auto rng = make_rng(31);
  int checked = 0;
  while (checked < 50) {
    const Vec2 x(uniform(rng, -0.3, 0.3), uniform(rng, -0.3, 0.3));
    Pose pose0 = random_pose(rng, 0.3, 0.3);
    if (pose0.t.norm() < 0.1) pose0.t = pose0.t * (0.2 / std::max(pose0.t.norm(), 1e-9));
    const double d0 = uniform(rng, 0.5, 2.0);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.3) continue;
    ++checked;
    const auto pc = make_proxy_constants(x, pose0, d0);
    const Vec7 dir = rand_dir7(rng);
    auto err = [&](double e) {
      const Vec7 dp = scale7(dir, e);
      const auto up = apply_ic_update(pose0, d0, pc, dp);
      const Vec2 a = project_warp(x, up.first, up.second);
      const Vec2 b = project_warp(proxy_warp_grad_form(x, pc, scale7(dp, -1.0)), pose0, d0);
      return (a - b).norm();
    };
    const double e1 = err(1e-3), e2 = err(5e-4);
    if (e2 < 1e-14) continue;
    CHECK(e1 < 10.0 * 1e-3);
    CHECK(approx(e1 / e2, 2.0, 0.15));
  }
}
// Survey §8c caveat: the per-pixel closed-form J row of IcSolver::build
// (solver.cpp:331-349) must equal grad^T * ic_jacobian_row with per-pixel
// constants for P > 1 (the reference pins only 1-px patches).
TEST_CASE("closed-form IC J rows equal grad^T ic_jacobian_row for 3x3 patches") {
  auto scene = render_sequence(small_spec(2, 3));
  ProblemState st = make_state(scene, 1);
  perturb_parameters(st.poses, st.inv_depths, 1e-3, 7);
  IcSolver solver(st, SolverConfig{});
  solver.build();
  const std::vector<double> g = solver.gradient();
  // Rebuild g from first principles with per-pixel proxy constants.
  const TemplateData tpl = build_template(st);
  const ObsList obs = ObsList::from(st);
  const HuberLoss h{0.03};
  const PassResult pass = residual_pass(st, obs, tpl, st.poses, st.inv_depths, h, nullptr);
  const int F = st.num_frames(), N = st.num_points(), P = 9;
  std::vector<double> g2(6 * F + N, 0.0);
  for (int n = 0; n < N; ++n)
    for (int f = 0; f < F; ++f)
      for (int k = 0; k < P; ++k) {
        const size_t idx = (static_cast<size_t>(n) * F + f) * P + k;
        if (!pass.active[idx]) continue;
        const Vec2 x = tpl.norm[n * P + k];
        const Vec2 grad = image_gradient(st.ref, x);
        const auto J = ic_jacobian_row(x, make_proxy_constants(x, st.poses[f], st.inv_depths[n]));
        const double wr = h.weight(pass.r[idx]) * pass.r[idx];
        for (int c = 0; c < 6; ++c) g2[6 * f + c] += (grad.x * J.image[0][c] + grad.y * J.image[1][c]) * wr;
        g2[6 * F + n] += (grad.x * J.image[0][6] + grad.y * J.image[1][6]) * wr;
      }
  double diff = 0;
  for (size_t i = 0; i < g.size(); ++i) diff += (g[i] - g2[i]) * (g[i] - g2[i]);
  CHECK(std::sqrt(diff) < 1e-10 * std::max(1.0, vnorm(g2)));
}

// ============================ image (test_image.cpp) ============================
static Image ramp_image(int w, int h, Intrinsics K) {
  Image img(w, h, K);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) img.at(u, v) = static_cast<double>(u) / w;
  return img;
}
static Image random_image(int w, int h, Intrinsics K, uint64_t seed) {
  Image img(w, h, K);
  auto rng = make_rng(seed);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) img.at(u, v) = uniform(rng, 0.0, 1.0);
  return img;
}
TEST_CASE("intrinsics round trip") {  // :34-41
  const Intrinsics K{525.0, 520.0, 319.5, 239.5};
  auto rng = make_rng(40);
  for (int i = 0; i < 100; ++i) {
    const Vec2 px(uniform(rng, 0, 640), uniform(rng, 0, 480));
    CHECK((K.to_pixel(K.to_normalized(px)) - px).norm() < 1e-12);
  }
}
TEST_CASE("bilinear sampling basics") {  // :43-53
  const Intrinsics K{1, 1, 0, 0};
  Image img(4, 4, K);
  img.at(1, 1) = 0.2;
  img.at(2, 1) = 0.6;
  CHECK(approx(sample_bilinear(img, Vec2(1, 1)), 0.2));
  CHECK(approx(sample_bilinear(img, Vec2(1.5, 1)), 0.4));
}
TEST_CASE("bilinear sampling is exact on a ramp") {  // :55-65
  const Intrinsics K{1, 1, 0, 0};
  const Image img = ramp_image(32, 16, K);
  auto rng = make_rng(41);
  for (int i = 0; i < 200; ++i) {
    const Vec2 px(uniform(rng, 0.0, 30.0), uniform(rng, 0.0, 13.0));
    CHECK(approx(sample_bilinear(img, px), px.x / 32, 1e-12));
  }
}
TEST_CASE("sampling outside the valid area throws") {  // :67-75
  const Intrinsics K{1, 1, 0, 0};
  const Image img = ramp_image(8, 8, K);
  CHECK_THROWS_AS(sample_bilinear(img, Vec2(-0.5, 3)), OutOfBounds);
  CHECK_THROWS_AS(sample_bilinear(img, Vec2(6.5, 3)), OutOfBounds);
  CHECK_THROWS_AS(sample_bilinear(img, Vec2(3, 6.5)), OutOfBounds);
  CHECK(img.in_bounds_px(Vec2(6.0, 6.0)));
  CHECK(!img.in_bounds_px(Vec2(6.01, 6.0)));
}
TEST_CASE("image_gradient of a constant image is zero") {  // :77-85
  const Intrinsics K{100, 100, 15.5, 15.5};
  Image img(32, 32, K);
  for (double& v : img.data()) v = 0.37;
  CHECK(image_gradient(img, K.to_normalized(Vec2(10.2, 20.7))).norm() == 0.0);
}
TEST_CASE("image_gradient of a ramp is the analytic slope") {  // :87-99
  const Intrinsics K{200, 150, 15.5, 15.5};
  const Image img = ramp_image(32, 32, K);
  auto rng = make_rng(42);
  for (int i = 0; i < 100; ++i) {
    const Vec2 px(uniform(rng, 2.0, 28.0), uniform(rng, 2.0, 28.0));
    const Vec2 g = image_gradient(img, K.to_normalized(px));
    CHECK(approx(g.x, K.fx / 32, 1e-10));
    CHECK(approx(g.y, 0.0));
  }
}
TEST_CASE("image_gradient is linear in the image") {  // :101-117
  const Intrinsics K{50, 50, 15.5, 15.5};
  const Image a = random_image(32, 32, K, 7), b = random_image(32, 32, K, 8);
  Image sum(32, 32, K);
  for (size_t i = 0; i < sum.data().size(); ++i) sum.data()[i] = a.data()[i] + b.data()[i];
  auto rng = make_rng(43);
  for (int i = 0; i < 50; ++i) {
    const Vec2 p = K.to_normalized(Vec2(uniform(rng, 2.0, 28.0), uniform(rng, 2.0, 28.0)));
    CHECK((image_gradient(sum, p) - (image_gradient(a, p) + image_gradient(b, p))).norm() < 1e-12);
  }
}
TEST_CASE("image_gradient matches finite differences of the interpolant") {  // :119-140
  const Intrinsics K{60, 45, 15.5, 15.5};
  const Image img = random_image(32, 32, K, 9);
  auto rng = make_rng(44);
  for (int i = 0; i < 100; ++i) {
    const double ux = std::floor(uniform(rng, 2.0, 28.0)) + 0.5;
    const double uy = std::floor(uniform(rng, 2.0, 28.0)) + 0.5;
    const Vec2 p = K.to_normalized(Vec2(ux, uy));
    const Vec2 g = image_gradient(img, p);
    const double hx = 1e-3 / K.fx, hy = 1e-3 / K.fy;
    const double fx = (sample_bilinear(img, p + Vec2(hx, 0)) - sample_bilinear(img, p - Vec2(hx, 0))) / (2 * hx);
    const double fy = (sample_bilinear(img, p + Vec2(0, hy)) - sample_bilinear(img, p - Vec2(0, hy))) / (2 * hy);
    CHECK(approx(g.x, fx, 1e-8));
    CHECK(approx(g.y, fy, 1e-8));
  }
}
TEST_CASE("patch patterns") {  // :142-157
  const auto p0 = PatchPattern::square(0);
  CHECK(p0.offsets.size() == 1);
  CHECK(p0.offsets[0][0] == 0 && p0.offsets[0][1] == 0);
  const auto p1 = PatchPattern::square(1);
  CHECK(p1.offsets.size() == 9);
  CHECK(p1.offsets[0][0] == 0 && p1.offsets[0][1] == 0);
  CHECK(p1.radius() == 1);
  for (size_t i = 0; i < p1.offsets.size(); ++i)
    for (size_t j = i + 1; j < p1.offsets.size(); ++j) CHECK(p1.offsets[i] != p1.offsets[j]);
}

// ============================ solver (test_solver.cpp) ============================
TEST_CASE("Huber weight and loss definitions") {  // :38-56
  const HuberLoss h{0.03};
  CHECK(h.weight(0.0) == 1.0);
  CHECK(h.weight(0.03) == 1.0);
  CHECK(approx(h.weight(0.06), 0.5));
  CHECK(approx(h.weight(-0.06), 0.5));
  CHECK(approx(h.loss(0.01), 0.5 * 0.01 * 0.01));
  CHECK(approx(h.loss(0.1), 0.03 * (0.1 - 0.015)));
  const double eps = 1e-9;
  CHECK(approx(h.loss(0.03 + eps) - h.loss(0.03 - eps), 2 * eps * 0.03, 1e-3));
  for (double r : {0.005, 0.02, 0.05, 0.4, -0.07}) {
    const double fd = (h.loss(r + 1e-7) - h.loss(r - 1e-7)) / 2e-7;
    CHECK(approx(fd, h.weight(r) * r, 1e-6));
  }
}
TEST_CASE("Huber IRLS fixed point matches golden-section minimization") {  // :58-82
  const double gamma = 0.03;
  const HuberLoss h{gamma};
  const std::vector<double> obs = {-0.5, -0.02, 0.0, 0.011, 0.04, 0.3, 0.9};
  auto objective = [&](double x) {
    double e = 0.0;
    for (double b : obs) e += h.loss(x - b);
    return e;
  };
  double x = 0.0;
  for (int it = 0; it < 200; ++it) {
    double num = 0.0, den = 0.0;
    for (double b : obs) {
      const double w = h.weight(x - b);
      num += w * b;
      den += w;
    }
    const double next = num / den;
    if (std::abs(next - x) < 1e-14) break;
    x = next;
  }
  CHECK(approx(x, golden_section_min(objective, -1.0, 1.0, 1e-13), 1e-8));
  CHECK(h.weight(2.0 * gamma) == 0.5);  // acceptance.cpp:377-378
}
TEST_CASE("energy_eval matches the naive double loop") {  // :84-101
  auto scene = render_sequence(small_spec(2, 3));
  ProblemState st = make_state(scene);
  perturb_parameters(st.poses, st.inv_depths, 2e-3, 5);
  const EnergyResult res = energy_eval(st, HuberLoss{0.03});
  CHECK(approx(res.energy, naive_energy(st, 0.03), 1e-12));
  CHECK(res.num_active > 0);
  SceneSpec stat = small_spec(2, 3);
  stat.trajectory.kind = TrajectorySpec::Kind::Dolly;
  stat.trajectory.extent = Vec3(0, 0, 0);
  const ProblemState st0 = make_state(render_sequence(stat));
  CHECK(approx(energy_eval(st0, HuberLoss{0.03}).energy, 0.0));
}
TEST_CASE("energy_eval throws when nothing is in bounds") {  // :103-108
  ProblemState st = make_state(render_sequence(small_spec(2, 3)));
  for (Pose& p : st.poses) p.t = Vec3(50.0, 0.0, 0.0);
  CHECK_THROWS_AS(energy_eval(st, HuberLoss{0.03}), EmptyProblem);
}
TEST_CASE("energy is invariant under the scale gauge") {  // :110-122
  ProblemState st = make_state(render_sequence(small_spec(3, 6)));
  perturb_parameters(st.poses, st.inv_depths, 1e-3, 6);
  const double e0 = energy_eval(st, HuberLoss{0.03}).energy;
  ProblemState scaled = st;
  for (double& d : scaled.inv_depths) d /= 1.7;
  for (Pose& p : scaled.poses) p.t = p.t * 1.7;
  CHECK(approx(energy_eval(scaled, HuberLoss{0.03}).energy, e0, 1e-12));
}
TEST_CASE("Schur-complement solve equals the dense solve") {  // :124-161
  auto rng = make_rng(50);
  const int F = 3, N = 8;
  BlockHessian H;
  H.F = F;
  H.N = N;
  H.pose_pose.assign(F, Mat66{});
  H.depth_depth.assign(N, 0.0);
  H.pose_depth.assign(static_cast<size_t>(N) * F, Vec6{});
  for (int n = 0; n <= N; ++n) H.obs_ptr.push_back(static_cast<int64_t>(n) * F);
  for (int n = 0; n < N; ++n)
    for (int f = 0; f < F; ++f) H.obs_frame.push_back(f);
  for (int n = 0; n < N; ++n)
    for (int f = 0; f < F; ++f)
      for (int k = 0; k < 5; ++k) {
        double row[7];
        for (int c = 0; c < 7; ++c) row[c] = uniform(rng, -1.0, 1.0);
        for (int i = 0; i < 6; ++i)
          for (int j = 0; j < 6; ++j) H.pose_pose[f][6 * i + j] += row[i] * row[j];
        H.depth_depth[n] += row[6] * row[6];
        for (int i = 0; i < 6; ++i) H.pose_depth[n * F + f][i] += row[i] * row[6];
      }
  std::vector<double> g(6 * F + N);
  for (double& v : g) v = uniform(rng, -1.0, 1.0);
  for (double lambda : {1e-6, 1e-2, 1.0}) {
    const auto a = solve_normal_equations_schur(H, g, lambda);
    const auto b = solve_normal_equations_dense(H, g, lambda);
    double d = 0;
    for (size_t i = 0; i < a.size(); ++i) d += (a[i] - b[i]) * (a[i] - b[i]);
    CHECK(std::sqrt(d) < 1e-8 * std::max(1.0, vnorm(b)));
    const auto A = H.dense(lambda);
    const int dim = 6 * F + N;
    double res = 0, asym = 0;
    for (int i = 0; i < dim; ++i) {
      double s = g[i];
      for (int j = 0; j < dim; ++j) {
        s += A[i * dim + j] * a[j];
        asym += std::abs(A[i * dim + j] - A[j * dim + i]);
      }
      res += s * s;
    }
    CHECK(std::sqrt(res) < 1e-8 * vnorm(g));
    CHECK(asym == 0.0);
  }
}
TEST_CASE("one IC Gauss-Newton step equals a dense naive implementation") {  // :163-206
  auto scene = render_sequence(small_spec(2, 3));
  ProblemState st = make_state(scene, 0);
  perturb_parameters(st.poses, st.inv_depths, 1e-3, 7);
  const int F = st.num_frames(), N = st.num_points();
  SolverConfig cfg;
  IcSolver solver(st, cfg);
  solver.build();
  const std::vector<double> dx = solver.compute_step();
  const HuberLoss h{cfg.gamma};
  const EnergyResult res = energy_eval(st, h);
  const auto& K = st.ref.intrinsics();
  const int dim = 6 * F + N;
  std::vector<double> J(static_cast<size_t>(N * F) * dim, 0.0), r(N * F, 0.0), w(N * F, 0.0);
  for (int n = 0; n < N; ++n) {
    const Vec2 x = K.to_normalized(st.anchors_px[n]);
    for (int f = 0; f < F; ++f) {
      const int row = n * F + f;
      if (!res.active[row]) continue;
      const Vec2 grad = image_gradient(st.ref, x);
      const auto Jr = ic_jacobian_row(x, make_proxy_constants(x, st.poses[f], st.inv_depths[n]));
      for (int c = 0; c < 6; ++c) J[row * dim + 6 * f + c] = grad.x * Jr.image[0][c] + grad.y * Jr.image[1][c];
      J[row * dim + 6 * F + n] = grad.x * Jr.image[0][6] + grad.y * Jr.image[1][6];
      r[row] = res.residuals[row];
      w[row] = h.weight(r[row]);
    }
  }
  std::vector<double> H(static_cast<size_t>(dim) * dim, 0.0), g(dim, 0.0);
  for (int i = 0; i < dim; ++i) {
    for (int j = 0; j < dim; ++j) {
      double s = 0;
      for (int q = 0; q < N * F; ++q) s += J[q * dim + i] * w[q] * J[q * dim + j];
      H[i * dim + j] = s + (i == j ? cfg.lambda0 : 0.0);
    }
    for (int q = 0; q < N * F; ++q) g[i] += J[q * dim + i] * (w[q] * r[q]);
  }
  DenseCholesky ch;
  CHECK(ch.compute(H, dim));
  std::vector<double> mg(dim);
  for (int i = 0; i < dim; ++i) mg[i] = -g[i];
  const auto dxn = ch.solve(mg);
  double d = 0;
  for (int i = 0; i < dim; ++i) d += (dx[i] - dxn[i]) * (dx[i] - dxn[i]);
  CHECK(static_cast<int>(dx.size()) == dim);
  CHECK(std::sqrt(d) < 1e-10 * std::max(1.0, vnorm(dxn)));
  // acceptance.cpp:312-314: energy vs naive to 1e-12
  const double naive = naive_energy(st, cfg.gamma);
  CHECK(std::abs(res.energy - naive) / std::max(1.0, naive) < 1e-12);
}
TEST_CASE("zero-noise start converges immediately for both solvers") {  // :208-223
  const ProblemState st = make_state(render_sequence(small_spec(2, 4)));
  SolverConfig cfg;
  const SolveReport fc = fc_solve(st, cfg);
  CHECK(fc.converged);
  CHECK(fc.iterations <= 5);
  const SolveReport ic = ic_solve(st, cfg);
  CHECK(ic.converged);
  CHECK(ic.iterations <= 5);
  CHECK(ic.hessian_builds == 1);
}
TEST_CASE("noisy start: both converge near ground truth, counters correct") {  // :225-249
  ProblemState st = make_state(render_sequence(small_spec(3, 10)));
  perturb_parameters(st.poses, st.inv_depths, 1e-3, 8);
  SolverConfig cfg;
  cfg.record_snapshots = true;
  const SolveReport fc = fc_solve(st, cfg);
  const SolveReport ic = ic_solve(st, cfg);
  CHECK(fc.converged);
  CHECK(ic.converged);
  CHECK(ic.hessian_builds == 1);
  for (size_t i = 1; i < fc.iters.size(); ++i)
    CHECK(fc.iters[i].energy <= fc.iters[i - 1].energy * (1 + 1e-12) + 1e-15);
  for (size_t i = 1; i < ic.iters.size(); ++i)
    CHECK(ic.iters[i].energy <= ic.iters[i - 1].energy * (1 + 1e-12) + 1e-15);
  for (const auto& it : fc.iters) CHECK(it.hessian_builds == it.iter);
  CHECK(std::abs(fc.final_energy - ic.final_energy) <= 0.01 * std::max(fc.final_energy, ic.final_energy));
}
TEST_CASE("flat texture: no-progress convergence, not a crash") {  // :251-264
  ProblemState st = make_state(render_sequence(small_spec(2, 3)));
  for (double& v : st.ref.data()) v = 0.5;
  for (auto& img : st.targets)
    for (double& v : img.data()) v = 0.5;
  const SolveReport ic = ic_solve(st, SolverConfig{});
  CHECK(ic.converged);
  CHECK(ic.iterations <= 1);
}
TEST_CASE("zero initial translation produces a depth-observability warning") {  // :266-278
  ProblemState st = make_state(render_sequence(small_spec(2, 3)));
  st.targets = {st.ref};
  st.poses = {Pose{}};
  IcSolver solver(st, SolverConfig{});
  solver.build();
  CHECK(!solver.warnings().empty());
  if (!solver.warnings().empty())
    CHECK(solver.warnings().front().find("zero initial translation") != std::string::npos);
  for (double dd : solver.hessian().depth_depth) CHECK(dd == 0.0);
}
TEST_CASE("large noise is reported, never thrown") {  // :280-289
  ProblemState st = make_state(render_sequence(small_spec(2, 6)));
  perturb_parameters(st.poses, st.inv_depths, 0.1, 9);
  SolverConfig cfg;
  cfg.max_iters = 50;
  bool threw = false;
  SolveReport ic;
  try {
    ic = ic_solve(st, cfg);
  } catch (...) {
    threw = true;
  }
  CHECK(!threw);
  CHECK(ic.converged || ic.diverged || ic.iterations == cfg.max_iters);
  if (ic.diverged) CHECK(!ic.message.empty());
}

// ============================ synth (test_synth.cpp) ============================
static SceneSpec tiny_spec() {  // test_synth.cpp:14-23
  SceneSpec s;
  s.width = 160;
  s.height = 120;
  s.intrinsics = {130.0, 130.0, 79.5, 59.5};
  s.num_points = 12;
  s.trajectory.frames = 3;
  s.trajectory.span_deg = 6.0;
  return s;
}
TEST_CASE("fbm noise is deterministic and in range") {  // :27-39
  auto rng = make_rng(60);
  for (int i = 0; i < 500; ++i) {
    const double x = uniform(rng, -100.0, 100.0), y = uniform(rng, -100.0, 100.0);
    const double a = fbm_noise(x, y, 4, 7);
    CHECK(a >= 0.0);
    CHECK(a <= 1.0);
    CHECK(fbm_noise(x, y, 4, 7) == a);
    CHECK(fbm_noise(x, y, 4, 8) != a);
  }
}
TEST_CASE("trajectory poses: orbit and dolly") {  // :41-62
  SceneSpec spec = tiny_spec();
  spec.trajectory.frames = 8;
  const auto orbit = trajectory_poses(spec);
  CHECK(orbit.size() == 8);
  for (const auto& p : orbit) {
    CHECK(so3_log(p.R).norm() > 1e-4);
    CHECK(approx(so3_log(p.R).x, 0.0));
    CHECK(approx(so3_log(p.R).z, 0.0));
  }
  spec.trajectory.kind = TrajectorySpec::Kind::Dolly;
  spec.trajectory.extent = Vec3(0.2, 0.0, 0.0);
  const auto dolly = trajectory_poses(spec);
  for (size_t f = 0; f < dolly.size(); ++f) {
    CHECK((dolly[f].R - Mat3::Identity()).norm() == 0.0);
    CHECK(approx(dolly[f].t.x, 0.2 * (f + 1.0) / dolly.size()));
  }
}
TEST_CASE("rendered scene: depth gauge, anchors, and determinism") {  // :64-95
  const SceneSpec spec = tiny_spec();
  const RenderedScene scene = render_sequence(spec);
  CHECK(static_cast<int>(scene.targets.size()) == spec.trajectory.frames);
  CHECK(static_cast<int>(scene.anchors_px.size()) == spec.num_points);
  double mean = 0.0;
  for (double d : scene.inv_depths) mean += d;
  mean /= scene.inv_depths.size();
  CHECK(approx(mean, 1.0, 1e-12));
  const double margin = spec.patch_radius + 3;
  for (const Vec2& a : scene.anchors_px) {
    CHECK(a.x >= margin);
    CHECK(a.x <= spec.width - 1 - margin);
    CHECK(a.y >= margin);
    CHECK(a.y <= spec.height - 1 - margin);
  }
  const RenderedScene again = render_sequence(spec);
  CHECK(again.ref.data() == scene.ref.data());
  for (size_t f = 0; f < scene.targets.size(); ++f) CHECK(again.targets[f].data() == scene.targets[f].data());
  CHECK(again.inv_depths == scene.inv_depths);
}
TEST_CASE("planar dolly produces exact uniform disparity") {  // :97-127
  SceneSpec spec = tiny_spec();
  spec.geometry.kind = GeometrySpec::Kind::Plane;
  spec.geometry.base_depth = 1.0;
  spec.trajectory.kind = TrajectorySpec::Kind::Dolly;
  spec.trajectory.frames = 2;
  spec.trajectory.extent = Vec3(0.2, 0.0, 0.0);
  const RenderedScene scene = render_sequence(spec);
  for (size_t f = 0; f < scene.targets.size(); ++f) {
    const double shift_px = spec.intrinsics.fx * scene.inv_depths[0] * scene.poses[f].t.x;
    int checked = 0;
    for (int v = 20; v < spec.height - 20; v += 11)
      for (int u = 20; u < spec.width - 20; u += 13) {
        if (u - shift_px < 1.0) continue;
        const double expect = scene.ref.sample_px_unchecked(Vec2(u - shift_px, v));
        CHECK(approx(scene.targets[f].at(u, v), expect, 1e-9));
        ++checked;
      }
    CHECK(checked > 50);
  }
}
TEST_CASE("rendering consistency: tiny residuals at ground truth") {  // :129-148
  const RenderedScene scene = render_sequence(tiny_spec());
  ProblemState st = make_state(scene, 1);
  const EnergyResult res = energy_eval(st, HuberLoss{0.03});
  double mean_abs = 0.0;
  for (size_t i = 0; i < res.residuals.size(); ++i)
    if (res.active[i]) mean_abs += std::abs(res.residuals[i]);
  mean_abs /= res.num_active;
  CHECK(mean_abs < 3e-4);
}
TEST_CASE("perturb_parameters: identity at zero, deterministic, calibrated") {  // :150-180
  const RenderedScene scene = render_sequence(tiny_spec());
  auto poses = scene.poses;
  auto depths = scene.inv_depths;
  perturb_parameters(poses, depths, 0.0, 42);
  for (size_t f = 0; f < poses.size(); ++f) {
    CHECK((poses[f].R - scene.poses[f].R).norm() == 0.0);
    CHECK((poses[f].t - scene.poses[f].t).norm() == 0.0);
  }
  CHECK(depths == scene.inv_depths);
  auto p1 = scene.poses, p2 = scene.poses;
  auto d1 = scene.inv_depths, d2 = scene.inv_depths;
  perturb_parameters(p1, d1, 1e-3, 42);
  perturb_parameters(p2, d2, 1e-3, 42);
  CHECK(d1 == d2);
  for (size_t f = 0; f < p1.size(); ++f) CHECK((p1[f].R - p2[f].R).norm() == 0.0);
  std::vector<Pose> none;
  std::vector<double> big(10000, 1.0);
  perturb_parameters(none, big, 1e-3, 1);
  double mean = 0.0, var = 0.0;
  for (double d : big) mean += d - 1.0;
  mean /= big.size();
  for (double d : big) var += (d - 1.0 - mean) * (d - 1.0 - mean);
  CHECK(approx(std::sqrt(var / (big.size() - 1)), 1e-3, 0.05));
}
TEST_CASE("infeasible trajectory names the first out-of-view anchor") {  // :182-197
  SceneSpec spec = tiny_spec();
  spec.trajectory.kind = TrajectorySpec::Kind::Dolly;
  spec.trajectory.extent = Vec3(2.0, 0.0, 0.0);
  CHECK_THROWS_AS(render_sequence(spec), SpecInfeasible);
  try {
    render_sequence(spec);
  } catch (const SpecInfeasible& e) {
    const std::string what = e.what();
    CHECK(what.find("anchor") != std::string::npos);
    CHECK(what.find("frame") != std::string::npos);
  }
}
TEST_CASE("gauge-aligned parameter RMS") {  // :223-255
  const RenderedScene scene = render_sequence(tiny_spec());
  const ParamRms zero = compute_param_rms(scene.poses, scene.inv_depths, scene.poses, scene.inv_depths);
  CHECK(approx(zero.rotation, 0.0));
  CHECK(approx(zero.translation, 0.0));
  CHECK(approx(zero.inv_depth, 0.0));
  auto poses = scene.poses;
  auto depths = scene.inv_depths;
  for (double& d : depths) d /= 1.3;
  for (Pose& p : poses) p.t = p.t * 1.3;
  const ParamRms gauge = compute_param_rms(poses, depths, scene.poses, scene.inv_depths);
  CHECK(gauge.rotation < 1e-12);
  CHECK(gauge.translation < 1e-12);
  CHECK(gauge.inv_depth < 1e-12);
  perturb_parameters(poses, depths, 1e-3, 3);
  const ParamRms moved = compute_param_rms(poses, depths, scene.poses, scene.inv_depths);
  CHECK(moved.rotation > 1e-4);
  CHECK(moved.rotation < 5e-3);
}

// ============================ acceptance.cpp ============================
TEST_CASE("acceptance 1: identity-pose depth column exactly zero over 1000 draws") {  // :57-74
  auto rng = make_rng(101);
  bool ok = true;
  for (int i = 0; i < 1000; ++i) {
    const Vec2 x(uniform(rng, -0.6, 0.6), uniform(rng, -0.6, 0.6));
    const double d = uniform(rng, 0.05, 20.0);
    const auto J = fc_warp_jacobian(x, Pose{}, d);
    if (J.image[0][6] != 0.0 || J.image[1][6] != 0.0) ok = false;
  }
  CHECK(ok);
}
TEST_CASE("acceptance 2: proxy observability and FD over 1000 configs") {  // :81-121
  auto rng = make_rng(102);
  double max_rel = 0.0, min_col = 1e300;
  int done = 0;
  while (done < 1000) {
    const Vec2 x(uniform(rng, -0.4, 0.4), uniform(rng, -0.4, 0.4));
    Pose pose0 = random_pose(rng, 0.4, 0.3);
    if (pose0.t.norm() < 0.1) pose0.t = pose0.t * (0.15 / std::max(pose0.t.norm(), 1e-12));
    const double d0 = uniform(rng, 0.4, 2.5);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.25) continue;
    ++done;
    const auto pc = make_proxy_constants(x, pose0, d0);
    const auto J = ic_jacobian_row(x, pc);
    min_col = std::min(min_col, std::hypot(J.image[0][6], J.image[1][6]));
    double num = 0, den = 0;
    for (int c = 0; c < 7; ++c) {
      Vec7 dp{};
      dp[c] = 1e-6;
      const Vec2 hi = proxy_warp_grad_form(x, pc, dp);
      dp[c] = -1e-6;
      const Vec2 lo = proxy_warp_grad_form(x, pc, dp);
      const double ex = (hi.x - lo.x) / 2e-6 - J.image[0][c], ey = (hi.y - lo.y) / 2e-6 - J.image[1][c];
      num += ex * ex + ey * ey;
      den += J.image[0][c] * J.image[0][c] + J.image[1][c] * J.image[1][c];
    }
    max_rel = std::max(max_rel, std::sqrt(num) / std::max(1.0, std::sqrt(den)));
  }
  CHECK(max_rel <= 1e-4);
  CHECK(min_col > 1e-8);
}
TEST_CASE("acceptance 4: template-side warp identity and round-trip slope") {  // :163-207
  auto rng = make_rng(104);
  double wi = 0, wt = 0, ws = 0;
  int configs = 0;
  while (configs < 200) {
    const Vec2 x(uniform(rng, -0.35, 0.35), uniform(rng, -0.35, 0.35));
    Pose pose0 = random_pose(rng, 0.3, 0.3);
    if (pose0.t.norm() < 0.1) pose0.t = pose0.t * (0.15 / std::max(pose0.t.norm(), 1e-12));
    const double d0 = uniform(rng, 0.5, 2.0);
    if ((pose0.R * homogeneous(x) + d0 * pose0.t).z < 0.3) continue;
    ++configs;
    const auto pc = make_proxy_constants(x, pose0, d0);
    wi = std::max(wi, (proxy_warp_grad_form(x, pc, Vec7{}) - x).norm());
    wi = std::max(wi, (proxy_warp_update_form(x, pc, Vec7{}) - x).norm());
    const Vec2 y = project_warp(x, pose0, d0);
    wt = std::max(wt, (project_warp(invert_warp(y, pc), pose0, d0) - y).norm());
    const Vec7 dir = rand_dir7(rng);
    std::vector<double> le, lr;
    for (double eps : {1e-2, 1e-3, 1e-4}) {
      const Vec7 dp = scale7(dir, eps);
      const Vec2 mid = proxy_warp_update_form(x, pc, dp);
      const double err = (proxy_warp_update_form(mid, pc, scale7(dp, -1.0)) - x).norm();
      if (err == 0.0) break;
      le.push_back(std::log10(eps));
      lr.push_back(std::log10(err));
    }
    if (lr.size() < 3) continue;
    double mx = 0, my = 0;
    for (int k = 0; k < 3; ++k) {
      mx += le[k] / 3.0;
      my += lr[k] / 3.0;
    }
    double num = 0, den = 0;
    for (int k = 0; k < 3; ++k) {
      num += (le[k] - mx) * (lr[k] - my);
      den += (le[k] - mx) * (le[k] - mx);
    }
    ws = std::max(ws, std::abs(num / den - 2.0));
  }
  CHECK(wi < 1e-12);
  CHECK(wt < 1e-10);
  CHECK(ws <= 0.1);
}
TEST_CASE("acceptance 5-7: default scene convergence, Hessian counts, IC wall-clock advantage") {  // :213-286
  const SceneSpec spec;
  const RenderedScene scene = render_sequence(spec);
  ProblemState st = make_state(scene, spec.patch_radius);
  perturb_parameters(st.poses, st.inv_depths, 1e-3, 42);
  SolverConfig cfg;
  const SolveReport fc = fc_solve(st, cfg);
  const SolveReport ic = ic_solve(st, cfg);
  const ParamRms fr = compute_param_rms(fc.final_poses, fc.final_inv_depths, scene.poses, scene.inv_depths);
  const ParamRms ir = compute_param_rms(ic.final_poses, ic.final_inv_depths, scene.poses, scene.inv_depths);
  const double max_rms = std::max({fr.rotation, fr.translation, fr.inv_depth, ir.rotation, ir.translation, ir.inv_depth});
  const double gap = std::abs(fc.final_energy - ic.final_energy) / std::max(fc.final_energy, ic.final_energy);
  CHECK(fc.converged);
  CHECK(ic.converged);
  CHECK(max_rms <= 1e-3);
  CHECK(gap <= 0.01);
  bool fc_per_iter = fc.hessian_builds == fc.iterations;
  for (const auto& it : fc.iters)
    if (it.hessian_builds != it.iter) fc_per_iter = false;
  CHECK(ic.hessian_builds == 1);
  CHECK(ic.hessian_factorizations <= 1 + ic.rejected_steps);
  CHECK(fc_per_iter);
  double fc_best = fc.total_wall_ms, ic_best = ic.total_wall_ms;
  for (int rep = 0; rep < 7; ++rep) {
    fc_best = std::min(fc_best, fc_solve(st, cfg).total_wall_ms);
    ic_best = std::min(ic_best, ic_solve(st, cfg).total_wall_ms);
  }
  std::printf("  [acceptance 7] best-of-8: IC %.1f ms vs FC %.1f ms (%.2fx)\n", ic_best, fc_best,
              fc_best / std::max(ic_best, 1e-9));
  CHECK(ic_best <= 0.5 * fc_best);
}

int main(int argc, char** argv) {
  const std::string filter = argc > 1 ? argv[1] : "";
  int failed_cases = 0, run = 0;
  for (const Case& c : cases()) {
    if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
    g_case = c.name;
    const int before = g_fail_checks;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail_checks;
      std::printf("  unexpected exception in [%s]: %s\n", c.name, e.what());
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool ok = g_fail_checks == before;
    ++run;
    if (!ok) ++failed_cases;
    std::printf("%s  %s (%.2f s)\n", ok ? "PASS" : "FAIL", c.name, s);
  }
  std::printf("%d/%d cases passed\n", run - failed_cases, run);
  return failed_cases == 0 ? 0 : 1;
}
