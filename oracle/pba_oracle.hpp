// ============================================================================
// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// An Eigen-free, single-threaded, fp64 restatement of the reference's
// photometric-bundle-adjustment hot path (/root/reference/proj/src/solver.cpp,
// geometry.cpp, image.cpp; reference test-scene generator synth.cpp).  Every
// function cites the reference file:line it follows.  It exists to CHECK the
// B200 path; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  The product library never links it.
//
// Parity pinning: the reference cannot be compiled here (needs Eigen3, libpng
// and an absent vendor/ tree: proj/CMakeLists.txt:5,12-13) and has no golden
// vectors on disk.  The oracle is pinned by restating the reference's own
// known-answer / property tests (oracle/tests/pins.cpp).
//
// Deliberate deviations (documented in DESIGN.md):
//  * Eigen::LDLT (pivoted) is replaced by an SPD Cholesky LL^T; factorization
//    "failure" = a non-positive or non-finite pivot.
//  * Observation-list extension: a point may be observed in a subset of frames
//    (SURVEY.md Appendix B).  With the dense list every loop visits exactly the
//    reference's (n, f, k) sequence.
// ============================================================================
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

// ---- errors (errors.hpp:9-40) ------------------------------------------------
struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct DegenerateDepth : Error {
  explicit DegenerateDepth(const std::string& w = "degenerate depth") : Error(w) {}
};
struct InvalidDepth : Error {
  explicit InvalidDepth(const std::string& w = "non-positive inverse depth") : Error(w) {}
};
struct OutOfBounds : Error {
  explicit OutOfBounds(const std::string& w = "sample out of bounds") : Error(w) {}
};
struct EmptyProblem : Error {
  explicit EmptyProblem(const std::string& w = "no in-bounds residuals") : Error(w) {}
};
struct SpecInfeasible : Error {
  explicit SpecInfeasible(const std::string& w) : Error(w) {}
};

// ---- tiny fixed-size algebra (stands in for Eigen fixed-size types) ---------
struct Vec2 {
  double x{0}, y{0};
  Vec2() = default;
  Vec2(double a, double b) : x(a), y(b) {}
  Vec2 operator+(const Vec2& o) const { return {x + o.x, y + o.y}; }
  Vec2 operator-(const Vec2& o) const { return {x - o.x, y - o.y}; }
  Vec2 operator*(double s) const { return {x * s, y * s}; }
  double norm() const { return std::sqrt(x * x + y * y); }
};
struct Vec3 {
  double x{0}, y{0}, z{0};
  Vec3() = default;
  Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  Vec3 operator-() const { return {-x, -y, -z}; }
  Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
  Vec3 cross(const Vec3& o) const {
    return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x};
  }
  double squaredNorm() const { return x * x + y * y + z * z; }
  double norm() const { return std::sqrt(squaredNorm()); }
};
inline Vec3 operator*(double s, const Vec3& v) { return v * s; }
inline Vec2 operator*(double s, const Vec2& v) { return v * s; }

struct Mat3 {
  double a[9]{1, 0, 0, 0, 1, 0, 0, 0, 1};  // row-major
  static Mat3 Identity() { return Mat3{}; }
  static Mat3 Zero() {
    Mat3 m;
    for (double& v : m.a) v = 0.0;
    return m;
  }
  double operator()(int r, int c) const { return a[3 * r + c]; }
  double& operator()(int r, int c) { return a[3 * r + c]; }
  Mat3 operator+(const Mat3& o) const {
    Mat3 m;
    for (int i = 0; i < 9; ++i) m.a[i] = a[i] + o.a[i];
    return m;
  }
  Mat3 operator-(const Mat3& o) const {
    Mat3 m;
    for (int i = 0; i < 9; ++i) m.a[i] = a[i] - o.a[i];
    return m;
  }
  Mat3 operator*(double s) const {
    Mat3 m;
    for (int i = 0; i < 9; ++i) m.a[i] = a[i] * s;
    return m;
  }
  Mat3 operator*(const Mat3& o) const {
    Mat3 m;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c)
        m(r, c) = (*this)(r, 0) * o(0, c) + (*this)(r, 1) * o(1, c) + (*this)(r, 2) * o(2, c);
    return m;
  }
  Vec3 operator*(const Vec3& v) const {
    return {a[0] * v.x + a[1] * v.y + a[2] * v.z, a[3] * v.x + a[4] * v.y + a[5] * v.z,
            a[6] * v.x + a[7] * v.y + a[8] * v.z};
  }
  Mat3 transpose() const {
    Mat3 m;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) m(r, c) = (*this)(c, r);
    return m;
  }
  double trace() const { return a[0] + a[4] + a[8]; }
  double norm() const {
    double s = 0;
    for (double v : a) s += v * v;
    return std::sqrt(s);
  }
};
inline Mat3 operator*(double s, const Mat3& m) { return m * s; }

using Vec6 = std::array<double, 6>;
using Vec7 = std::array<double, 7>;
using Mat66 = std::array<double, 36>;  // row-major

// ---- geometry (geometry.hpp / geometry.cpp) ----------------------------------
inline constexpr double kDegenerateDepthEps = 1e-12;  // geometry.hpp:16
inline constexpr double kSmallAngleEps = 1e-8;        // geometry.hpp:19

struct Pose {  // geometry.hpp:25-28
  Mat3 R{Mat3::Identity()};
  Vec3 t{};
};

struct WarpJacobian {  // geometry.hpp:82-85
  double image[2][7]{};
  double pre[3][7]{};
};

struct ProxyConstants {  // geometry.hpp:96-102
  Mat3 R0{Mat3::Identity()};
  Vec3 t0{};
  double d0{1.0};
  double zbar0{1.0};
  Mat3 M{Mat3::Identity()};
};

inline Vec3 homogeneous(const Vec2& x) { return {x.x, x.y, 1.0}; }
Mat3 skew(const Vec3& w);
Mat3 so3_exp(const Vec3& w);
Vec3 so3_log(const Mat3& R);
Pose pose_boxplus(const Pose& pose, const Vec6& delta);
Vec2 project(const Vec3& v);
void project_jacobian(const Vec3& v, double J[2][3]);
Vec2 project_warp(const Vec2& x, const Pose& pose, double inv_depth);
WarpJacobian fc_warp_jacobian(const Vec2& x, const Pose& pose, double inv_depth);
ProxyConstants make_proxy_constants(const Vec2& x, const Pose& pose0, double d0);
Vec2 proxy_warp_grad_form(const Vec2& x, const ProxyConstants& pc, const Vec7& dp);
Vec2 proxy_warp_update_form(const Vec2& x, const ProxyConstants& pc, const Vec7& dp);
Vec2 invert_warp(const Vec2& y, const ProxyConstants& pc);
WarpJacobian ic_jacobian_row(const Vec2& x, const ProxyConstants& pc);
std::pair<Pose, double> apply_ic_update(const Pose& pose_k, double d_k, const ProxyConstants& pc,
                                        const Vec7& dp);

// ---- image (image.hpp / image.cpp) -------------------------------------------
struct Intrinsics {  // image.hpp:14-23
  double fx{1.0}, fy{1.0}, cx{0.0}, cy{0.0};
  Vec2 to_pixel(const Vec2& n) const { return {fx * n.x + cx, fy * n.y + cy}; }
  Vec2 to_normalized(const Vec2& p) const { return {(p.x - cx) / fx, (p.y - cy) / fy}; }
};

class Image {  // image.hpp:28-62
 public:
  Image() = default;
  Image(int w, int h, Intrinsics K = {})
      : width_(w), height_(h), K_(K), data_(static_cast<size_t>(w) * h, 0.0) {}
  int width() const { return width_; }
  int height() const { return height_; }
  const Intrinsics& intrinsics() const { return K_; }
  void set_intrinsics(const Intrinsics& K) { K_ = K; }
  double& at(int u, int v) { return data_[static_cast<size_t>(v) * width_ + u]; }
  double at(int u, int v) const { return data_[static_cast<size_t>(v) * width_ + u]; }
  const std::vector<double>& data() const { return data_; }
  std::vector<double>& data() { return data_; }
  bool in_bounds_px(const Vec2& px) const {  // image.hpp:47-50
    return px.x >= 0.0 && px.x <= width_ - 2 && px.y >= 0.0 && px.y <= height_ - 2;
  }
  double sample_px_unchecked(const Vec2& px) const;  // image.cpp:14-25

 private:
  int width_{0}, height_{0};
  Intrinsics K_{};
  std::vector<double> data_;
};

double sample_bilinear(const Image& img, const Vec2& norm_pt);  // image.cpp:27-34
Vec2 image_gradient(const Image& img, const Vec2& norm_pt);     // image.cpp:36-49

struct PatchPattern {  // image.hpp:74-80
  std::vector<std::array<int, 2>> offsets;
  static PatchPattern square(int radius);  // image.cpp:51-61
  int radius() const;                      // image.cpp:63-69
};

// ---- solver (solver.hpp) ------------------------------------------------------
struct HuberLoss {  // solver.hpp:18-29
  double gamma{0.03};
  double weight(double r) const {
    const double a = std::abs(r);
    return a <= gamma ? 1.0 : gamma / a;
  }
  double loss(double r) const {
    const double a = std::abs(r);
    return a <= gamma ? 0.5 * r * r : gamma * (a - 0.5 * gamma);
  }
};

struct ProblemState {  // solver.hpp:33-43 (+ observation-list extension)
  Image ref;
  std::vector<Image> targets;
  std::vector<Pose> poses;
  std::vector<Vec2> anchors_px;
  std::vector<double> inv_depths;
  PatchPattern patch{PatchPattern::square(1)};
  // Extension: CSR observation list (empty => every point in every frame).
  std::vector<int64_t> obs_ptr;
  std::vector<int32_t> obs_frame;
  int num_frames() const { return static_cast<int>(targets.size()); }
  int num_points() const { return static_cast<int>(anchors_px.size()); }
};

struct SolverConfig {  // solver.hpp:45-54
  double gamma{0.03};
  double threshold_px{5e-3};
  int max_iters{200};
  double lambda0{1e-6};
  int max_bad_steps{8};
  bool normalize_depth_gauge{true};
  bool refresh_ic_hessian{false};
  bool record_snapshots{false};
};

// Observation list derived from a ProblemState (dense when obs_ptr is empty).
struct ObsList {
  std::vector<int64_t> ptr;    // N+1
  std::vector<int32_t> frame;  // N_obs
  int64_t size() const { return static_cast<int64_t>(frame.size()); }
  static ObsList from(const ProblemState& st);
};

struct BlockHessian {  // solver.hpp:59-69
  int F{0}, N{0};
  std::vector<Mat66> pose_pose;   // per frame
  std::vector<double> depth_depth;  // per point
  std::vector<Vec6> pose_depth;   // per observation (dense: n*F + f)
  std::vector<int64_t> obs_ptr;   // extension: observation list of pose_depth
  std::vector<int32_t> obs_frame;
  double lambda{0.0};
  std::vector<double> dense(double lambda_add) const;  // solver.cpp:147-163, (6F+N)^2
};

struct IterationStats {  // solver.hpp:71-80
  int iter{0};
  double energy{0.0};
  double max_update_px{0.0};
  double wall_ms{0.0};
  int hessian_builds{0};
  int hessian_factorizations{0};
  int64_t num_active{0};  // extension
  bool accepted{true};    // extension
  std::vector<Pose> poses;
  std::vector<double> inv_depths;
};

struct SolveReport {  // solver.hpp:82-97
  std::vector<IterationStats> iters;
  bool converged{false};
  bool diverged{false};
  int iterations{0};
  int hessian_builds{0};
  int hessian_factorizations{0};
  int rejected_steps{0};
  double final_energy{0.0};
  double total_wall_ms{0.0};
  int64_t masked_residuals{0};
  std::vector<Pose> final_poses;
  std::vector<double> final_inv_depths;
  std::vector<std::string> warnings;
  std::string message;
};

struct EnergyResult {  // solver.hpp:99-105
  double energy{0.0};
  std::vector<double> residuals;
  std::vector<uint8_t> active;
  int64_t num_active{0};
  int64_t num_out_of_bounds{0};
};

EnergyResult energy_eval(const ProblemState& state, const HuberLoss& huber,
                         const std::vector<uint8_t>* mask = nullptr);

// Internal pieces exposed for the C API and tests.
struct TemplateData {  // solver.cpp:27-31
  std::vector<Vec2> norm;
  std::vector<Vec2> px;
  std::vector<double> val;
};
TemplateData build_template(const ProblemState& st);  // solver.cpp:33-53
struct PassResult {                                   // solver.cpp:55-61
  std::vector<double> r;
  std::vector<uint8_t> active;
  double energy{0.0};
  int64_t num_active{0};
  int64_t num_oob{0};
};
PassResult residual_pass(const ProblemState& st, const ObsList& obs, const TemplateData& tpl,
                         const std::vector<Pose>& poses, const std::vector<double>& depths,
                         const HuberLoss& huber, const std::vector<uint8_t>* mask);
double max_reprojection_update_px(const ProblemState& st, const ObsList& obs,
                                  const TemplateData& tpl, const std::vector<Pose>& old_poses,
                                  const std::vector<double>& old_depths,
                                  const std::vector<Pose>& new_poses,
                                  const std::vector<double>& new_depths);
void normalize_depth_gauge(std::vector<Pose>& poses, std::vector<double>& depths);

// Dense SPD factorization standing in for Eigen::LDLT (see header comment).
struct DenseCholesky {
  int n{0};
  std::vector<double> L;  // row-major lower factor
  bool ok{false};
  bool compute(const std::vector<double>& A, int n);
  std::vector<double> solve(const std::vector<double>& b) const;
};

class IcSolver {  // solver.hpp:115-169
 public:
  explicit IcSolver(ProblemState state, SolverConfig config = {});
  void build();
  std::vector<double> compute_step();
  std::vector<double> gradient();
  SolveReport run();
  const ProblemState& state() const { return state_; }
  const BlockHessian& hessian() const { return hessian_; }
  const std::vector<std::string>& warnings() const { return warnings_; }
  // exposed (private in the reference) for the C API mirror
  void factorize(double lambda);
  std::vector<double> solve_step(const std::vector<double>& g, int depth = 0);
  double lambda() const { return lambda_; }
  const std::vector<Pose>& pose0() const { return pose0_; }
  const std::vector<double>& d0() const { return d0_; }

 private:
  struct ResidualPass {
    std::vector<double> r;
    std::vector<uint8_t> active;
    double energy{0.0};
    int64_t num_active{0};
  };
  ResidualPass eval_residuals(const std::vector<Pose>& poses,
                              const std::vector<double>& depths) const;
  std::vector<double> assemble_gradient(const ResidualPass& pass) const;

  ProblemState state_;
  SolverConfig config_;
  HuberLoss huber_;
  ObsList obs_;
  bool built_{false};
  std::vector<Pose> pose0_;
  std::vector<double> d0_;
  std::vector<Vec2> tpl_norm_;
  std::vector<double> tpl_val_;
  std::vector<Vec7> jrow_;
  std::vector<double> w0_;
  std::vector<uint8_t> mask_;
  BlockHessian hessian_;
  double lambda_{1e-6};
  DenseCholesky reduced_ldlt_;
  std::vector<std::string> warnings_;
  int builds_{0};
  int factorizations_{0};
};

class FcSolver {  // solver.hpp:172-182
 public:
  explicit FcSolver(ProblemState state, SolverConfig config = {});
  SolveReport run();
  // One Hessian/gradient build at the state's parameters (solver.cpp:688-724).
  void build_once(BlockHessian& H, std::vector<double>& g) const;

 private:
  ProblemState state_;
  SolverConfig config_;
};

SolveReport ic_solve(const ProblemState& state, const SolverConfig& config);
SolveReport fc_solve(const ProblemState& state, const SolverConfig& config);

// ---- joint multi-host window + per-frame affine brightness (multihost.cpp) ----------
// OUR model (the reference has no multi-host solver): forwards
// compositional, reduces to fc_solve when every point is hosted in frame 0 and the affine
// parameters are held.  See multihost.cpp for the equations.
struct MhProblem {
  std::vector<Image> images;          // K frames, each with its intrinsics
  std::vector<Pose> poses;            // K (X_i = R_i X_w + t_i); frame 0 held
  std::vector<double> affine_a, affine_b;  // K or empty (= 0); frame 0 held
  std::vector<int> host;              // N host frame of each point
  std::vector<Vec2> anchors_px;       // N, pixels of the host image
  std::vector<double> inv_depths;     // N, in the host camera
  PatchPattern patch{PatchPattern::square(1)};
  std::vector<int64_t> obs_ptr;       // CSR by point of target frames (!= host); empty = all others
  std::vector<int32_t> obs_frame;
  bool optimize_affine{true};
};
struct MhEnergy {
  double energy{0.0};
  int64_t num_active{0}, num_oob{0};
};
struct MhReport {
  SolveReport base;                   // poses of all K frames, depths, counters
  std::vector<double> final_a, final_b;
};
MhEnergy mh_energy(const MhProblem& p, const HuberLoss& huber);
MhReport mh_fc_solve(const MhProblem& p, const SolverConfig& config);
std::vector<double> solve_normal_equations_schur(const BlockHessian& H,
                                                 const std::vector<double>& g, double lambda);
std::vector<double> solve_normal_equations_dense(const BlockHessian& H,
                                                 const std::vector<double>& g, double lambda);

// ---- reference test-scene generator (synth.hpp / synth.cpp) -----------------
struct TextureSpec {  // synth.hpp:14-20
  int octaves{4};
  double base_wavelength_px{64.0};
  double lo{0.15};
  double hi{0.85};
};
struct GeometrySpec {  // synth.hpp:22-28
  enum class Kind { Plane, Heightfield };
  Kind kind{Kind::Heightfield};
  double base_depth{1.0};
  double amplitude{0.1};
  double wavelength_px{160.0};
};
struct TrajectorySpec {  // synth.hpp:30-36
  enum class Kind { Orbit, Dolly };
  Kind kind{Kind::Orbit};
  int frames{20};
  double span_deg{10.0};
  Vec3 extent{0.1, 0.0, 0.0};
};
struct SceneSpec {  // synth.hpp:38-49
  int width{640};
  int height{480};
  Intrinsics intrinsics{525.0, 525.0, 319.5, 239.5};
  TextureSpec texture;
  GeometrySpec geometry;
  TrajectorySpec trajectory;
  int num_points{200};
  int patch_radius{1};
  std::uint64_t seed{7};
  int supersample{2};
};
struct RenderedScene {  // synth.hpp:53-60
  Image ref;
  std::vector<Image> targets;
  std::vector<Pose> poses;
  std::vector<double> inv_depths;
  std::vector<Vec2> anchors_px;
  SceneSpec spec;
};
RenderedScene render_sequence(const SceneSpec& spec);
std::vector<Pose> trajectory_poses(const SceneSpec& spec);
void perturb_parameters(std::vector<Pose>& poses, std::vector<double>& inv_depths, double sigma,
                        std::uint64_t seed);
double fbm_noise(double x, double y, int octaves, std::uint64_t seed);

// Gauge-aligned parameter RMS (scene_io.cpp:169-196), used by convergence pins.
struct ParamRms {
  double rotation{0.0}, translation{0.0}, inv_depth{0.0};
};
ParamRms compute_param_rms(const std::vector<Pose>& est_poses, const std::vector<double>& est_depths,
                           const std::vector<Pose>& gt_poses, const std::vector<double>& gt_depths);

}  // namespace oracle
