// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see pba_oracle.hpp).
// Restates /root/reference/proj/src/geometry.cpp and image.cpp without Eigen.
#include <algorithm>
#include <cmath>

#include "pba_oracle.hpp"

namespace oracle {

// geometry.cpp:7-13
Mat3 skew(const Vec3& w) {
  Mat3 S = Mat3::Zero();
  S(0, 1) = -w.z;
  S(0, 2) = w.y;
  S(1, 0) = w.z;
  S(1, 2) = -w.x;
  S(2, 0) = -w.y;
  S(2, 1) = w.x;
  return S;
}

// geometry.cpp:15-24 (Rodrigues; series below kSmallAngleEps)
Mat3 so3_exp(const Vec3& w) {
  const double theta = w.norm();
  const Mat3 W = skew(w);
  if (theta < kSmallAngleEps) {
    return Mat3::Identity() + W + 0.5 * (W * W);
  }
  const double s = std::sin(theta) / theta;
  const double c = (1.0 - std::cos(theta)) / (theta * theta);
  return Mat3::Identity() + s * W + c * (W * W);
}

// geometry.cpp:26-51
Vec3 so3_log(const Mat3& R) {
  const double tr = R.trace();
  const double cos_theta = std::max(-1.0, std::min(1.0, 0.5 * (tr - 1.0)));
  const double theta = std::acos(cos_theta);
  const Vec3 axis_raw(R(2, 1) - R(1, 2), R(0, 2) - R(2, 0), R(1, 0) - R(0, 1));
  if (theta < kSmallAngleEps) return 0.5 * axis_raw;
  if (theta > M_PI - 1e-6) {
    const Mat3 A = 0.5 * (R + Mat3::Identity());
    Vec3 axis(std::sqrt(std::max(0.0, A(0, 0))), std::sqrt(std::max(0.0, A(1, 1))),
              std::sqrt(std::max(0.0, A(2, 2))));
    int k = 0;
    for (int i = 1; i < 3; ++i)
      if (std::abs(axis[i]) > std::abs(axis[k])) k = i;
    for (int i = 0; i < 3; ++i)
      if (i != k && A(k, i) < 0) axis[i] = -axis[i];
    axis = axis * (1.0 / axis.norm());
    if (axis_raw.dot(axis) < 0) axis = -axis;
    return theta * axis;
  }
  return (theta / (2.0 * std::sin(theta))) * axis_raw;
}

// geometry.cpp:93-98 — left-multiplicative rotation, additive translation
Pose pose_boxplus(const Pose& pose, const Vec6& delta) {
  Pose out;
  out.R = so3_exp(Vec3(delta[0], delta[1], delta[2])) * pose.R;
  out.t = pose.t + Vec3(delta[3], delta[4], delta[5]);
  return out;
}

// geometry.cpp:107-112
Vec2 project(const Vec3& v) {
  if (std::abs(v.z) < kDegenerateDepthEps) throw DegenerateDepth();
  return {v.x / v.z, v.y / v.z};
}

// geometry.cpp:114-123
void project_jacobian(const Vec3& v, double J[2][3]) {
  if (std::abs(v.z) < kDegenerateDepthEps) throw DegenerateDepth();
  const double iz = 1.0 / v.z;
  J[0][0] = iz;
  J[0][1] = 0;
  J[0][2] = -v.x * iz * iz;
  J[1][0] = 0;
  J[1][1] = iz;
  J[1][2] = -v.y * iz * iz;
}

// geometry.cpp:125-127 — <R x~ + d t>
Vec2 project_warp(const Vec2& x, const Pose& pose, double inv_depth) {
  return project(pose.R * homogeneous(x) + inv_depth * pose.t);
}

static void chain_image(const double P[2][3], const double pre[3][7], double out[2][7]) {
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 7; ++c)
      out[r][c] = P[r][0] * pre[0][c] + P[r][1] * pre[1][c] + P[r][2] * pre[2][c];
}

// geometry.cpp:129-139 — pre = [-[R x~]x | d I | t]
WarpJacobian fc_warp_jacobian(const Vec2& x, const Pose& pose, double inv_depth) {
  const Vec3 Rx = pose.R * homogeneous(x);
  const Vec3 v0 = Rx + inv_depth * pose.t;
  WarpJacobian J;
  const Mat3 S = skew(Rx);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) {
      J.pre[r][c] = -S(r, c);
      J.pre[r][3 + c] = (r == c) ? inv_depth : 0.0;
    }
    J.pre[r][6] = pose.t[r];
  }
  double P[2][3];
  project_jacobian(v0, P);
  chain_image(P, J.pre, J.image);
  return J;
}

// geometry.cpp:141-160
ProxyConstants make_proxy_constants(const Vec2& x, const Pose& pose0, double d0) {
  if (d0 <= 0.0) throw InvalidDepth("make_proxy_constants: d0 must be positive");
  const Vec3 v = pose0.R * homogeneous(x) + d0 * pose0.t;
  if (v.z < kDegenerateDepthEps) {
    throw DegenerateDepth("make_proxy_constants: point at/behind proxy plane");
  }
  ProxyConstants pc;
  pc.R0 = pose0.R;
  pc.t0 = pose0.t;
  pc.d0 = d0;
  pc.zbar0 = v.z / d0;
  Mat3 T = Mat3::Zero();
  T(0, 2) = pc.t0.x;
  T(1, 2) = pc.t0.y;
  T(2, 2) = pc.t0.z;
  pc.M = pc.R0.transpose() * (pc.zbar0 * Mat3::Identity() - T);
  return pc;
}

// geometry.cpp:162-168
Vec2 proxy_warp_grad_form(const Vec2& x, const ProxyConstants& pc, const Vec7& dp) {
  const Mat3 Rp = so3_exp(Vec3(dp[0], dp[1], dp[2])) * pc.R0;
  const Vec3 tp = pc.t0 + Vec3(dp[3], dp[4], dp[5]);
  const double dpth = pc.d0 + dp[6];
  return project(pc.M * (Rp * homogeneous(x) + dpth * tp));
}

// geometry.cpp:170-180
Vec2 proxy_warp_update_form(const Vec2& x, const ProxyConstants& pc, const Vec7& dp) {
  const double dpth = pc.d0 + dp[6];
  if (dpth <= 0.0) throw InvalidDepth("proxy_warp_update_form: d' <= 0");
  const Mat3 Rp = so3_exp(Vec3(dp[0], dp[1], dp[2])) * pc.R0;
  const Vec3 v =
      pc.R0.transpose() * ((1.0 / dpth) * (Rp * homogeneous(x)) + Vec3(dp[3], dp[4], dp[5]));
  return project(v);
}

// geometry.cpp:182-184
Vec2 invert_warp(const Vec2& y, const ProxyConstants& pc) {
  return project(pc.R0.transpose() * (pc.zbar0 * homogeneous(y) - pc.t0));
}

// geometry.cpp:186-195
WarpJacobian ic_jacobian_row(const Vec2& x, const ProxyConstants& pc) {
  const Vec3 R0x = pc.R0 * homogeneous(x);
  const Vec3 v0 = pc.M * (R0x + pc.d0 * pc.t0);
  WarpJacobian J;
  const Mat3 MS = pc.M * skew(R0x);
  const Vec3 Mt = pc.M * pc.t0;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) {
      J.pre[r][c] = -MS(r, c);
      J.pre[r][3 + c] = pc.d0 * pc.M(r, c);
    }
    J.pre[r][6] = Mt[r];
  }
  double P[2][3];
  project_jacobian(v0, P);
  chain_image(P, J.pre, J.image);
  return J;
}

// geometry.cpp:197-209
std::pair<Pose, double> apply_ic_update(const Pose& pose_k, double d_k, const ProxyConstants& pc,
                                        const Vec7& dp) {
  const Mat3 dR = so3_exp(Vec3(dp[0], dp[1], dp[2]));
  Pose next;
  next.R = pose_k.R * pc.R0.transpose() * dR.transpose() * pc.R0;
  next.t = pose_k.t - pose_k.R * pc.R0.transpose() * Vec3(dp[3], dp[4], dp[5]);
  const double d_next = ((pc.d0 - dp[6]) / pc.d0) * d_k;
  if (d_next <= 0.0) throw InvalidDepth("apply_ic_update: updated inverse depth <= 0");
  return {next, d_next};
}

// ---- image.cpp -----------------------------------------------------------------

// image.cpp:14-25
double Image::sample_px_unchecked(const Vec2& px) const {
  const int u0 = static_cast<int>(std::floor(px.x));
  const int v0 = static_cast<int>(std::floor(px.y));
  const double a = px.x - u0;
  const double b = px.y - v0;
  const double i00 = at(u0, v0);
  const double i10 = at(u0 + 1, v0);
  const double i01 = at(u0, v0 + 1);
  const double i11 = at(u0 + 1, v0 + 1);
  return (1 - a) * (1 - b) * i00 + a * (1 - b) * i10 + (1 - a) * b * i01 + a * b * i11;
}

// image.cpp:27-34
double sample_bilinear(const Image& img, const Vec2& norm_pt) {
  const Vec2 px = img.intrinsics().to_pixel(norm_pt);
  if (!img.in_bounds_px(px)) throw OutOfBounds("sample_bilinear: pixel out of bounds");
  return img.sample_px_unchecked(px);
}

// image.cpp:36-49 — half-pixel central differences of the interpolant, x fx / fy
Vec2 image_gradient(const Image& img, const Vec2& norm_pt) {
  const Vec2 px = img.intrinsics().to_pixel(norm_pt);
  const Vec2 hu(0.5, 0.0), hv(0.0, 0.5);
  if (!img.in_bounds_px(px - hu) || !img.in_bounds_px(px + hu) || !img.in_bounds_px(px - hv) ||
      !img.in_bounds_px(px + hv)) {
    throw OutOfBounds("image_gradient: footprint out of bounds");
  }
  const double du = img.sample_px_unchecked(px + hu) - img.sample_px_unchecked(px - hu);
  const double dv = img.sample_px_unchecked(px + hv) - img.sample_px_unchecked(px - hv);
  return {du * img.intrinsics().fx, dv * img.intrinsics().fy};
}

// image.cpp:51-61 — (0,0) first, then row-major
PatchPattern PatchPattern::square(int radius) {
  PatchPattern p;
  p.offsets.push_back({0, 0});
  for (int dy = -radius; dy <= radius; ++dy)
    for (int dx = -radius; dx <= radius; ++dx) {
      if (dx == 0 && dy == 0) continue;
      p.offsets.push_back({dx, dy});
    }
  return p;
}

// image.cpp:63-69
int PatchPattern::radius() const {
  int r = 0;
  for (const auto& o : offsets) r = std::max(r, std::max(std::abs(o[0]), std::abs(o[1])));
  return r;
}

}  // namespace oracle
