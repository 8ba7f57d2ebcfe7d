// Host engine: device state of one PBA problem + the reference's LM control flow.
// Control flow mirrors /root/reference/proj/src/solver.cpp line by line (cited);
// every per-pixel / per-point / per-frame computation is a kernel in kernels.cu.
#include <algorithm>
#include <charconv>
#include <unordered_map>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>

#include "engine.hpp"

namespace pba_b200 {

void trace_mark(cudaStream_t s, const char* what) {
  static const bool on = [] {
    const char* e = std::getenv("PBA_TRACE");
    return e && e[0] == '1';
  }();
  if (!on) return;
  static thread_local auto last = std::chrono::steady_clock::now();
  if (s) cudaStreamSynchronize(s);
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[pba trace] %-28s %8.2f ms\n", what,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

namespace {
size_t round_block(size_t b) {
  const size_t g = b >= (size_t(1) << 20) ? (size_t(2) << 20) : 256;
  return (b + g - 1) / g * g;
}
struct BlockCache {
  struct Block {
    void* p;
    cudaEvent_t ev;
  };
  std::mutex m;
  std::unordered_multimap<size_t, Block> free;
  size_t cached = 0;
  static constexpr size_t kCap = size_t(96) << 30;  // bytes parked at most (then returned to the pool)
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();  // never destroyed: blocks may be released at process exit
  return *c;
}
}  // namespace

void* dev_alloc(size_t bytes, cudaStream_t s) {
  const size_t rb = round_block(bytes);
  BlockCache& c = block_cache();
  {
    std::lock_guard<std::mutex> lk(c.m);
    auto it = c.free.find(rb);
    if (it != c.free.end()) {
      const BlockCache::Block b = it->second;
      c.free.erase(it);
      c.cached -= rb;
      ck(cudaStreamWaitEvent(s, b.ev, 0), "block reuse wait");  // after the previous owner's work
      cudaEventDestroy(b.ev);
      return b.p;
    }
  }
  void* p = nullptr;
  ck(cudaMallocAsync(&p, rb, s), "cudaMallocAsync");
  if (rb >= (size_t(64) << 20) && std::getenv("PBA_TRACE"))
    std::fprintf(stderr, "[pba trace] cache miss %.1f MB (cached %.1f GB, %zu blocks)\n", rb / 1048576.0,
                 c.cached / 1073741824.0, c.free.size());
  return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t s) {
  const size_t rb = round_block(bytes);
  BlockCache& c = block_cache();
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(ev, s) != cudaSuccess) {
    if (ev) cudaEventDestroy(ev);
    cudaFreeAsync(p, s);
    return;
  }
  std::lock_guard<std::mutex> lk(c.m);
  if (c.cached + rb > BlockCache::kCap) {
    if (std::getenv("PBA_TRACE"))
      std::fprintf(stderr, "[pba trace] cache full: %.1f MB to the pool\n", rb / 1048576.0);
    cudaEventDestroy(ev);
    cudaFreeAsync(p, s);
    return;
  }
  c.free.emplace(rb, BlockCache::Block{p, ev});
  c.cached += rb;
}

namespace {
thread_local cudaStream_t t_alloc_stream = nullptr;

}  // namespace

cudaStream_t alloc_stream() { return t_alloc_stream; }
void set_alloc_stream(cudaStream_t s) { t_alloc_stream = s; }
void init_memory_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  cudaMemPool_t pool;
  ck(cudaDeviceGetDefaultMemPool(&pool, dev), "mempool");
  uint64_t thr = ~uint64_t(0);
  ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr), "mempool threshold");
  done = true;
}

// =====================================================================================
// construction: upload the ProblemState (solver.hpp:33-43) into the device layout
// =====================================================================================
Engine::Engine(const pba_problem* p, bool deferred) {
  if (!p) throw PbaError(PBA_E_ARG, "null problem");
  if (p->num_frames < 0 || p->num_points < 0) throw PbaError(PBA_E_ARG, "negative sizes");
  if (p->pattern_size < 1 || p->pattern_size > 32 || !p->pattern)
    throw PbaError(PBA_E_ARG, "pattern_size must be in [1, 32]");
  N_ = p->num_points;
  F_ = p->num_frames;
  P_ = p->pattern_size;
  pat_.P = P_;
  for (int k = 0; k < P_; ++k) {
    pat_.dx[k] = p->pattern[2 * k];
    pat_.dy[k] = p->pattern[2 * k + 1];
  }
  if (!p->ref.data || p->ref.width < 4 || p->ref.height < 4) throw PbaError(PBA_E_ARG, "bad reference image");
  if (F_ > 0 && (!p->targets || !p->pose_R || !p->pose_t)) throw PbaError(PBA_E_ARG, "missing frames");
  if (N_ > 0 && (!p->anchors_px || !p->inv_depths)) throw PbaError(PBA_E_ARG, "missing points");
  ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  if (const char* e = std::getenv("PBA_TAB_MIN_OBS")) tab_min_obs_ = std::atoll(e);
  sh_.s = stream_;
  init_memory_pool();
  set_alloc_stream(stream_);

  // ---- images: one fp32 buffer, reference first ----
  std::vector<int64_t> off(F_ + 2, 0);
  off[1] = static_cast<int64_t>(p->ref.width) * p->ref.height;
  for (int f = 0; f < F_; ++f) {
    const pba_image& im = p->targets[f];
    if (!im.data || im.width < 4 || im.height < 4) throw PbaError(PBA_E_ARG, "bad target image");
    off[f + 2] = off[f + 1] + static_cast<int64_t>(im.width) * im.height;
  }
  trace_mark(nullptr, "create: start");
  images_.alloc(off[F_ + 1]);
  ck(cudaMemcpyAsync(images_.p, p->ref.data, off[1] * sizeof(float), cudaMemcpyHostToDevice, stream_), "upload ref");
  ref_ = FrameD{images_.p, p->ref.width, p->ref.height, p->ref.fx, p->ref.fy, p->ref.cx, p->ref.cy};
  frames_h_.resize(F_);
  for (int f = 0; f < F_; ++f) {
    const pba_image& im = p->targets[f];
    frames_h_[f] = FrameD{images_.p + off[f + 1], im.width, im.height, im.fx, im.fy, im.cx, im.cy};
  }
  frames_.alloc(std::max(F_, 1));
  if (F_ > 0)
    ck(cudaMemcpyAsync(frames_.p, frames_h_.data(), F_ * sizeof(FrameD), cudaMemcpyHostToDevice, stream_), "frames");
  // target images go up on a second stream once the observation list and anchors are up
  // (they gate the layout build), so the image upload overlaps the layout build
  ck(cudaStreamCreateWithFlags(&up_stream_, cudaStreamNonBlocking), "upload stream");
  ck(cudaEventCreateWithFlags(&img_done_, cudaEventDisableTiming), "upload event");
  cudaEvent_t obs_up = nullptr;
  ck(cudaEventCreateWithFlags(&obs_up, cudaEventDisableTiming), "obs upload event");
  struct EvRes {
    cudaEvent_t& e;
    ~EvRes() { if (e) cudaEventDestroy(e); }
  } obs_res{obs_up};
  cudaStream_t up = up_stream_;
  auto upload_targets = [&]() {
    ck(cudaEventRecord(obs_up, stream_), "obs upload record");
    ck(cudaStreamWaitEvent(up, obs_up, 0), "obs upload wait");
    for (int f = 0; f < F_; ++f)
      ck(cudaMemcpyAsync(images_.p + off[f + 1], p->targets[f].data, (off[f + 2] - off[f + 1]) * sizeof(float),
                         cudaMemcpyHostToDevice, up),
         "upload target");
    ck(cudaEventRecord(img_done_, up), "upload record");
    images_pending_ = true;
  };

  build_layout(p, upload_targets);
  trace_mark(stream_, "create: layout");
  const int ntiles = ov_.ntiles;
  tval_.alloc(std::max<size_t>(static_cast<size_t>(N_) * P_, 1));
  tgrad_.alloc(std::max<size_t>(static_cast<size_t>(N_) * P_, 1));
  launch_template_values(N_, pat_, ref_, anchor_.p, tval_.p, tgrad_.p, stream_);

  const size_t nN = std::max(N_, 1), nF = std::max(F_, 1), nO = std::max<int64_t>(NO_, 1);
  pose_state_.alloc(nF);
  pose_cur_.alloc(nF);
  pose_cand_.alloc(nF);
  pose0_.alloc(nF);
  d_state_.alloc(nN);
  d_cur_.alloc(nN);
  d_cand_.alloc(nN);
  d0_.alloc(nN);
  mask_[0].alloc(nO + 8);
  mask_[1].alloc(nO + 8);
  scratch_bits_.alloc(nO + 8);
  rec_.alloc(nO);
  rec_g_.alloc(nO);
  gfix_.alloc(nN);
  gscale_.alloc(nN);
  ck(cudaMemsetAsync(gfix_.p, 0, nN * sizeof(unsigned long long), stream_), "gfix zero");
  if (const char* e = std::getenv("PBA_IC_GFIX")) use_gfix_ = e[0] != '0';
  s_n_.alloc(nN);
  dx_n_.alloc(nN);
  xp_.alloc(6 * nF);
  g_tmp_.alloc(6 * nF + nN);
  for (int b = 0; b < 2; ++b) {
    gn_[b].alloc(nN);
    gf_[b].alloc(6 * nF);
    rhs_[b].alloc(6 * nF);
  }
  partial_.alloc(static_cast<size_t>(std::max(ntiles, 1)) * PT_STRIDE);
  partial_cf_.alloc(static_cast<size_t>(std::max(ntiles, 1)) * 8);
  partial_bs_.alloc(static_cast<size_t>(std::max(backsub_blocks(N_), 1)) * 4);
  fscal_.alloc(4 * static_cast<size_t>(std::max(F_, 1)));
  ticket_.alloc(4);
  ck(cudaMemsetAsync(ticket_.p, 0, 4 * sizeof(unsigned int), ticket_.s), "ticket");
  partial_pt_.alloc(static_cast<size_t>(std::max(point_blocks(N_), 1)) * 2);
  partial_mr_.alloc(1024);
  S_.alloc(static_cast<size_t>(36) * nF * nF);
  schur_acc_.alloc(static_cast<size_t>(36) * nF * nF);
  schur_scale_.alloc(6 * nF);
  if (const char* e = std::getenv("PBA_CHOL_INV")) chol_inv_ = e[0] == '1';
  Linv_.alloc(static_cast<size_t>(36) * nF * nF);
  LinvT_.alloc(static_cast<size_t>(36) * nF * nF);
  if (!chol_inv_) {
    chol_flags_.alloc(2 * std::max(chol_tile_flags(6 * F_), 1));
    ck(cudaMemsetAsync(chol_flags_.p, 0, chol_flags_.bytes(), stream_), "chol flags");
  }
  Dinv_.alloc(static_cast<size_t>((6 * nF + 31) / 32) * 32 * 32);
  ytmp_.alloc(6 * nF);
  gauge_.alloc(1);
  status_.alloc(1);
  flags_.alloc(4);
  ck(cudaMallocHost(&status_h_, sizeof(Status)), "pinned");
  ck(cudaMallocHost(&flags_h_, 4 * sizeof(int)), "pinned");

  R_state_.assign(p->pose_R, p->pose_R + 9 * F_);
  t_state_.assign(p->pose_t, p->pose_t + 3 * F_);
  set_params(p->pose_R, p->pose_t, p->inv_depths);
  trace_mark(stream_, "create: buffers+tval+params");
  if (!deferred) {  // the caller's image buffers are free once create returns: finish the upload here
    ensure_images();
    ck(cudaEventSynchronize(img_done_), "upload sync");
  }
  trace_mark(stream_, "create: image upload tail");
}

// Order the handle's stream after the whole target-image upload (deferred handles: before the
// first work that reads the images; the stream syncs of that call then also complete the upload).
void Engine::ensure_images() {
  if (!images_pending_) return;
  ck(cudaStreamWaitEvent(stream_, img_done_, 0), "upload wait");
  images_pending_ = false;
}

Engine::~Engine() {
  if (stream_) cudaStreamSynchronize(stream_);
  if (up_stream_) {
    cudaStreamSynchronize(up_stream_);
    cudaStreamDestroy(up_stream_);
  }
  if (img_done_) cudaEventDestroy(img_done_);
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto& pd : pending_) {
    cudaEventDestroy(pd.a);
    cudaEventDestroy(pd.b);
  }
  if (status_h_) cudaFreeHost(status_h_);
  if (side_) {
    cudaStreamSynchronize(side_);
    cudaStreamDestroy(side_);
    cudaEventDestroy(fork_);
    cudaEventDestroy(join_);
  }
  if (flags_h_) cudaFreeHost(flags_h_);
  set_alloc_stream(stream_);  // members free stream-ordered; sh_ destroys the stream last
}

int64_t Engine::device_bytes() const {  // every device buffer the handle holds
  int64_t b = 0;
  auto add = [&b](const auto&... bufs) { ((b += static_cast<int64_t>(bufs.bytes())), ...); };
  add(images_, frames_, anchor_, anchor_fm_, tval_, tgrad_, pm_ptr_, fm_ptr_, tile_q0_, tile_q1_, pm_frame_, pm2fm_, fm2pm_,
      fm_point_, tile_frame_, ftile_ptr_, tile_order_, uo2q_d_, perm_d_, zero_idx_, perm_tmp_, pose_state_,
      pose_cur_, pose_cand_, pose0_, d_state_, d_cur_, d_cand_, d0_, scratch_bits_, J_, Bic_, Dic_, Hic_, Bpm_,
      rec_, rec_g_, gfix_, gscale_, s_n_, dx_n_, xp_, g_tmp_, r_out_, partial_, partial_cf_, partial_bs_, partial_pt_, partial_mr_,
      fscal_, ticket_, S_, schur_scale_, Linv_, LinvT_, Dinv_, chol_flags_, ytmp_, gauge_, schur_acc_, chunk_pts_,
      schur_chunk_of_, schur_blocks_, schur_chunks_, schur_chunk_off_, schur_dense_, schur_wsort_, dense_row_,
      status_, flags_, xsend_, xrecv_, cf_, gauge_sum_);
  for (int i = 0; i < 2; ++i) add(mask_[i], B_[i], D_[i], H_[i], gn_[i], gf_[i], rhs_[i]);
  return b;
}

// =====================================================================================
// parameters
// =====================================================================================
void Engine::upload_poses(DBuf<PoseD>& dst, const double* R, const double* t) {
  std::vector<PoseD> h(F_);
  for (int f = 0; f < F_; ++f) {
    std::memcpy(h[f].R, R + 9 * f, 9 * sizeof(double));
    std::memcpy(h[f].t, t + 3 * f, 3 * sizeof(double));
  }
  if (F_ > 0) ck(cudaMemcpyAsync(dst.p, h.data(), F_ * sizeof(PoseD), cudaMemcpyHostToDevice, stream_), "poses");
  ck(cudaStreamSynchronize(stream_), "sync");
}
void Engine::upload_depths_user(DBuf<double>& dst, const double* d_user) {
  if (N_ > 0) {  // user order -> internal order on the device
    perm_tmp_.alloc(N_);
    ck(cudaMemcpyAsync(perm_tmp_.p, d_user, N_ * sizeof(double), cudaMemcpyHostToDevice, stream_), "depths");
    launch_permute(N_, perm_d_.p, perm_tmp_.p, dst.p, false, stream_);
  }
  ck(cudaStreamSynchronize(stream_), "sync");
}
void Engine::download_poses(const DBuf<PoseD>& src, double* R, double* t) {
  std::vector<PoseD> h(F_);
  if (F_ > 0) ck(cudaMemcpyAsync(h.data(), src.p, F_ * sizeof(PoseD), cudaMemcpyDeviceToHost, stream_), "poses");
  ck(cudaStreamSynchronize(stream_), "sync");
  for (int f = 0; f < F_; ++f) {
    if (R) std::memcpy(R + 9 * f, h[f].R, 9 * sizeof(double));
    if (t) std::memcpy(t + 3 * f, h[f].t, 3 * sizeof(double));
  }
}
void Engine::download_depths_user(const DBuf<double>& src, double* d_user) {
  if (N_ > 0) {  // internal order -> user order on the device
    perm_tmp_.alloc(N_);
    launch_permute(N_, perm_d_.p, src.p, perm_tmp_.p, true, stream_);
    ck(cudaMemcpyAsync(d_user, perm_tmp_.p, N_ * sizeof(double), cudaMemcpyDeviceToHost, stream_), "depths");
  }
  ck(cudaStreamSynchronize(stream_), "sync");
}

void Engine::set_params(const double* R, const double* t, const double* d) {
  R_state_.assign(R, R + 9 * F_);
  t_state_.assign(t, t + 3 * F_);
  d_state_.alloc(std::max(N_, 1));
  upload_poses(pose_state_, R, t);
  upload_depths_user(d_state_, d);
}

void Engine::get_params(double* R, double* t, double* d) const {
  auto* self = const_cast<Engine*>(this);
  self->download_poses(pose_state_, R, t);
  self->download_depths_user(d_state_, d);
}

// =====================================================================================
// small helpers
// =====================================================================================
cudaEvent_t Engine::ev_begin(int kid) {
  (void)kid;
  if (!prof_) return nullptr;
  cudaEvent_t a;
  if (!ev_pool_.empty()) {
    a = ev_pool_.back();
    ev_pool_.pop_back();
  } else {
    ck(cudaEventCreate(&a), "event");
  }
  ck(cudaEventRecord(a, stream_), "event record");
  return a;
}
void Engine::ev_end(int kid, cudaEvent_t a) {
  if (!prof_ || !a) return;
  cudaEvent_t b;
  if (!ev_pool_.empty()) {
    b = ev_pool_.back();
    ev_pool_.pop_back();
  } else {
    ck(cudaEventCreate(&b), "event");
  }
  ck(cudaEventRecord(b, stream_), "event record");
  pending_.push_back({kid, a, b});
}
void Engine::drain_profile() {
  for (auto& pd : pending_) {
    float ms = 0.f;
    ck(cudaEventSynchronize(pd.b), "event sync");
    ck(cudaEventElapsedTime(&ms, pd.a, pd.b), "elapsed");
    kms_[pd.kid] += ms;
    kcount_[pd.kid] += 1;
    ev_pool_.push_back(pd.a);
    ev_pool_.push_back(pd.b);
  }
  pending_.clear();
}
void Engine::set_profiling(bool on) {
  drain_profile();
  prof_ = on;
  for (int i = 0; i < PBA_K_COUNT; ++i) {
    kcount_[i] = 0;
    kms_[i] = 0.0;
  }
}
void Engine::kernel_times(int64_t* counts, double* total_ms) {
  ck(cudaStreamSynchronize(stream_), "sync");
  drain_profile();
  for (int i = 0; i < PBA_K_COUNT; ++i) {
    if (counts) counts[i] = kcount_[i];
    if (total_ms) total_ms[i] = kms_[i];
  }
}

void Engine::check_template() {
  xcheck(template_ok_, PBA_E_OUT_OF_BOUNDS, "template patch pixel outside reference image");
}

Status Engine::read_status() {
  ck(cudaMemcpyAsync(status_h_, status_.p, sizeof(Status), cudaMemcpyDeviceToHost, stream_), "status");
  ck(cudaMemcpyAsync(flags_h_, flags_.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, stream_), "flags");
  ck(cudaStreamSynchronize(stream_), "sync status");
  ck(cudaGetLastError(), "kernel");
  drain_profile();
  return *status_h_;
}
int Engine::read_flag(int i) {
  ck(cudaMemcpyAsync(flags_h_, flags_.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, stream_), "flags");
  ck(cudaStreamSynchronize(stream_), "sync flags");
  ck(cudaGetLastError(), "kernel");
  drain_profile();
  return flags_h_[i];
}
void Engine::clear_flags() { ck(cudaMemsetAsync(flags_.p, 0, 4 * sizeof(int), stream_), "memset flags"); }

MaxUpdArgs Engine::maxupd_args(const PoseD* pose_old, const PoseD* pose_new, const double* d_old,
                                const double* d_new) const {
  MaxUpdArgs m{};
  m.pose_cur = pose_old;
  m.pose_cand = pose_new;
  m.d_cur = d_old;
  m.d_cand = d_new;
  m.frames = frames_.p;
  m.anchor = anchor_.p;
  m.ref_cx = ref_.cx;
  m.ref_cy = ref_.cy;
  m.ref_ifx = 1.0 / ref_.fx;
  m.ref_ify = 1.0 / ref_.fy;
  m.dx0 = pat_.dx[0];
  m.dy0 = pat_.dy[0];
  return m;
}

ObsArgs Engine::obs_args(double gamma) const {
  ObsArgs a{};
  a.ov = ov_;
  a.ref = ref_;
  a.ref_ifx = 1.0 / ref_.fx;
  a.ref_ify = 1.0 / ref_.fy;
  a.frames = frames_.p;
  a.pat = pat_;
  a.anchor_fm = anchor_fm_.p;
  a.tval = tval_.p;
  for (int k = 0; k < 8 && k < P_; ++k) a.pat_d[k] = make_double2(pat_.dx[k], pat_.dy[k]);
  for (int k = 0; k < 8 && k < P_; ++k) a.pat_n[k] = make_double2(pat_.dx[k] * a.ref_ifx, pat_.dy[k] * a.ref_ify);
  a.tgrad = tgrad_.p;
  a.d0 = d0_.p;
  a.pose0 = pose0_.p;  // frozen IC poses (rows of the factored IC Jacobian)
  a.gamma = gamma;
  a.partial = partial_.p;
  a.rec = rec_.p;
  return a;
}

// ---- rank exchange (point-sharded runs) ----
void Engine::set_exchange(int rank, int world, int64_t n_total, pba_exchange_fn fn, void* ctx) {
  if (fn && (world < 1 || rank < 0 || rank >= world || n_total < N_))
    throw PbaError(PBA_E_ARG, "set_exchange: need 0 <= rank < world and num_points_total >= this shard's points");
  xch_ = Xch{};
  xch_owner_.reset();
  if (!fn) return;
  xch_ = Xch{rank, world, n_total, fn, ctx};
  cf_.alloc(6 * static_cast<size_t>(std::max(F_, 1)));
  gauge_sum_.alloc(1);
}

void Engine::xreduce(const std::vector<XSeg>& segs) {
  XPlan plan{};
  int K = 0;
  for (const XSeg& g : segs) {
    if (!g.p || g.n <= 0) continue;
    if (plan.nseg == 8) throw PbaError(PBA_E_ARG, "xreduce: too many segments");
    K += g.n;
    plan.seg_end[plan.nseg] = K;
    plan.seg_max[plan.nseg] = g.max ? 1 : 0;
    ++plan.nseg;
  }
  if (K == 0) return;
  const size_t W = static_cast<size_t>(xch_.world);
  if (xsend_.n < static_cast<size_t>(K)) xsend_.alloc(K);
  if (xrecv_.n < W * K) xrecv_.alloc(W * K);
  int off = 0;
  for (const XSeg& g : segs) {
    if (!g.p || g.n <= 0) continue;
    ck(cudaMemcpyAsync(xsend_.p + off, g.p, g.n * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "x pack");
    off += g.n;
  }
  if (xch_.fn(xch_.ctx, PBA_X_GATHER, xsend_.p, xrecv_.p, K, stream_) != 0)
    throw PbaError(PBA_E_ARG, "rank exchange (gather) failed");
  launch_xreduce(xrecv_.p, xch_.world, K, plan, xsend_.p, stream_);
  off = 0;
  for (const XSeg& g : segs) {
    if (!g.p || g.n <= 0) continue;
    ck(cudaMemcpyAsync(g.p, xsend_.p + off, g.n * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "x unpack");
    off += g.n;
  }
}

void Engine::xsum_i64(unsigned long long* p, int64_t n) {
  if (n <= 0) return;
  if (xch_.fn(xch_.ctx, PBA_X_SUM_I64, p, nullptr, n, stream_) != 0)
    throw PbaError(PBA_E_ARG, "rank exchange (int64 sum) failed");
}

void Engine::xcheck(bool ok, int code, const std::string& msg) {
  if (!sharded()) {
    if (!ok) throw PbaError(code, msg);
    return;
  }
  gauge_sum_.alloc(1);
  const double bad = ok ? 0.0 : 1.0;
  ck(cudaMemcpyAsync(gauge_sum_.p, &bad, sizeof(double), cudaMemcpyHostToDevice, stream_), "xcheck");
  xreduce({{gauge_sum_.p, 1, false}});
  double tot = 0.0;
  ck(cudaMemcpyAsync(&tot, gauge_sum_.p, sizeof(double), cudaMemcpyDeviceToHost, stream_), "xcheck");
  ck(cudaStreamSynchronize(stream_), "xcheck");
  if (tot > 0.0) throw PbaError(code, ok ? msg + " (on another shard)" : msg);
}

void Engine::finalize(const double* partial, const double* partial_cf, bool bs, bool pt, bool want_h, double* g_f,
                      double* rhs, const double* g_f_in, double* H, bool status, int e_slot) {
  if (sharded() && rhs && partial && !g_f) g_f = g_tmp_.p;  // the rank sum needs g itself
  FinalizeArgs f{};
  f.ov = ov_;
  f.partial = partial;
  f.partial_cf = partial_cf;
  f.partial_bs = bs ? partial_bs_.p : nullptr;
  f.nbs = backsub_blocks(N_);
  f.partial_pt = pt ? partial_pt_.p : nullptr;
  f.npt = point_blocks(N_);
  f.want_h = want_h ? 1 : 0;
  f.g_f = g_f;
  f.rhs = rhs;
  f.g_f_in = g_f_in;
  f.H = H;
  f.status = status ? status_.p : nullptr;
  f.fscal = fscal_.p;
  f.ticket = ticket_.p + 1;
  f.e_slot = e_slot;
  if (sharded()) {  // rhs = -g + c_f is formed from the rank sums of g and c_f
    f.rhs = nullptr;
    f.cf_out = rhs ? cf_.p : nullptr;
  }
  const auto e = ev_begin(PBA_K_REDUCE);
  launch_finalize(f, stream_);
  if (sharded()) {
    double* st = status ? reinterpret_cast<double*>(status_.p) : nullptr;
    static_assert(sizeof(Status) == 8 * sizeof(double), "Status layout");
    xreduce({{partial ? g_f : nullptr, 6 * F_, false},
             {rhs ? cf_.p : nullptr, 6 * F_, false},
             {(want_h && partial) ? H : nullptr, 21 * F_, false},
             {st, 3, false},                          // energy, #active, #oob
             {st ? st + 3 : nullptr, 1, true},        // max reprojection update
             {st ? st + 4 : nullptr, 4, false}});     // sum d, #invalid, #non-finite, |g_n|^2
    if (rhs) launch_rhs(6 * F_, g_f ? g_f : g_f_in, cf_.p, rhs, stream_);
  }
  ev_end(PBA_K_REDUCE, e);
}

// =====================================================================================
// energy_eval (solver.cpp:229-244)
// =====================================================================================
void Engine::energy(double gamma, const uint8_t* mask, pba_energy_result* out, double* residuals, uint8_t* active) {
  check_template();
  ic_.init_from_build = false;  // the pass overwrites the tile partials
  ensure_images();
  ObsArgs a = obs_args(gamma);
  a.pose_eval = pose_state_.p;
  a.active_out = scratch_bits_.p;
  a.d_eval = d_state_.p;
  if (mask) {
    DBuf<uint32_t> mb;
    mb.alloc(std::max<int64_t>(NO_, 1) + 8);
    mask_to_bits(mask, mb.p);
    a.mask_in = mb.p;
    if (residuals) {
      r_out_.alloc(std::max<int64_t>(NO_ * P_, 1));
      ck(cudaMemsetAsync(r_out_.p, 0, r_out_.bytes(), stream_), "memset r");
      a.r_out = r_out_.p;
    }
    const auto e = ev_begin(PBA_K_OBS_PASS);
    launch_obs(OBS_ENERGY, a, stream_);
    ev_end(PBA_K_OBS_PASS, e);
    finalize(partial_.p, nullptr, false, false, false, nullptr, nullptr, nullptr, nullptr, true);
    ck(cudaStreamSynchronize(stream_), "sync");
  } else {
    if (residuals) {
      r_out_.alloc(std::max<int64_t>(NO_ * P_, 1));
      ck(cudaMemsetAsync(r_out_.p, 0, r_out_.bytes(), stream_), "memset r");
      a.r_out = r_out_.p;
    }
    const auto e = ev_begin(PBA_K_OBS_PASS);
    launch_obs(OBS_ENERGY, a, stream_);
    ev_end(PBA_K_OBS_PASS, e);
    finalize(partial_.p, nullptr, false, false, false, nullptr, nullptr, nullptr, nullptr, true);
  }
  const Status s = read_status();
  if (s.num_active == 0) throw PbaError(PBA_E_EMPTY_PROBLEM, "no in-bounds residuals");
  if (out) {
    out->energy = s.energy;
    out->num_active = static_cast<int64_t>(s.num_active);
    out->num_out_of_bounds = static_cast<int64_t>(s.num_oob);
  }
  if (residuals) rows_to_user(r_out_.p, P_, residuals);
  if (active) bits_to_user(scratch_bits_.p, active);
}

// =====================================================================================
// IC pieces
// =====================================================================================
void Engine::ic_eval(const PoseD* pose, const double* d, const uint32_t* mask_in, uint32_t* active_out, int buf,
                     double lambda, const PoseD* pose_old, const double* d_old) {
  // eval_residuals + assemble_gradient (solver.cpp:436-468) + solve_step rhs (:407-416)
  ic_.init_from_build = false;  // the pass overwrites the tile partials and the g_n records
  ObsArgs a = obs_args(ic_.cfg.gamma);
  a.pose_eval = pose;
  a.pose_old = pose_old;
  a.d_eval = d;
  a.d_old = d_old;
  a.mask_in = mask_in;
  a.active_out = active_out;
  a.Jm = J_.p;
  a.rec_g = rec_g_.p;
  if (use_gfix_) {
    a.gfix = gfix_.p;
    a.gscale = gscale_.p;
    a.gfix_bad = flags_.p + 3;
    ck(cudaMemsetAsync(flags_.p + 3, 0, sizeof(int), stream_), "gfix flag");
  }
  last_ic_eval_ = IcEvalArgs{pose, d, mask_in, active_out, buf, lambda, pose_old, d_old};
  // Large problems read the frame-uniform records from kernel-parameter frame tables (one host
  // read-back of the evaluation poses per pass); small, launch-bound ones keep the shared-memory
  // path and avoid the mid-iteration synchronisation.
  const bool use_tab = NO_ >= tab_min_obs_;
  if (use_tab) build_frame_tabs(pose);
  auto e = ev_begin(PBA_K_OBS_PASS);
  if (use_tab) {
    if (!side_) {
      ck(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "side stream");
      ck(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "fork event");
      ck(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming), "join event");
    }
    launch_obs_ic_tab(a, tabs_.data(), static_cast<int>(tabs_.size()), frame_recs_.p, stream_, side_, fork_, join_);
  } else {
    launch_obs(OBS_IC, a, stream_);
  }
  ev_end(PBA_K_OBS_PASS, e);
  PointArgs pa{ov_, PT_GRAD, rec_.p, gn_[buf].p, Dic_.p, lambda, s_n_.p, partial_pt_.p};
  pa.rec_g = rec_g_.p;
  if (use_gfix_) {
    pa.gfix = gfix_.p;
    pa.gscale = gscale_.p;
  }
  e = ev_begin(PBA_K_REDUCE);
  launch_point(pa, stream_);
  const MaxUpdArgs mu = maxupd_args(pose_old, pose, d_old, d);
  launch_cf(ov_, Bic_.p, s_n_.p, partial_cf_.p, stream_, pose_old ? &mu : nullptr);
  ev_end(PBA_K_REDUCE, e);
  finalize(partial_.p, partial_cf_.p, pose_old != nullptr, true, false, gf_[buf].p, rhs_[buf].p, nullptr, nullptr,
           true);
}

// IcSolver::run's initial pass (solver.cpp:487-495) evaluates the residuals at (pose0, d0) under the
// build's mask with fresh weights: exactly what the build pass evaluated.  The build pass therefore
// also sums J^T W r per frame (tile partials, PT_G), the g_n terms per observation (rec_g), and the
// energy and count of the masked pixels (slots PT_MAXUPD, + 1); this forms the gradient, the Schur
// rhs and the status from them without another observation pass (2.5 ms at C4).  The mask is
// unchanged (every masked pixel is active at the build point), so the mask buffers do not flip.
void Engine::ic_initial_from_build() {
  PointArgs pa{ov_, PT_GRAD, rec_.p, gn_[0].p, Dic_.p, ic_.lambda, s_n_.p, partial_pt_.p};
  pa.rec_g = rec_g_.p;  // per-observation records and the point-major gather (the fixed-point scales
                        // of the later passes are set by the build itself)
  const auto e = ev_begin(PBA_K_REDUCE);
  launch_point(pa, stream_);
  launch_cf(ov_, Bic_.p, s_n_.p, partial_cf_.p, stream_, nullptr);
  ev_end(PBA_K_REDUCE, e);
  finalize(partial_.p, partial_cf_.p, false, true, false, gf_[0].p, rhs_[0].p, nullptr, nullptr, true, PT_MAXUPD);
}

// Status of the last IC pass.  The fixed-point g_n sums hold every term whose magnitude the build's
// bound covers; a non-finite term (NaN texels) or one beyond the bound raises flag 3, and the pass
// is then re-run with the per-observation records and point-major gather (exact for any value),
// which this handle keeps using from then on.
Status Engine::ic_read_status() {
  Status s = read_status();
  if (!use_gfix_) return s;
  bool bad = flags_h_[3] != 0;
  if (sharded()) {  // the same decision on every rank (the re-run pass exchanges again)
    gauge_sum_.alloc(1);
    const double v = bad ? 1.0 : 0.0;
    ck(cudaMemcpyAsync(gauge_sum_.p, &v, sizeof(double), cudaMemcpyHostToDevice, stream_), "gfix flag");
    xreduce({{gauge_sum_.p, 1, false}});
    double tot = 0.0;
    ck(cudaMemcpyAsync(&tot, gauge_sum_.p, sizeof(double), cudaMemcpyDeviceToHost, stream_), "gfix flag");
    ck(cudaStreamSynchronize(stream_), "gfix flag");
    bad = tot > 0.0;
  }
  if (bad) {
    use_gfix_ = false;
    const IcEvalArgs& e = last_ic_eval_;
    ic_eval(e.pose, e.d, e.mask_in, e.active_out, e.buf, e.lambda, e.pose_old, e.d_old);
    s = read_status();
  }
  return s;
}

// Frame tables of the IC pass (kTabFrames frames per launch): the chunk geometry is fixed per
// handle; the records are built on the device from the evaluation poses (no host read-back) and
// copied into constant memory by launch_obs_ic_tab on the launching stream.
void Engine::build_frame_tabs(const PoseD* pose_d) {
  const int ntab = (F_ + kTabFrames - 1) / kTabFrames;
  if (static_cast<int>(tabs_.size()) != ntab) {
    tabs_.resize(ntab);
    for (int i = 0; i < ntab; ++i) {
      FrameTab& T = tabs_[i];
      T.f0 = i * kTabFrames;
      T.nf = std::min(kTabFrames, F_ - T.f0);
      T.tile0 = ftile_ptr_h_[T.f0];
      T.ntiles = ftile_ptr_h_[T.f0 + T.nf] - T.tile0;
      T.slot = i % kTabSlots;
    }
  }
  frame_recs_.alloc(std::max(F_, 1));
  launch_frame_recs(F_, pose_d, pose0_.p, frames_.p, frame_recs_.p, stream_);
}

void Engine::ic_rescale_rhs(int buf, double lambda) {
  PointArgs pa{ov_, PT_RESCALE, rec_.p, gn_[buf].p, Dic_.p, lambda, s_n_.p, partial_pt_.p};
  const auto e = ev_begin(PBA_K_REDUCE);
  launch_point(pa, stream_);
  launch_cf(ov_, Bic_.p, s_n_.p, partial_cf_.p, stream_);
  ev_end(PBA_K_REDUCE, e);
  finalize(nullptr, partial_cf_.p, false, false, false, nullptr, rhs_[buf].p, gf_[buf].p, nullptr, false);
}

// User indices (ascending) of the points with D_n == 0.
// D_n == 0 points (solver.cpp:359-364): compacted on the device at the build (count only); the
// user-order list is downloaded and sorted when a warning text is first requested.
int64_t Engine::zero_depth_points(const double* D) {
  if (N_ == 0) return 0;
  return launch_zero_d(N_, D, perm_d_.p, zero_idx_.p, stream_);
}

const std::vector<int32_t>& Engine::zero_d_list() const {
  if (!ic_.zero_d_ready) {
    ic_.zero_d.resize(static_cast<size_t>(ic_.zero_d_count));
    if (ic_.zero_d_count > 0) {  // compacted unordered by k_zero_d: sort the user indices on the device
      sort_i32(zero_idx_.p, static_cast<int>(ic_.zero_d_count), stream_);
      ck(cudaMemcpyAsync(ic_.zero_d.data(), zero_idx_.p, ic_.zero_d_count * sizeof(int32_t), cudaMemcpyDeviceToHost,
                         stream_), "zero-D list");
      ck(cudaStreamSynchronize(stream_), "zero-D sync");
    }
    ic_.zero_d_ready = true;
  }
  return ic_.zero_d;
}

int64_t Engine::warning_points(int32_t* out, int64_t cap) const {
  const std::vector<int32_t>& zd = zero_d_list();
  if (out && cap > 0) std::memcpy(out, zd.data(), std::min<int64_t>(cap, static_cast<int64_t>(zd.size())) * sizeof(int32_t));
  return static_cast<int64_t>(zd.size());
}

// Dense Schur chunk scratch: allocated when a solver is built (not inside a timed factorization).
void Engine::alloc_schur() {
  if (schur_plan_.nblocks > 0 && !schur_plan_.dense) {
    schur_dense_.alloc(static_cast<size_t>(std::max<int64_t>(schur_dense_elems_, 1)));
    schur_wsort_.alloc(static_cast<size_t>(std::max(schur_plan_.npts, 1)));
    schur_plan_.dense = schur_dense_.p;
    schur_plan_.wsort = schur_wsort_.p;
    // slots of frames a point does not observe stay zero: the passes only ever write observed slots
    ck(cudaMemsetAsync(schur_dense_.p, 0, static_cast<size_t>(std::max<int64_t>(schur_dense_elems_, 1)) * sizeof(double),
                       stream_), "dense zero");
    dense_row_.alloc(static_cast<size_t>(std::max(N_, 1)));
    launch_dense_rows(schur_plan_, dense_row_.p, stream_);
  }
}

// The Hessian-building passes write each b_n block into its Schur chunk row as well (no separate
// densify kernel: FC saves it every iteration, IC at the build); the dense rows then hold B_out.
void Engine::fuse_dense(ObsArgs& a) {
  alloc_schur();
  a.B_dense = schur_plan_.dense;
  a.dense_row = dense_row_.p;
  dense_B_ = a.B_dense ? a.B_out : nullptr;
}

bool Engine::factor_reduced(const double* H, const double* B, const double* D, double lambda) {
  const int n = 6 * F_;
  clear_flags();
  auto e = ev_begin(PBA_K_SCHUR);
  alloc_schur();
  const bool densify = dense_B_ != B;  // the dense blocks depend on B only (not on D or lambda)
  launch_schur_acc(ov_, H, B, D, lambda, schur_scale_.p, schur_acc_.p, &schur_plan_, densify, stream_,
                   schur_scale_in_);
  if (sharded()) xsum_i64(schur_acc_.p, 36 * static_cast<int64_t>(F_) * F_);  // exact: fixed point
  launch_schur_final(ov_, H, lambda, schur_scale_.p, schur_acc_.p, S_.p, stream_);
  dense_B_ = B;
  ev_end(PBA_K_SCHUR, e);
  e = ev_begin(PBA_K_CHOLESKY);
  if (chol_inv_) {  // env PBA_CHOL_INV=1: the grid-barrier factor + inverse kernel (round-1 path)
    launch_chol_inv(S_.p, n, Dinv_.p, Linv_.p, LinvT_.p, flags_.p, ticket_.p + 2, stream_);  // L, L^-1, L^-T
  } else {          // dataflow over the tiles: L in place, Dinv, L^-1 and L^-T
    launch_chol_tiles(S_.p, n, Dinv_.p, Linv_.p, LinvT_.p, chol_flags_.p, ++chol_epoch_, flags_.p, stream_);
  }
  ev_end(PBA_K_CHOLESKY, e);
  if (read_flag(0) != 0) return false;
  return true;
}

// IcSolver::factorize (solver.cpp:370-402)
void Engine::ic_factorize_loop(double lambda) {
  for (int attempt = 0; attempt < 60; ++attempt) {
    ++ic_.factorizations;
    if (factor_reduced(Hic_.p, Bic_.p, Dic_.p, lambda)) {
      ic_.lambda = lambda;
      return;
    }
    lambda *= 10.0;
  }
  throw PbaError(PBA_E_SINGULAR_HESSIAN, "SingularHessian: damping retries exhausted");
}

void Engine::solve_xp(const double* rhs) {
  const auto e = ev_begin(PBA_K_TRISOLVE);
  if (F_ > 0) launch_trisolve(Linv_.p, LinvT_.p, 6 * F_, rhs, ytmp_.p, xp_.p, flags_.p + 1, stream_);
  ev_end(PBA_K_TRISOLVE, e);
}

static const char kZeroD[] = ": zero depth Hessian entry (unobservable depth)";

std::string Engine::warning(int64_t i) const {
  if (i < static_cast<int64_t>(ic_.warnings.size())) return ic_.warnings[i];
  return "point " + std::to_string(zero_d_list()[i - ic_.warnings.size()]) + kZeroD;
}

const std::string& Engine::warnings_text() const {
  if (wtext_ok_) return wtext_;
  wtext_.clear();
  const std::vector<int32_t>& zd = zero_d_list();
  wtext_.reserve(ic_.warnings.size() * 80 + zd.size() * (sizeof(kZeroD) + 16));
  for (const auto& w : ic_.warnings) {
    if (!wtext_.empty()) wtext_ += '\n';
    wtext_ += w;
  }
  char num[16];
  for (const int32_t u : zd) {
    if (!wtext_.empty()) wtext_ += '\n';
    wtext_ += "point ";
    const auto r = std::to_chars(num, num + sizeof(num), u);
    wtext_.append(num, r.ptr);
    wtext_.append(kZeroD, sizeof(kZeroD) - 1);
  }
  wtext_ok_ = true;
  return wtext_;
}

// IcSolver::build (solver.cpp:254-368)
void Engine::ic_build(const pba_config* cfg) {
  ic_ = SolverState{};
  wtext_ok_ = false;
  if (cfg) {
    ic_.cfg = *cfg;
  } else {
    pba_config_default(&ic_.cfg);
  }
  ic_.lambda = ic_.cfg.lambda0;
  check_template();
  trace_mark(stream_, "ic_build:   template check");
  if (F_ > 0) ck(cudaMemcpyAsync(pose0_.p, pose_state_.p, F_ * sizeof(PoseD), cudaMemcpyDeviceToDevice, stream_), "p0");
  if (N_ > 0) ck(cudaMemcpyAsync(d0_.p, d_state_.p, N_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_), "d0");
  for (int f = 0; f < F_; ++f) {  // :265-271
    const double* t = &t_state_[3 * f];
    if (std::sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]) < 1e-9)
      ic_.warnings.push_back("frame " + std::to_string(f) +
                             ": zero initial translation, inverse depth unobservable from this frame");
  }
  const size_t nO = std::max<int64_t>(NO_, 1);
  if (N_ > 0) ck(cudaMemsetAsync(gfix_.p, 0, N_ * sizeof(unsigned long long), stream_), "gfix zero");  // no stale sums
  {  // Frozen IC rows: rebuilt in every pass from the per-(point, pixel) template gradients (no
     // per-pixel store; the pass is not HBM-bound, so this costs no time and saves 24 B/px of HBM),
     // or, PBA_IC_RECOMPUTE=0, stored factored as m (24 B per pixel) when that fits comfortably.
    const size_t jm_bytes = static_cast<size_t>(std::max<int64_t>(jm_doubles(NO_, P_), 1)) * sizeof(double);
    // cudaMemGetInfo only when the stored variant is asked for: it intermittently costs 20-40 ms
    // with a large stream-ordered pool resident (measured inside ic_solve at C4)
    const char* env = std::getenv("PBA_IC_RECOMPUTE");
    size_t free_b = 0, total_b = 0;
    if (env && env[0] == '0') cudaMemGetInfo(&free_b, &total_b);
    const bool store = env && env[0] == '0' && jm_bytes <= free_b / 3;
    if (store) J_.alloc(jm_bytes / sizeof(double));
    else J_.release();
  }
  trace_mark(stream_, "ic_build:   meminfo");
  Bic_.alloc(6 * nO);
  Dic_.alloc(std::max(N_, 1));
  Hic_.alloc(21 * std::max(F_, 1));
  trace_mark(stream_, "ic_build:   B/D/H alloc");

  ObsArgs a = obs_args(ic_.cfg.gamma);
  a.pose_eval = pose0_.p;
  a.pose0 = pose0_.p;
  a.d_eval = d0_.p;
  a.active_out = mask_[0].p;
  a.Jmw = J_.p;
  a.B_out = Bic_.p;
  Bpm_.alloc(6 * nO);
  a.Bpm_out = Bpm_.p;  // point-major copy written by the pass itself
  a.fm2pm = fm2pm_.p;
  a.rec_g = rec_g_.p;  // the initial pass's g_n terms (ic_initial_from_build)
  fuse_dense(a);
  trace_mark(stream_, "ic_build: setup+alloc");
  ensure_images();
  auto e = ev_begin(PBA_K_IC_BUILD);
  launch_obs(OBS_BUILD, a, stream_);
  ev_end(PBA_K_IC_BUILD, e);
  trace_mark(stream_, "ic_build: build pass");
  PointArgs pa{ov_, PT_DONLY, rec_.p, nullptr, Dic_.p, 0.0, nullptr, partial_pt_.p};
  pa.gscale = gscale_.p;  // fixed-point scales of the IC g_n sums
  pa.gbound = ic_.cfg.gamma;
  if (const char* e = std::getenv("PBA_IC_GFIX_EXP")) pa.gexp = std::atoi(e);  // tests: force the fallback
  e = ev_begin(PBA_K_REDUCE);
  launch_point(pa, stream_);
  ev_end(PBA_K_REDUCE, e);
  finalize(partial_.p, nullptr, false, false, true, nullptr, nullptr, nullptr, Hic_.p, true);
  trace_mark(stream_, "ic_build: D pass");
  alloc_schur();
  trace_mark(stream_, "ic_build: schur alloc");
  const Status s = read_status();
  if (s.num_active == 0) throw PbaError(PBA_E_EMPTY_PROBLEM, "no in-bounds residuals");  // :275
  ic_.mcur = 0;
  ic_.zero_d_count = zero_depth_points(Dic_.p);  // :359-364 (list fetched on request)
  wtext_ok_ = false;
  ic_.builds = 1;
  trace_mark(stream_, "ic_build: D, B copy, warnings");
  ic_factorize_loop(ic_.lambda);
  ic_.built = true;
  ic_.init_from_build = !(std::getenv("PBA_IC_INIT_FROM_BUILD") && std::getenv("PBA_IC_INIT_FROM_BUILD")[0] == '0');
  trace_mark(stream_, "ic_build: factorize");
}

// =====================================================================================
// gradient / compute_step / solve_step mirrors (evaluated at the solver's p0)
// =====================================================================================
static void need_built(const SolverState& s) {
  if (!s.built) throw PbaError(PBA_E_STATE, "IC solver not built (call pba_gpu_ic_build first)");
}

void Engine::ic_gradient(double* g) {
  need_built(ic_);
  ic_eval(pose0_.p, d0_.p, mask_[ic_.mcur].p, scratch_bits_.p, 0, ic_.lambda, nullptr, nullptr);
  (void)ic_read_status();
  if (F_ > 0) ck(cudaMemcpy(g, gf_[0].p, 6 * F_ * sizeof(double), cudaMemcpyDeviceToHost), "g_f");
  download_depths_user(gn_[0], g + 6 * F_);
}

void Engine::ic_factorize(double lambda) {
  need_built(ic_);
  ic_factorize_loop(lambda);
}

}  // namespace pba_b200
