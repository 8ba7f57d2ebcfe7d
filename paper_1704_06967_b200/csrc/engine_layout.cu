// Device-side construction of the observation layout for one handle:
// Morton order of the points, point-major and frame-major observation lists, the
// maps between them and the caller's order, frame-major tiles and the Schur chunk
// plan.  Sorting uses CUB radix sorts (stable), everything else is gather/scatter
// kernels, so handle creation costs milliseconds even at 4*10^7 observations.
#include <algorithm>
#include <cstdlib>
#include <cub/cub.cuh>
#include <cstring>
#include <numeric>

#include "engine.hpp"

namespace pba_b200 {

namespace {

__global__ void k_dense_obs(int N, int F, int64_t* __restrict__ uptr, int32_t* __restrict__ uframe) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i <= N) uptr[i] = i * F;
  const int64_t NO = static_cast<int64_t>(N) * F;
  for (int64_t o = i; o < NO; o += static_cast<int64_t>(gridDim.x) * blockDim.x) uframe[o] = static_cast<int32_t>(o % F);
}

__global__ void k_validate_obs(int N, int F, const int64_t* __restrict__ uptr, const int32_t* __restrict__ uframe,
                               int* __restrict__ err) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int64_t a = uptr[n], b = uptr[n + 1];
  if (b < a) {
    atomicOr(err, 1);
    return;
  }
  for (int64_t o = a; o < b; ++o) {
    const int f = uframe[o];
    if (f < 0 || f >= F) atomicOr(err, 2);
    if (o > a && f <= uframe[o - 1]) atomicOr(err, 4);
  }
}

__device__ __forceinline__ uint32_t part1by1(uint32_t x) {
  x &= 0xffff;
  x = (x | (x << 8)) & 0x00FF00FF;
  x = (x | (x << 4)) & 0x0F0F0F0F;
  x = (x | (x << 2)) & 0x33333333;
  x = (x | (x << 1)) & 0x55555555;
  return x;
}

__global__ void k_morton(int N, const double2* __restrict__ anc, uint32_t* __restrict__ key, int32_t* __restrict__ idx) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const double cu = fmin(fmax(floor(anc[n].x), 0.0), 65535.0);
  const double cv = fmin(fmax(floor(anc[n].y), 0.0), 65535.0);
  key[n] = part1by1(static_cast<uint32_t>(cu)) | (part1by1(static_cast<uint32_t>(cv)) << 1);
  idx[n] = n;
}

__global__ void k_iota(int64_t n, int32_t* __restrict__ v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[i] = static_cast<int32_t>(i);
}

__global__ void k_counts(int N, const int32_t* __restrict__ perm, const int64_t* __restrict__ uptr,
                         int64_t* __restrict__ cnt, int32_t* __restrict__ iperm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) {
    const int u = perm[i];
    cnt[i] = uptr[u + 1] - uptr[u];
    iperm[u] = i;
  }
  if (i == N) cnt[N] = 0;
}

// warp per internal point: copy its frames from the caller's CSR
__global__ void k_fill_pm(int N, const int32_t* __restrict__ perm, const int64_t* __restrict__ uptr,
                          const int32_t* __restrict__ uframe, const int64_t* __restrict__ pm_ptr,
                          int32_t* __restrict__ pm_frame, int32_t* __restrict__ pm_point, int32_t* __restrict__ pm2uo) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= N) return;
  const int u = perm[i];
  const int64_t a = uptr[u], o0 = pm_ptr[i];
  const int k = static_cast<int>(uptr[u + 1] - a);
  for (int j = lane; j < k; j += 32) {
    pm_frame[o0 + j] = uframe[a + j];
    pm_point[o0 + j] = i;
    pm2uo[o0 + j] = static_cast<int32_t>(a + j);
  }
}

// four independent observations per thread and step: their dependent gathers (o -> n -> anchor)
// are issued together instead of one chain at a time
__global__ void k_fm_scatter(int64_t NO, const int32_t* __restrict__ fm2pm, const int32_t* __restrict__ pm_point,
                             const int32_t* __restrict__ pm2uo, const double2* __restrict__ anc,
                             int32_t* __restrict__ pm2fm, int32_t* __restrict__ fm_point, int32_t* __restrict__ uo2q,
                             double2* __restrict__ anchor_fm) {
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q0 < NO; q0 += U * stride) {
    int o[U], n[U], uo[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * stride;
      o[u] = q < NO ? __ldg(fm2pm + q) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      n[u] = __ldg(pm_point + o[u]);
      uo[u] = __ldg(pm2uo + o[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * stride;
      if (q >= NO) break;
      pm2fm[o[u]] = static_cast<int32_t>(q);
      fm_point[q] = n[u];
      uo2q[uo[u]] = static_cast<int32_t>(q);
      anchor_fm[q] = __ldg(anc + n[u]);
    }
  }
}

// fm_ptr[f] = first q whose frame is >= f (sorted frame keys)
__global__ void k_fm_ptr(int F, int64_t NO, const int32_t* __restrict__ sorted, int64_t* __restrict__ fm_ptr) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f > F) return;
  int64_t lo = 0, hi = NO;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < f) lo = mid + 1; else hi = mid;
  }
  fm_ptr[f] = lo;
}

__global__ void k_anchor_internal(int N, const int32_t* __restrict__ perm, const double2* __restrict__ anc_user,
                                  double2* __restrict__ anc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) anc[i] = anc_user[perm[i]];
}

// template feasibility (solver.cpp:40-45): every template pixel inside [1, W-3] x [1, H-3]
__global__ void k_template_check(int N, const double2* __restrict__ anc, PatternD pat, int W, int H,
                                 int* __restrict__ bad) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  for (int k = 0; k < pat.P; ++k) {
    const double u = anc[n].x + static_cast<double>(pat.dx[k]);
    const double v = anc[n].y + static_cast<double>(pat.dy[k]);
    if (!(u >= 1.0 && u <= W - 3 && v >= 1.0 && v <= H - 3)) {
      atomicOr(bad, 1);
      return;
    }
  }
}

// visibility-window key of each point for the Schur chunk plan; empty points sort last
__global__ void k_window_keys(int N, const int64_t* __restrict__ pm_ptr, const int32_t* __restrict__ pm_frame,
                              uint32_t* __restrict__ key, int32_t* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int64_t a = pm_ptr[i], b = pm_ptr[i + 1];
  key[i] = (b > a) ? (static_cast<uint32_t>(pm_frame[a]) << 16) | static_cast<uint32_t>(pm_frame[b - 1]) : 0xffffffffu;
  idx[i] = i;
}

// ---- caller-order <-> frame-major conversions of per-observation arrays ----
__global__ void k_mask_bytes_to_bits(int64_t NO, int P, const int32_t* __restrict__ uo2q, const uint8_t* __restrict__ m,
                                     uint32_t* __restrict__ bits) {
  for (int64_t ou = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; ou < NO;
       ou += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t b = 0;
    for (int k = 0; k < P; ++k)
      if (m[ou * P + k]) b |= 1u << k;
    bits[uo2q[ou]] = b;
  }
}
__global__ void k_bits_to_bytes(int64_t NO, int P, const int32_t* __restrict__ uo2q, const uint32_t* __restrict__ bits,
                                uint8_t* __restrict__ m) {
  for (int64_t ou = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; ou < NO;
       ou += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t b = bits[uo2q[ou]];
    for (int k = 0; k < P; ++k) m[ou * P + k] = (b >> k) & 1u;
  }
}
// dst[ou*w + c] = src[uo2q[ou]*w + c] (to_user) or the inverse scatter
__global__ void k_perm_rows(int64_t NO, int w, const int32_t* __restrict__ uo2q, const double* __restrict__ src,
                            double* __restrict__ dst, int to_user) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < NO * w;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ou = e / w, c = e % w;
    const int64_t q = uo2q[ou];
    if (to_user) dst[e] = src[q * w + c]; else dst[q * w + c] = src[e];
  }
}

int grid_for(int64_t n, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 32)));
}

template <typename K, typename V>
void radix_sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int end_bit, cudaStream_t s) {
  size_t tmp = 0;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, end_bit, s), "cub sort size");
  DBuf<unsigned char> t;
  t.alloc(std::max<size_t>(tmp, 1));
  ck(cub::DeviceRadixSort::SortPairs(t.p, tmp, kin, kout, vin, vout, n, 0, end_bit, s), "cub sort");
  ck(cudaStreamSynchronize(s), "sort sync");
}

int bits_for(int64_t v) {
  int b = 1;
  while ((int64_t(1) << b) <= v) ++b;
  return b;
}

}  // namespace

template struct DBuf<unsigned char>;

// ascending in-place sort of n int32 keys on the device (the zero-depth warning list)
void sort_i32(int32_t* keys, int n, cudaStream_t s) {
  if (n <= 1) return;
  DBuf<int32_t> tmp_keys;
  tmp_keys.alloc(n);
  size_t tmp = 0;
  ck(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, tmp_keys.p, n, 0, 32, s), "cub sort size");
  DBuf<unsigned char> t;
  t.alloc(std::max<size_t>(tmp, 1));
  ck(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys, tmp_keys.p, n, 0, 32, s), "cub sort keys");
  ck(cudaMemcpyAsync(keys, tmp_keys.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s), "sorted keys");
  ck(cudaStreamSynchronize(s), "sort sync");
}

void Engine::build_layout(const pba_problem* p, const std::function<void()>& after_obs_upload) {
  cudaStream_t s = stream_;
  // ---- caller CSR on the device (dense problems are generated in place) ----
  DBuf<int64_t> uptr;
  DBuf<int32_t> uframe;
  uptr.alloc(static_cast<size_t>(N_) + 1);
  if (p->obs_ptr) {
    if (p->obs_ptr[0] != 0) throw PbaError(PBA_E_ARG, "obs_ptr[0] must be 0");
    NO_ = p->obs_ptr[N_];
    if (NO_ < 0) throw PbaError(PBA_E_ARG, "obs_ptr must be non-decreasing");
  } else {
    NO_ = static_cast<int64_t>(N_) * F_;
  }
  if (NO_ >= (int64_t(1) << 31) - 16) throw PbaError(PBA_E_ARG, "more than 2^31 observations");
  uframe.alloc(static_cast<size_t>(std::max<int64_t>(NO_, 1)));
  DBuf<int> flags;
  flags.alloc(4);
  ck(cudaMemsetAsync(flags.p, 0, 4 * sizeof(int), s), "memset");
  if (p->obs_ptr) {
    ck(cudaMemcpyAsync(uptr.p, p->obs_ptr, (N_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s), "obs_ptr");
    if (NO_ > 0)
      ck(cudaMemcpyAsync(uframe.p, p->obs_frame, NO_ * sizeof(int32_t), cudaMemcpyHostToDevice, s), "obs_frame");
    if (N_ > 0) k_validate_obs<<<(N_ + 255) / 256, 256, 0, s>>>(N_, F_, uptr.p, uframe.p, flags.p);
  } else {
    k_dense_obs<<<grid_for(std::max<int64_t>(NO_, N_ + 1)), 256, 0, s>>>(N_, F_, uptr.p, uframe.p);
  }
  count_launches(1);

  trace_mark(s, "layout: obs upload+validate");
  // ---- internal point order: Morton order of the anchor pixel (texture locality) ----
  DBuf<double2> anc_user;
  anc_user.alloc(std::max(N_, 1));
  if (N_ > 0)
    ck(cudaMemcpyAsync(anc_user.p, p->anchors_px, N_ * sizeof(double2), cudaMemcpyHostToDevice, s), "anchors");
  after_obs_upload();  // the caller starts the image upload behind the layout inputs
  DBuf<uint32_t> key, key_sorted;
  DBuf<int32_t> idx, perm_d, iperm_d;
  key.alloc(std::max(N_, 1));
  key_sorted.alloc(std::max(N_, 1));
  idx.alloc(std::max(N_, 1));
  perm_d.alloc(std::max(N_, 1));
  iperm_d.alloc(std::max(N_, 1));
  if (N_ > 0) {
    k_morton<<<(N_ + 255) / 256, 256, 0, s>>>(N_, anc_user.p, key.p, idx.p);
    k_template_check<<<(N_ + 255) / 256, 256, 0, s>>>(N_, anc_user.p, pat_, ref_.W, ref_.H, flags.p + 1);
    count_launches(2);
    radix_sort_pairs(key.p, key_sorted.p, idx.p, perm_d.p, N_, 32, s);
  }

  trace_mark(s, "layout: morton sort");
  // ---- point-major list ----
  DBuf<int64_t> cnt;
  cnt.alloc(static_cast<size_t>(N_) + 1);
  pm_ptr_.alloc(static_cast<size_t>(N_) + 1);
  k_counts<<<(N_ + 1 + 255) / 256, 256, 0, s>>>(N_, perm_d.p, uptr.p, cnt.p, iperm_d.p);
  count_launches(1);
  {
    size_t tmp = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, pm_ptr_.p, N_ + 1, s), "scan size");
    DBuf<unsigned char> t;
    t.alloc(std::max<size_t>(tmp, 1));
    ck(cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt.p, pm_ptr_.p, N_ + 1, s), "scan");
    ck(cudaStreamSynchronize(s), "scan sync");
  }
  const size_t nO = static_cast<size_t>(std::max<int64_t>(NO_, 1));
  pm_frame_.alloc(nO);
  DBuf<int32_t> pm_point, pm2uo;
  pm_point.alloc(nO);
  pm2uo.alloc(nO);
  if (N_ > 0) {
    k_fill_pm<<<(N_ * 32 + 255) / 256, 256, 0, s>>>(N_, perm_d.p, uptr.p, uframe.p, pm_ptr_.p, pm_frame_.p, pm_point.p,
                                                    pm2uo.p);
    count_launches(1);
  }

  trace_mark(s, "layout: point-major list");
  // ---- frame-major list (stable radix sort of observations by frame) ----
  DBuf<int32_t> frames_sorted, iota_o;
  DBuf<int32_t>& fm2pm = fm2pm_;  // kept: the IC build writes the point-major B blocks through it
  frames_sorted.alloc(nO);
  iota_o.alloc(nO);
  fm2pm.alloc(nO);
  pm2fm_.alloc(nO);
  fm_point_.alloc(nO + 8);  // padding: 16-byte aligned TMA windows may read 3 past the end
  uo2q_d_.alloc(nO);
  anchor_.alloc(std::max(N_, 1));
  anchor_fm_.alloc(nO);
  ck(cudaMemsetAsync(fm_point_.p, 0, (nO + 8) * sizeof(int32_t), s), "memset");
  trace_mark(s, "layout:   fm allocs");
  if (N_ > 0) {
    k_anchor_internal<<<(N_ + 255) / 256, 256, 0, s>>>(N_, perm_d.p, anc_user.p, anchor_.p);
    count_launches(1);
  }
  if (NO_ > 0) {
    k_iota<<<grid_for(NO_), 256, 0, s>>>(NO_, iota_o.p);
    count_launches(1);
    trace_mark(s, "layout:   iota");
    radix_sort_pairs(pm_frame_.p, frames_sorted.p, iota_o.p, fm2pm.p, NO_, bits_for(F_), s);
    trace_mark(s, "layout:   frame sort");
    k_fm_scatter<<<grid_for((NO_ + 3) / 4), 256, 0, s>>>(NO_, fm2pm.p, pm_point.p, pm2uo.p, anchor_.p, pm2fm_.p,
                                                         fm_point_.p, uo2q_d_.p, anchor_fm_.p);
    count_launches(1);
  }
  trace_mark(s, "layout: frame-major sort+scatter");
  fm_ptr_.alloc(static_cast<size_t>(F_) + 1);
  k_fm_ptr<<<(F_ + 1 + 255) / 256, 256, 0, s>>>(F_, NO_, frames_sorted.p, fm_ptr_.p);
  count_launches(1);

  // ---- small host-side results ----
  int fl[4];
  ck(cudaMemcpyAsync(fl, flags.p, sizeof(fl), cudaMemcpyDeviceToHost, s), "flags");
  std::vector<int64_t> fm_ptr(F_ + 1);
  ck(cudaMemcpyAsync(fm_ptr.data(), fm_ptr_.p, (F_ + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "fm_ptr");
  perm_.resize(N_);
  iperm_.resize(N_);
  if (N_ > 0) {
    ck(cudaMemcpyAsync(perm_.data(), perm_d.p, N_ * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "perm");
    ck(cudaMemcpyAsync(iperm_.data(), iperm_d.p, N_ * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "iperm");
  }
  perm_d_.alloc(std::max(N_, 1));
  zero_idx_.alloc(static_cast<size_t>(N_) + 1);
  if (N_ > 0) ck(cudaMemcpyAsync(perm_d_.p, perm_d.p, N_ * sizeof(int32_t), cudaMemcpyDeviceToDevice, s), "perm copy");
  ck(cudaStreamSynchronize(s), "layout sync");
  if (fl[0] & 1) throw PbaError(PBA_E_ARG, "obs_ptr must be non-decreasing");
  if (fl[0] & 2) throw PbaError(PBA_E_ARG, "obs_frame out of range");
  if (fl[0] & 4) throw PbaError(PBA_E_ARG, "obs_frame must be strictly increasing per point");
  template_ok_ = fl[1] == 0;

  trace_mark(s, "layout: host results");
  // The Schur chunk plan goes first: its device sort, key download and host chunking overlap the
  // target-image upload; the small host->device copies of both plans queue behind that upload.
  // ---- Schur chunk plan: points sorted by visibility window (first frame, last frame) and cut
  //      greedily into chunks whose union window keeps the padded width LD = roundup(6 W, kSchurTB)
  //      of the chunk's first window (so merging windows costs no extra DMMA columns), up to
  //      kMaxChunk points; one work item per kSchurTB^2 upper tile-block of each chunk's window.
  //      Long chunks mean long K loops and few fixed-point folds of each tile into S. ----
  {
    const int kMaxChunk = [] {
      const char* e = std::getenv("PBA_SCHUR_CHUNK");
      return e ? std::max(32, std::atoi(e)) : 4096;
    }();
    DBuf<uint32_t> wkey, wkey_sorted;
    DBuf<int32_t> widx;
    wkey.alloc(std::max(N_, 1));
    wkey_sorted.alloc(std::max(N_, 1));
    widx.alloc(std::max(N_, 1));
    chunk_pts_.alloc(std::max(N_, 1));
    int npts = 0;
    std::vector<int4> sblocks;
    if (N_ > 0) {
      k_window_keys<<<(N_ + 255) / 256, 256, 0, s>>>(N_, pm_ptr_.p, pm_frame_.p, wkey.p, widx.p);
      count_launches(1);
      radix_sort_pairs(wkey.p, wkey_sorted.p, widx.p, chunk_pts_.p, N_, 32, s);
      std::vector<uint32_t> keys(N_);
      ck(cudaMemcpy(keys.data(), wkey_sorted.p, N_ * sizeof(uint32_t), cudaMemcpyDeviceToHost), "window keys");
      // points without observations carry key 0xffffffff and sort last
      while (npts < N_ && keys[npts] != 0xffffffffu) ++npts;
      std::vector<int4> chunks;
      std::vector<int64_t> off;
      std::vector<int32_t> chunk_of(std::max(npts, 1));
      int64_t total = 0;
      for (int p = 0; p < npts;) {
        int fmin = static_cast<int>(keys[p] >> 16), fmax = static_cast<int>(keys[p] & 0xffffu);
        const int LD = ((6 * (fmax - fmin + 1) + kSchurTB - 1) / kSchurTB) * kSchurTB;
        int q = p + 1;
        while (q < npts && q - p < kMaxChunk) {
          const int a0 = std::min(fmin, static_cast<int>(keys[q] >> 16));
          const int a1 = std::max(fmax, static_cast<int>(keys[q] & 0xffffu));
          if (6 * (a1 - a0 + 1) > LD) break;
          fmin = a0;
          fmax = a1;
          ++q;
        }
        const int nb = LD / kSchurTB;
        if (nb > 0xffff) throw PbaError(PBA_E_ARG, "Schur chunk window too large");
        const int c = static_cast<int>(chunks.size());
        chunks.push_back(make_int4(p, q, fmin, LD));
        off.push_back(total);
        total += static_cast<int64_t>(q - p) * LD;
        for (int i = p; i < q; ++i) chunk_of[i] = c;
        for (int rb = 0; rb < nb; ++rb)
          for (int cb = rb; cb < nb; ++cb) sblocks.push_back(make_int4(c, 0, 0, rb | (cb << 16)));
        p = q;
      }
      const int nchunks = static_cast<int>(chunks.size());
      schur_chunks_.alloc(std::max(nchunks, 1));
      schur_chunk_off_.alloc(std::max(nchunks, 1));
      schur_chunk_of_.alloc(std::max(npts, 1));
      if (nchunks > 0) {
        ck(cudaMemcpyAsync(schur_chunks_.p, chunks.data(), nchunks * sizeof(int4), cudaMemcpyHostToDevice, s), "chunks");
        ck(cudaMemcpyAsync(schur_chunk_off_.p, off.data(), nchunks * sizeof(int64_t), cudaMemcpyHostToDevice, s),
           "chunk off");
        ck(cudaMemcpyAsync(schur_chunk_of_.p, chunk_of.data(), npts * sizeof(int32_t), cudaMemcpyHostToDevice, s),
           "chunk of");
      }
      schur_dense_elems_ = total;
      ck(cudaStreamSynchronize(s), "chunks sync");
    }
    schur_blocks_.alloc(std::max<size_t>(sblocks.size(), 1));
    if (!sblocks.empty())
      ck(cudaMemcpyAsync(schur_blocks_.p, sblocks.data(), sblocks.size() * sizeof(int4), cudaMemcpyHostToDevice, s),
         "blocks");
    ck(cudaStreamSynchronize(s), "plan sync");
    schur_plan_ = SchurPlan{chunk_pts_.p, npts, schur_chunk_of_.p, schur_chunks_.p, schur_chunk_off_.p, nullptr,
                            nullptr, schur_blocks_.p, static_cast<int>(sblocks.size())};
  }

  trace_mark(s, "layout: schur plan");
  // ---- frame-major tiles (a tile never crosses a frame) ----
  {
    const int G = [this] {
      int g = 1;
      while (g < P_) g <<= 1;
      return g;
    }();
    const int ops = 256 / G;
    const int64_t steps = std::min<int64_t>(64, std::max<int64_t>(1, (NO_ + 148 * 8 * ops - 1) / (148 * 8 * ops)));
    const int64_t T = ops * steps;
    std::vector<int32_t> tile_frame, ftile_ptr(F_ + 1, 0);
    std::vector<int64_t> tq0, tq1;
    for (int f = 0; f < F_; ++f) {
      for (int64_t q = fm_ptr[f]; q < fm_ptr[f + 1]; q += T) {
        tile_frame.push_back(f);
        tq0.push_back(q);
        tq1.push_back(std::min(q + T, fm_ptr[f + 1]));
      }
      ftile_ptr[f + 1] = static_cast<int32_t>(tile_frame.size());
    }
    auto up = [&](auto& buf, const auto& vec) {
      using T2 = std::remove_reference_t<decltype(*buf.p)>;
      buf.alloc(std::max<size_t>(vec.size(), 1));
      if (!vec.empty())
        ck(cudaMemcpyAsync(buf.p, vec.data(), vec.size() * sizeof(T2), cudaMemcpyHostToDevice, s), "upload");
    };
    up(tile_frame_, tile_frame);
    up(tile_q0_, tq0);
    up(tile_q1_, tq1);
    up(ftile_ptr_, ftile_ptr);
    ftile_ptr_h_ = ftile_ptr;
    ov_.ntiles = static_cast<int>(tile_frame.size());
    // Launch order of the lane passes: within each group of kTabFrames frames (one IC-pass launch),
    // tiles sorted by their first point, then frame, so that the CTAs resident together work on
    // the same points in neighbouring frames and share the points' template records in L2.
    // Env PBA_TILE_ORDER=0 keeps the frame-major order.
    tile_order_.release();
    const char* env = std::getenv("PBA_TILE_ORDER");
    if (!(env && env[0] == '0') && ov_.ntiles > 0) {
      DBuf<int32_t> key;
      key.alloc(ov_.ntiles);
      launch_tile_first_point(ov_.ntiles, tile_q0_.p, fm_point_.p, key.p, s);
      std::vector<int32_t> kh(ov_.ntiles);
      ck(cudaMemcpyAsync(kh.data(), key.p, ov_.ntiles * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "tile keys");
      ck(cudaStreamSynchronize(s), "tile keys sync");
      std::vector<int32_t> order(ov_.ntiles);
      for (int g0 = 0; g0 < F_; g0 += kTabFrames) {
        const int t0 = ftile_ptr[g0], t1 = ftile_ptr[std::min(F_, g0 + kTabFrames)];
        for (int t = t0; t < t1; ++t) order[t] = t;
        std::stable_sort(order.begin() + t0, order.begin() + t1,
                         [&](int32_t x, int32_t y) { return kh[x] < kh[y]; });  // ties: frame order
      }
      up(tile_order_, order);
      ck(cudaStreamSynchronize(s), "tile order sync");
    }
  }

  trace_mark(s, "layout: tiles");
  ov_.N = N_;
  ov_.F = F_;
  ov_.P = P_;
  ov_.NO = NO_;
  ov_.pm_ptr = pm_ptr_.p;
  ov_.pm_frame = pm_frame_.p;
  ov_.pm2fm = pm2fm_.p;
  ov_.fm_ptr = fm_ptr_.p;
  ov_.fm_point = fm_point_.p;
  ov_.tile_frame = tile_frame_.p;
  ov_.tile_q0 = tile_q0_.p;
  ov_.tile_q1 = tile_q1_.p;
  ov_.ftile_ptr = ftile_ptr_.p;
  ov_.tile_order = tile_order_.p;
}

// ---- per-observation conversions between the caller's order and the frame-major layout ----
void Engine::mask_to_bits(const uint8_t* mask_user, uint32_t* bits_d) {
  DBuf<uint8_t> m;
  m.alloc(std::max<size_t>(static_cast<size_t>(NO_) * P_, 1));
  if (NO_ > 0) {
    ck(cudaMemcpyAsync(m.p, mask_user, static_cast<size_t>(NO_) * P_, cudaMemcpyHostToDevice, stream_), "mask");
    k_mask_bytes_to_bits<<<grid_for(NO_), 256, 0, stream_>>>(NO_, P_, uo2q_d_.p, m.p, bits_d);
    count_launches(1);
  }
  ck(cudaStreamSynchronize(stream_), "mask sync");
}

void Engine::bits_to_user(const uint32_t* bits_d, uint8_t* active_user) {
  DBuf<uint8_t> m;
  m.alloc(std::max<size_t>(static_cast<size_t>(NO_) * P_, 1));
  if (NO_ > 0) {
    k_bits_to_bytes<<<grid_for(NO_), 256, 0, stream_>>>(NO_, P_, uo2q_d_.p, bits_d, m.p);
    count_launches(1);
    ck(cudaMemcpyAsync(active_user, m.p, static_cast<size_t>(NO_) * P_, cudaMemcpyDeviceToHost, stream_), "active");
  }
  ck(cudaStreamSynchronize(stream_), "bits sync");
}

void Engine::rows_to_user(const double* src_fm, int w, double* dst_user) {
  DBuf<double> t;
  t.alloc(std::max<size_t>(static_cast<size_t>(NO_) * w, 1));
  if (NO_ > 0) {
    k_perm_rows<<<grid_for(NO_ * w), 256, 0, stream_>>>(NO_, w, uo2q_d_.p, src_fm, t.p, 1);
    count_launches(1);
    ck(cudaMemcpyAsync(dst_user, t.p, static_cast<size_t>(NO_) * w * sizeof(double), cudaMemcpyDeviceToHost, stream_),
       "rows");
  }
  ck(cudaStreamSynchronize(stream_), "rows sync");
}

void Engine::rows_from_user(const double* src_user, int w, double* dst_fm) {
  DBuf<double> t;
  t.alloc(std::max<size_t>(static_cast<size_t>(NO_) * w, 1));
  if (NO_ > 0) {
    ck(cudaMemcpyAsync(t.p, src_user, static_cast<size_t>(NO_) * w * sizeof(double), cudaMemcpyHostToDevice, stream_),
       "rows");
    k_perm_rows<<<grid_for(NO_ * w), 256, 0, stream_>>>(NO_, w, uo2q_d_.p, t.p, dst_fm, 0);
    count_launches(1);
  }
  ck(cudaStreamSynchronize(stream_), "rows sync");
}

}  // namespace pba_b200
