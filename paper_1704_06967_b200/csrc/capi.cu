// extern "C" boundary: include/pba_gpu.h.  Exceptions never cross it; every
// pba:: exception class of the reference maps to one status code.
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "engine.hpp"

using pba_b200::Engine;
using pba_b200::PbaError;

struct pba_handle {
  std::unique_ptr<Engine> e;
  std::string err;
};

namespace {

thread_local std::string g_create_error;

template <typename Fn>
int guarded(pba_handle* h, Fn&& fn) {
  if (!h || !h->e) return PBA_E_ARG;
  try {
    h->e->bind();
    fn(*h->e);
    return PBA_OK;
  } catch (const PbaError& ex) {
    h->err = ex.what();
    return ex.code;
  } catch (const std::exception& ex) {
    h->err = ex.what();
    return PBA_E_ARG;
  }
}

}  // namespace

extern "C" {

const char* pba_status_string(int s) {
  switch (s) {
    case PBA_OK: return "ok";
    case PBA_E_EMPTY_PROBLEM: return "EmptyProblem";
    case PBA_E_OUT_OF_BOUNDS: return "OutOfBounds";
    case PBA_E_INVALID_DEPTH: return "InvalidDepth";
    case PBA_E_DEGENERATE_DEPTH: return "DegenerateDepth";
    case PBA_E_SINGULAR_HESSIAN: return "SingularHessian";
    case PBA_E_CUDA: return "CudaError";
    case PBA_E_ARG: return "InvalidArgument";
    case PBA_E_STATE: return "InvalidState";
    case PBA_E_SPEC_INFEASIBLE: return "SpecInfeasible";
    default: return "unknown";
  }
}

// perturb_parameters (synth.cpp:308-320): one std::mt19937_64 stream, N(0, sigma) draws on the six
// tangent coordinates of every pose (pose_boxplus, geometry.cpp:93-98: R <- exp(w) R, t <- t + v),
// then one per inverse depth.  Host only (the CLI's `solve` input, pba.cpp:55-62).
int pba_perturb_parameters(int32_t F, double* R, double* t, int32_t N, double* d, double sigma, uint64_t seed) {
  if (F < 0 || N < 0 || (F > 0 && (!R || !t)) || (N > 0 && !d)) return PBA_E_ARG;
  if (!(sigma > 0.0)) return PBA_OK;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, sigma);
  for (int f = 0; f < F; ++f) {
    double delta[6];
    for (int i = 0; i < 6; ++i) delta[i] = gauss(rng);
    double E[9], Rn[9];
    pba_b200::so3_exp(delta, E);
    pba_b200::mat3_mul(E, R + 9 * f, Rn);
    for (int i = 0; i < 9; ++i) R[9 * f + i] = Rn[i];
    for (int i = 0; i < 3; ++i) t[3 * f + i] += delta[3 + i];
  }
  for (int n = 0; n < N; ++n) d[n] += gauss(rng);
  return PBA_OK;
}

void pba_config_default(pba_config* c) {  // SolverConfig{} (solver.hpp:45-54)
  c->gamma = 0.03;
  c->threshold_px = 5e-3;
  c->max_iters = 200;
  c->lambda0 = 1e-6;
  c->max_bad_steps = 8;
  c->normalize_depth_gauge = 1;
  c->refresh_ic_hessian = 0;
  c->record_snapshots = 0;
}

static int create_impl(const pba_problem* problem, pba_handle** out, bool deferred) {
  if (!out) return PBA_E_ARG;
  *out = nullptr;
  try {
    auto h = std::make_unique<pba_handle>();
    h->e = std::make_unique<Engine>(problem, deferred);
    *out = h.release();
    return PBA_OK;
  } catch (const PbaError& ex) {
    g_create_error = ex.what();
    return ex.code;
  } catch (const std::exception& ex) {
    g_create_error = ex.what();
    return PBA_E_ARG;
  }
}
int pba_gpu_create(const pba_problem* problem, pba_handle** out) { return create_impl(problem, out, false); }
int pba_gpu_create_deferred(const pba_problem* problem, pba_handle** out) { return create_impl(problem, out, true); }

void pba_gpu_destroy(pba_handle* h) { delete h; }

const char* pba_gpu_last_error(const pba_handle* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

int64_t pba_gpu_num_observations(const pba_handle* h) { return (h && h->e) ? h->e->num_obs() : -1; }

int pba_gpu_set_params(pba_handle* h, const double* R, const double* t, const double* d) {
  return guarded(h, [&](Engine& e) { e.set_params(R, t, d); });
}
int pba_gpu_get_params(pba_handle* h, double* R, double* t, double* d) {
  return guarded(h, [&](Engine& e) { e.get_params(R, t, d); });
}
int pba_gpu_energy(pba_handle* h, double gamma, const uint8_t* mask, pba_energy_result* out, double* residuals,
                   uint8_t* active) {
  return guarded(h, [&](Engine& e) { e.energy(gamma, mask, out, residuals, active); });
}
int pba_gpu_ic_build(pba_handle* h, const pba_config* cfg) {
  return guarded(h, [&](Engine& e) { e.ic_build(cfg); });
}
int pba_gpu_ic_gradient(pba_handle* h, double* g) {
  return guarded(h, [&](Engine& e) { e.ic_gradient(g); });
}
int pba_gpu_ic_compute_step(pba_handle* h, double* dx) {
  return guarded(h, [&](Engine& e) { e.ic_compute_step(dx); });
}
int pba_gpu_ic_solve_step(pba_handle* h, const double* g, double* dx) {
  return guarded(h, [&](Engine& e) { e.ic_solve_step(g, dx); });
}
int pba_gpu_ic_factorize(pba_handle* h, double lambda) {
  return guarded(h, [&](Engine& e) { e.ic_factorize(lambda); });
}
int pba_gpu_ic_hessian(pba_handle* h, double* pp, double* dd, double* pd, double* lambda) {
  return guarded(h, [&](Engine& e) { e.ic_hessian(pp, dd, pd, lambda); });
}
int pba_gpu_warning_count(const pba_handle* h) {
  return (h && h->e) ? static_cast<int>(h->e->warning_count()) : 0;
}
int64_t pba_gpu_warnings_text(const pba_handle* h, char* buf, int64_t len) {
  if (!h || !h->e) return 0;
  const std::string& all = h->e->warnings_text();
  if (buf && len > 0) {
    const size_t n = std::min<size_t>(all.size(), static_cast<size_t>(len - 1));
    std::memcpy(buf, all.data(), n);
    buf[n] = '\0';
  }
  return static_cast<int64_t>(all.size());
}
int64_t pba_gpu_warning_points(const pba_handle* h, int32_t* idx, int64_t cap) {
  if (!h || !h->e) return 0;
  try {
    return h->e->warning_points(idx, cap);
  } catch (...) {
    return 0;
  }
}
int pba_gpu_warning(const pba_handle* h, int i, char* buf, int len) {
  if (!h || !h->e || i < 0 || i >= h->e->warning_count() || !buf || len <= 0) return PBA_E_ARG;
  std::snprintf(buf, len, "%s", h->e->warning(i).c_str());
  return PBA_OK;
}
int pba_gpu_ic_begin(pba_handle* h, const pba_config* cfg) {
  return guarded(h, [&](Engine& e) { e.begin(true, cfg); });
}
int pba_gpu_fc_begin(pba_handle* h, const pba_config* cfg) {
  return guarded(h, [&](Engine& e) { e.begin(false, cfg); });
}
int pba_gpu_iterate(pba_handle* h, pba_iter_stats* stats, int* done) {
  return guarded(h, [&](Engine& e) {
    const bool d = e.iterate(stats);
    if (done) *done = d ? 1 : 0;
  });
}
int pba_gpu_end(pba_handle* h, pba_report* rep) {
  return guarded(h, [&](Engine& e) { e.end(rep); });
}
static int run_all(pba_handle* h, bool ic, const pba_config* cfg, pba_report* rep) {
  return guarded(h, [&](Engine& e) {
    e.begin(ic, cfg);
    try {
      while (!e.iterate(nullptr)) {
      }
    } catch (...) {
      e.end(nullptr);
      throw;
    }
    e.end(rep);
  });
}
int pba_gpu_ic_run(pba_handle* h, const pba_config* cfg, pba_report* rep) { return run_all(h, true, cfg, rep); }
int pba_gpu_fc_run(pba_handle* h, const pba_config* cfg, pba_report* rep) { return run_all(h, false, cfg, rep); }
int pba_gpu_fc_build(pba_handle* h, double gamma, double* pp, double* dd, double* pd, double* g) {
  return guarded(h, [&](Engine& e) { e.fc_build(gamma, pp, dd, pd, g); });
}
int pba_gpu_solve_normal_equations_schur(int32_t F, int32_t N, const int64_t* obs_ptr, const int32_t* obs_frame,
                                         const double* pp, const double* dd, const double* pd, const double* g,
                                         double lambda, double* dx) {
  try {
    Engine::solve_schur_free(F, N, obs_ptr, obs_frame, pp, dd, pd, g, lambda, dx);
    return PBA_OK;
  } catch (const PbaError& ex) {
    g_create_error = ex.what();
    return ex.code;
  } catch (const std::exception& ex) {
    g_create_error = ex.what();
    return PBA_E_ARG;
  }
}
int pba_gpu_apply_update(pba_handle* h, int mode, const double* dx, double* R, double* t, double* d, int* invalid) {
  return guarded(h, [&](Engine& e) { e.apply_update(mode, dx, R, t, d, invalid); });
}
int pba_gpu_max_reproj_update(pba_handle* h, const double* R, const double* t, const double* d, double* px) {
  return guarded(h, [&](Engine& e) { *px = e.max_reproj_update(R, t, d); });
}
int pba_gpu_normalize_gauge(pba_handle* h) {
  return guarded(h, [&](Engine& e) { e.normalize_gauge(); });
}
int pba_gpu_set_exchange(pba_handle* h, int32_t rank, int32_t world, int64_t num_points_total, pba_exchange_fn fn,
                         void* ctx) {
  return guarded(h, [&](Engine& e) { e.set_exchange(rank, world, num_points_total, fn, ctx); });
}
int pba_gpu_nccl_unique_id(void* id128) {
  if (!id128) return PBA_E_ARG;
  try {
    pba_b200::nccl_unique_id(id128);
    return PBA_OK;
  } catch (const pba_b200::PbaError& e) {
    return e.code;
  } catch (...) {
    return PBA_E_CUDA;
  }
}
int pba_gpu_set_exchange_nccl(pba_handle* h, const void* id128, int32_t rank, int32_t world,
                              int64_t num_points_total) {
  if (!id128) return PBA_E_ARG;
  return guarded(h, [&](Engine& e) { e.set_exchange_nccl(id128, rank, world, num_points_total); });
}
void* pba_gpu_stream(pba_handle* h) { return (h && h->e) ? static_cast<void*>(h->e->stream()) : nullptr; }
int pba_gpu_set_profiling(pba_handle* h, int on) {
  return guarded(h, [&](Engine& e) { e.set_profiling(on != 0); });
}
int pba_gpu_kernel_times(pba_handle* h, int64_t* counts, double* total_ms) {
  return guarded(h, [&](Engine& e) { e.kernel_times(counts, total_ms); });
}
int64_t pba_gpu_launch_count(void) { return pba_b200::launch_count(); }

int64_t pba_gpu_device_bytes(const pba_handle* h) { return (h && h->e) ? h->e->device_bytes() : 0; }

}  // extern "C"
