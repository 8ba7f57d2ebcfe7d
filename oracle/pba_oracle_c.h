/*
 * CPU ORACLE C API — TEST INFRASTRUCTURE ONLY.
 * Mirrors include/pba_gpu.h function-for-function (prefix pba_oracle_) so the
 * parity tests drive the GPU library and the oracle through the same calls.
 */
#ifndef PBA_ORACLE_C_H
#define PBA_ORACLE_C_H

#include "../include/pba_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pba_oracle_handle pba_oracle_handle;

int pba_oracle_create(const pba_problem* problem, pba_oracle_handle** out);
void pba_oracle_destroy(pba_oracle_handle* h);
const char* pba_oracle_last_error(const pba_oracle_handle* h);
int64_t pba_oracle_num_observations(const pba_oracle_handle* h);
int pba_oracle_set_params(pba_oracle_handle* h, const double* R, const double* t, const double* d);
int pba_oracle_get_params(pba_oracle_handle* h, double* R, double* t, double* d);
int pba_oracle_energy(pba_oracle_handle* h, double gamma, const uint8_t* mask,
                      pba_energy_result* out, double* residuals, uint8_t* active);
int pba_oracle_ic_build(pba_oracle_handle* h, const pba_config* cfg);
int pba_oracle_ic_gradient(pba_oracle_handle* h, double* g);
int pba_oracle_ic_compute_step(pba_oracle_handle* h, double* dx);
int pba_oracle_ic_solve_step(pba_oracle_handle* h, const double* g, double* dx);
int pba_oracle_ic_factorize(pba_oracle_handle* h, double lambda);
int pba_oracle_ic_hessian(pba_oracle_handle* h, double* pose_pose, double* depth_depth,
                          double* pose_depth, double* lambda);
int pba_oracle_warning_count(const pba_oracle_handle* h);
int pba_oracle_warning(const pba_oracle_handle* h, int i, char* buf, int len);
int64_t pba_oracle_warnings_text(const pba_oracle_handle* h, char* buf, int64_t len);
int64_t pba_oracle_warning_points(const pba_oracle_handle* h, int32_t* idx, int64_t cap);
int pba_oracle_ic_run(pba_oracle_handle* h, const pba_config* cfg, pba_report* rep);
int pba_oracle_fc_build(pba_oracle_handle* h, double gamma, double* pose_pose, double* depth_depth,
                        double* pose_depth, double* g);
int pba_oracle_fc_run(pba_oracle_handle* h, const pba_config* cfg, pba_report* rep);
int pba_oracle_solve_normal_equations_schur(int32_t F, int32_t N, const int64_t* obs_ptr,
                                            const int32_t* obs_frame, const double* pose_pose,
                                            const double* depth_depth, const double* pose_depth,
                                            const double* g, double lambda, double* dx);
int pba_oracle_solve_normal_equations_dense(int32_t F, int32_t N, const int64_t* obs_ptr,
                                            const int32_t* obs_frame, const double* pose_pose,
                                            const double* depth_depth, const double* pose_depth,
                                            const double* g, double lambda, double* dx);
int pba_oracle_apply_update(pba_oracle_handle* h, int mode, const double* dx, double* R_out,
                            double* t_out, double* d_out, int* invalid);
int pba_oracle_max_reproj_update(pba_oracle_handle* h, const double* R, const double* t,
                                 const double* d, double* px);
int pba_oracle_normalize_gauge(pba_oracle_handle* h);

/* Reference test-scene generator (synth.hpp:14-80). */
/* joint multi-host window (oracle/multihost.cpp); mirrors pba_gpu_mh_* */
typedef struct pba_oracle_mh_handle pba_oracle_mh_handle;
int pba_oracle_mh_create(const pba_mh_problem* problem, pba_oracle_mh_handle** out);
void pba_oracle_mh_destroy(pba_oracle_mh_handle* h);
const char* pba_oracle_mh_last_error(const pba_oracle_mh_handle* h);
int pba_oracle_mh_energy(pba_oracle_mh_handle* h, double gamma, pba_energy_result* out);
int pba_oracle_mh_fc_run(pba_oracle_mh_handle* h, const pba_config* cfg, pba_report* rep, double* a_out,
                         double* b_out);

typedef struct pba_oracle_scene_spec {
  int32_t width, height;
  double fx, fy, cx, cy;
  int32_t octaves;
  double base_wavelength_px, lo, hi;
  int32_t geometry_kind;  /* 0 = Plane, 1 = Heightfield */
  double base_depth, amplitude, wavelength_px;
  int32_t trajectory_kind; /* 0 = Orbit, 1 = Dolly */
  int32_t frames;
  double span_deg;
  double extent[3];
  int32_t num_points;
  int32_t patch_radius;
  uint64_t seed;
  int32_t supersample;
} pba_oracle_scene_spec;

void pba_oracle_scene_spec_default(pba_oracle_scene_spec* spec);
/* Outputs: ref W*H, targets F*W*H (fp64 [0,1]), R F*9, t F*3, anchors N*2, inv_depths N. */
int pba_oracle_render_sequence(const pba_oracle_scene_spec* spec, double* ref, double* targets,
                               double* R, double* t, double* anchors, double* inv_depths,
                               char* err, int errlen);
int pba_oracle_perturb_parameters(int32_t F, double* R, double* t, int32_t N, double* d,
                                  double sigma, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
