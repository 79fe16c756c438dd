/*
 * potflow_b200.h -- C ABI of the B200 (sm_100a) partial-optimal-transport hot
 * path.  Plain pointers and sizes only; every array argument is a DEVICE
 * pointer unless its name ends in _host.  `stream` is a cudaStream_t passed as
 * void* (0 = legacy default stream).  Functions return 0 on success and a
 * negative code on error (message via pf_last_error()); functions that mirror
 * a reference kernel returning a flag word return that word (>= 0).
 *
 * Reference interfaces replaced (all under /root/reference/pkg/src/potflow):
 *   pf_set_domain       laguerre._DomainPack / domain_pack     laguerre.py:113-139
 *   pf_grid_build       laguerre.SpatialGrid.__init__          laguerre.py:52-80
 *   pf_grid_export      SpatialGrid.bucket_start/bucket_sites  laguerre.py:78-79
 *   pf_dpsi_max         laguerre._dpsi_max                     laguerre.py:142-145
 *   pf_batch_evaluate   _kernels._batch_evaluate               _kernels.py:1362-1478
 *   pf_batch_evaluate_host  (same, host arrays in and out)     _kernels.py:1362-1478
 *   pf_knn              _kernels._knn / laguerre.knn            _kernels.py:1562-1620, laguerre.py:90-96
 *   pf_newton_*         ot_solver.newton_solve (spec only)
 *   pf_fluid_*          fluid_sim.step (spec only)
 */
#ifndef POTFLOW_B200_H
#define POTFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pf_ctx pf_ctx; /* opaque: device domain, grid, scratch */

/* cell status (_kernels.py:43-45) and flag bits (_kernels.py:48-50) */
#define PF_CELL_EMPTY 0
#define PF_CELL_FULLBALL 1
#define PF_CELL_CLIPPED 2
#define PF_FLAG_OVERFLOW 1
#define PF_FLAG_DEGENERATE_INTERIOR 2
#define PF_FLAG_UNSTABLE_PROJECTION 4

const char *pf_version(void);
const char *pf_last_error(void);
/* number of kernels this library has launched so far (benchmark evidence) */
unsigned long long pf_launch_count(void);
/* measured FP64 FMA throughput of the current device, TFLOP/s (FMA = 2 flops) */
int pf_fp64_peak(double *tflops_host, double *ms_host);

/* context lifetime; device = CUDA ordinal the context's buffers live on */
int pf_ctx_create(pf_ctx **out, int device);
int pf_ctx_destroy(pf_ctx *ctx);

/* Domain polytope in the reference packed layout (geom.pack_cell,
 * geom.py:353-375): dv[512*3], dc[3], dp[160*4], dt[160], dlp[161],
 * dlv[2048] (host arrays), tol = DEFAULT_REL_TOL * diagonal
 * (laguerre.py:120). */
int pf_set_domain(pf_ctx *ctx, const double *dv_host, const int64_t *dc_host,
                  const double *dp_host, const int64_t *dt_host, const int64_t *dlp_host,
                  const int64_t *dlv_host, double tol);

/* Parity mode (default off, or PF_PARITY_MODE=1 at context creation): every
 * evaluation restricts the facets exactly as the reference does
 * (_kernels.py:411-675, 678-716, 838-1001), including its spurious-entry and
 * wrapped-arc outcomes on cells whose loop vertex lies within tol outside the
 * sphere.  Off, those outcomes are corrected. */
int pf_set_parity_mode(pf_ctx *ctx, int on);
int pf_get_parity_mode(pf_ctx *ctx);

/* Uniform bucket grid over the domain bounding box by counting sort.
 * cell_size <= 0 picks the bucket edge from the weights (half the mean
 * ball-aware search radius, psi may be NULL -> (|domain|/n)^(1/3)/2).
 * Sites are stored bucket-sorted (SoA) for coalesced candidate gathers. */
int pf_grid_build(pf_ctx *ctx, int64_t n, const double *pts, const double *psi,
                  double cell_size, void *stream);
/* same with explicit bucket counts per axis (dims_host int[3]), as the
 * reference's SpatialGrid chooses them (laguerre.py:63-64) */
int pf_grid_build_dims(pf_ctx *ctx, int64_t n, const double *pts, const int *dims_host, void *stream);
/* grid dims (int[3]), origin (double[3]) and edge (double[3]) of the last build */
int pf_grid_info(pf_ctx *ctx, int *dims_host, double *lo_host, double *h_host);
/* reference-layout CSR of the last grid (int64 bucket_start[ncell+1],
 * bucket_sites[n]; within a bucket sites are in increasing index order) */
int pf_grid_export(pf_ctx *ctx, int64_t *bucket_start, int64_t *bucket_sites, void *stream);

/* dpsi = max(psi) - min(psi) (>= 0) into the context's device scalar;
 * dpsi_host (optional) receives it synchronously. */
int pf_dpsi_max(pf_ctx *ctx, int64_t n, const double *psi, double *dpsi_host, void *stream);

/* _kernels._batch_evaluate.  Outputs are caller-allocated device arrays with
 * the reference shapes: status i64[n], vol f64[n], ksur f64[n], cent f64[n,3],
 * ipt f64[n,3], m2 f64[n], fcount i64[n], ftag i64[n,smf], farea f64[n,smf],
 * fh f64[n,smf], fnrm f64[n,smf,3], fcent f64[n,smf,3].  Any output may be
 * NULL (skipped).  dpsi_max < 0 uses the device value of pf_dpsi_max.
 * rebuild_grid != 0 rebuilds the bucket grid from pts first.
 * Returns the OR of the per-cell flag words (synchronises the stream). */
int64_t pf_batch_evaluate(pf_ctx *ctx, int64_t n, const double *pts, const double *psi,
                          double tol, double dpsi_max, int ball_aware, int want_m2, int64_t smf,
                          int64_t *status, double *vol, double *ksur, double *cent, double *ipt,
                          double *m2, int64_t *fcount, int64_t *ftag, double *farea, double *fh,
                          double *fnrm, double *fcent, int rebuild_grid, void *stream);

/* Extended form: optional subset of cells to evaluate (cells int32[ncells],
 * original indices; NULL = all), per-cell flag words (cell_flags int32[n],
 * optional) and the algorithmic-work census (census16 int32[n,16], optional;
 * slots = SURVEY.md §8(d) S_cell terms). */
int64_t pf_batch_evaluate_ex(pf_ctx *ctx, int64_t n, const double *pts, const double *psi,
                             double tol, double dpsi_max, int ball_aware, int want_m2, int64_t smf,
                             int64_t *status, double *vol, double *ksur, double *cent, double *ipt,
                             double *m2, int64_t *fcount, int64_t *ftag, double *farea, double *fh,
                             double *fnrm, double *fcent, const int32_t *cells, int64_t ncells,
                             int32_t *cell_flags, int32_t *census16, int rebuild_grid, void *stream);

/* Asynchronous lean variant used by the Newton solver: writes vol, ksur and
 * the restricted facet list (int32 tags / f64 areas, stride smf) and ORs the
 * flag word into *flags (device int64).  No host synchronisation. */
int pf_evaluate_lean(pf_ctx *ctx, int64_t n, const double *pts, const double *psi,
                     int ball_aware, int64_t smf, double *vol, double *ksur, int32_t *fcount,
                     int32_t *ftag, double *farea, double *cent, int64_t *flags, void *stream);

/* pf_batch_evaluate_ex without host synchronisation: the flag word of this
 * call is OR-ed into *err_accum (device int64).  Used to pipeline the host
 * round trip of the drop-in (_kernels._batch_evaluate on host arrays) in
 * chunks of cells: device->host copies of one chunk overlap the next. */
int pf_batch_evaluate_async(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double tol,
                            double dpsi_max, int ball_aware, int want_m2, int64_t smf, int64_t *status,
                            double *vol, double *ksur, double *cent, double *ipt, double *m2,
                            int64_t *fcount, int64_t *ftag, double *farea, double *fh, double *fnrm,
                            double *fcent, const int32_t *cells, int64_t ncells, int32_t *cell_flags,
                            int64_t *err_accum, int rebuild_grid, void *stream);
/* _kernels._batch_evaluate on HOST arrays (the numba call's own argument
 * space: plain, pageable host memory; outputs with the reference shapes).
 * Writes exactly what the reference writes (_kernels.py:1362-1478): every
 * cell's status / vol / ksur / fcount, cent / ipt / m2 except on
 * build-overflow cells, facet slots < fcount only (slots past it untouched).
 * The cells run in `chunks` index ranges (0 = 16); each range's outputs are
 * packed on the device (96 B per cell + 72 B per restricted facet), copied
 * into a pinned ring and scattered into the caller's arrays by a host worker
 * pool while the next ranges compute.  *h2d_bytes / *d2h_bytes (optional)
 * receive the bytes copied.  Returns the OR of the cells' flag words. */
int64_t pf_batch_evaluate_host(pf_ctx *ctx, int64_t n, const double *pts_host, const double *psi_host,
                               double tol, double dpsi_max, int ball_aware, int want_m2, int64_t smf,
                               int64_t *status_host, double *vol_host, double *ksur_host, double *cent_host,
                               double *ipt_host, double *m2_host, int64_t *fcount_host, int64_t *ftag_host,
                               double *farea_host, double *fh_host, double *fnrm_host, double *fcent_host,
                               int chunks, int64_t *h2d_bytes_host, int64_t *d2h_bytes_host);

/* _kernels._batch_build (_kernels.py:1481-1559): every
 * unrestricted Laguerre cell into fixed-stride packed arrays in the reference's
 * layout -- status (0 ok / 1 empty / 3 overflow), counts, verts f64[n,smv,3],
 * planes f64[n,smf,4], tags/lp/lv int64 -- and the OR of the cell flags.
 * Used by laguerre.build_diagram_packed (laguerre.py:226-265). */
int64_t pf_batch_build(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double tol,
                       double dpsi_max, int ball_aware, int64_t smv, int64_t smf, int64_t sml,
                       int64_t *status, int64_t *nv, int64_t *nf, int64_t *nl, double *verts, double *planes,
                       int64_t *tags, int64_t *lp, int64_t *lv, int rebuild_grid, void *stream);

/* bucket-ordered permutation of the sites of the current grid (int32[n]) */
int pf_grid_order(pf_ctx *ctx, int32_t *order, void *stream);

/* per-cell processed-candidate census of the last evaluation (int32[n]) */
int pf_last_census(pf_ctx *ctx, int32_t *census, void *stream);
/* device time (ms) of the cell kernels (both tiers) of the last evaluation */
int pf_last_cells_ms(pf_ctx *ctx, double *ms_host);
/* per-stage device timing of every evaluation after pf_stage_timing(ctx, 1) (resets):
 * total build-kernel ms ("Laguerre") and evaluation-kernel ms ("Evaluation",
 * incl. the capacity-overflow tier) and the evaluation count (cmd_bench) */
int pf_stage_timing(pf_ctx *ctx, int enable);
int pf_stage_times(pf_ctx *ctx, double *build_ms_host, double *eval_ms_host, int64_t *evaluations_host);
/* number of cells that overflowed the shared-memory tier in the last evaluation */
int pf_last_retry_count(pf_ctx *ctx, int64_t *count_host);

/* _kernels._knn for a batch of queries: out_idx i64[nq,k] holds the k
 * nearest sites (by (d^2, index)) of each query (queries f64[nq,3]).
 * rebuild_grid != 0 rebuilds the bucket grid from pts first; 0 reuses the
 * context's grid when it was built on the same (n, pts) -- only for callers
 * that own pts unchanged since that build (the Newton solve).  Returns min(k, n). */
int64_t pf_knn(pf_ctx *ctx, int64_t n, const double *pts, int64_t nq, const double *queries,
               int64_t k, int64_t *out_idx, int rebuild_grid, void *stream);

/* ---- damped Newton solve for the weights ---------------- */
typedef struct {
    int status;           /* 0 converged, 1 max_newton reached, 2 DampingStall, 3 InitFailure */
    int iterations;       /* accepted Newton steps */
    int evaluations;      /* cell evaluations (init + every damping trial) */
    int cg_iterations;    /* total Jacobi-PCG iterations */
    int damping_halvings; /* rejected KMT trials */
    int init_doublings;   /* kappa doublings of the cold start */
    double worst_initial; /* max_i |V_i - nu_i| / nu_i before the first step */
    double worst_final;
    double last_alpha;
    int64_t flags;        /* OR of cell flag words of the last evaluation */
} pf_newton_stats;

/* g = nu - vol; stats_host[3] = (max |vol-nu|/nu, min vol, min nu) */
int pf_newton_gradient(int64_t n, const double *nu, const double *vol, double *g,
                       double *stats_host, void *stream);
/* ELL Hessian rows from a lean evaluation: H_ij = -|B_ij|/(2 D_ij) (site facets only,
 * compacted to hcnt[i] entries), diag = sum_j |B_ij|/(2 D_ij) + |K_i|/(2 sqrt(max(psi, tau))) */
int pf_newton_hessian(int64_t n, int smf, const double *pts, const double *psi, const int32_t *fcount,
                      const int32_t *ftag, const double *farea, const double *ksur, double tau_psi,
                      int32_t *hcnt, int32_t *hcol, double *hval, double *diag, void *stream);
/* Jacobi-PCG, x = H^-1 b to ||r|| <= rtol ||b||; returns the iteration count */
int pf_pcg(int64_t n, int smf, const int32_t *hcnt, const int32_t *hcol, const double *hval,
           const double *diag, const double *b, double *x, double rtol, int max_iter, void *stream);
/* full solve: psi (device, in/out) to max_i |V_i - nu_i|/nu_i <= eps_vol;
 * cold_start != 0 initialises psi = kappa (3 nu / 4 pi)^(2/3) (kappa doubling) */
int pf_newton_solve(pf_ctx *ctx, int64_t n, const double *pts, const double *nu, double *psi,
                    int cold_start, double eps_vol, int max_newton, int smf, double tau_psi,
                    int ball_aware, pf_newton_stats *stats, void *stream);
/* vol / ksur / restricted facets of the solve's final evaluation */
int pf_newton_last_state(double *vol, double *ksur, int32_t *fcount, int32_t *ftag, double *farea,
                         int64_t n, int smf, void *stream);

/* same, plus the centroids of the final evaluation (cent f64[n,3]) */
int pf_newton_last_state_ex(double *vol, double *ksur, int32_t *fcount, int32_t *ftag, double *farea,
                            double *cent, int64_t n, int smf, void *stream);

/* ---- spatially partitioned solve ------------------------
 * A rank owns the cells of its slab; local arrays hold owned + ghost sites in
 * global index order and `rows` lists the owned local indices.  Scalars land
 * in device memory (stats_dev / outN_dev) for the cross-rank all-reduce; the
 * halo exchange of ghost vector entries is done by the host (dist_solver.py).
 * Replaces, per rank, the single-device pf_newton_solve pieces above. */
/* lean evaluation of cells[0:ncells] with the given (global) weight slack;
 * rebuild_grid as in pf_knn */
int pf_evaluate_lean_cells(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double dpsi,
                           int ball_aware, int64_t smf, const int32_t *cells, int64_t ncells,
                           double *vol, double *ksur, int32_t *fcount, int32_t *ftag, double *farea,
                           double *cent, int64_t *flags, int rebuild_grid, void *stream);
/* g = nu - vol on rows; stats_dev[3] = (max rel. error, -min vol, -min nu), MAX-reducible */
int pf_rows_gradient(int nrows, const int32_t *rows, const double *nu, const double *vol, double *g,
                     double *stats_dev, void *stream);
/* Hessian rows (entries as pf_newton_hessian) */
int pf_rows_hessian(int nrows, const int32_t *rows, int smf, const double *pts, const double *psi,
                    const int32_t *fcount, const int32_t *ftag, const double *farea, const double *ksur,
                    double tau_psi, int32_t *hcnt, int32_t *hcol, double *hval, double *diag, void *stream);
/* Jacobi-PCG pieces: init (out2 = partial r.z, b.b), SpMV (out1 = partial p.Ap),
 * update with alpha = *rz / *pAp (out2 = partial r.z, r.r), direction p = z + (*rz_new / *rz_old) p */
int pf_dcg_init(int nrows, const int32_t *rows, const double *b, const double *diag, double *x, double *r,
                double *z, double *p, double *out2_dev, void *stream);
int pf_dcg_spmv(int nrows, const int32_t *rows, int smf, const int32_t *hcnt, const int32_t *hcol,
                const double *hval, const double *diag, const double *p, double *Ap, double *out1_dev,
                void *stream);
int pf_dcg_update(int nrows, const int32_t *rows, const double *diag, double *x, double *r, double *z,
                  const double *p, const double *Ap, const double *rz_dev, const double *pAp_dev,
                  double *out2_dev, void *stream);
int pf_dcg_pdir(int nrows, const int32_t *rows, const double *z, double *p, const double *rz_new_dev,
                const double *rz_old_dev, void *stream);
/* single-reduction Jacobi-PCG (Chronopoulos-Gear), one all-reduce per iteration:
 * init (x = 0, r = b, u = D^-1 b, p = s = 0); spmv_dots: w = A u (u's ghosts exchanged)
 * and out3 = partial (r.u, w.u, r.r); step: scalars from the all-reduced (r.u, w.u)
 * into sc_dev[0..2] (gamma, alpha, beta), then p = u + beta p, s = w + beta s,
 * x += alpha p, r -= alpha s, u = D^-1 r */
int pf_cg1_init(int nrows, const int32_t *rows, const double *b, const double *diag, double *x, double *r,
                double *u, double *p, double *s, void *stream);
int pf_cg1_spmv_dots(int nrows, const int32_t *rows, int smf, const int32_t *hcnt, const int32_t *hcol,
                     const double *hval, const double *diag, const double *u, const double *r, double *w,
                     double *out3_dev, void *stream);
int pf_cg1_step(int nrows, const int32_t *rows, const double *diag, double *x, double *r, double *u,
                const double *w, double *p, double *s, const double *red_dev, double *sc_dev, int first,
                void *stream);
/* the same iteration with the convergence test on the device, so the host
 * reads one flag per batch of iterations instead of one scalar per iteration:
 * sc_dev[3] = ||b||^2, [4] done flag, [5] iterations (zero sc_dev[3..5] before the
 * first iteration).  step_conv applies the test of pf_pcg (||r|| <= rtol ||b||,
 * it >= max_iter, non-finite) to the all-reduced r.r and skips the update once
 * done; spmv_dots_c skips its work once done. */
int pf_cg1_spmv_dots_c(int nrows, const int32_t *rows, int smf, const int32_t *hcnt, const int32_t *hcol,
                       const double *hval, const double *diag, const double *u, const double *r, double *w,
                       double *out3_dev, const double *sc_dev, void *stream);
int pf_cg1_step_conv(int nrows, const int32_t *rows, const double *diag, double *x, double *r, double *u,
                     const double *w, double *p, double *s, const double *red_dev, double *sc_dev, double rtol,
                     int max_iter, void *stream);
/* out = a + s b (n entries) */
int pf_daxpy(int64_t n, const double *a, double s, const double *b, double *out, void *stream);

/* ---- fluid step --------------------------------------- */
/* x += dt v, reflected into the box [lo+tau, hi-tau] (velocity component flipped) */
int pf_fluid_advect(int64_t n, double *x, double *v, double dt, const double *lo_host,
                    const double *hi_host, double tau, void *stream);
/* spring pressure force F_p = k (c - x) / eps^2 (SPEC.md pressure_force):
 * spring = PF_SPRING_SPEC: k = 1, the SPEC as printed (c - x = (eps^2,0,0) -> (1,0,0));
 * spring = PF_SPRING_GM: k = m = rho nu, the Gallouet-Merigot acceleration
 * (c - x)/eps^2 the paper follows.  F f64[n,3]. */
#define PF_SPRING_GM 0
#define PF_SPRING_SPEC 1
int pf_pressure_force(int64_t n, const double *x, const double *cent, const double *nu, const double *rho,
                      double eps, int spring, double *F, void *stream);
/* v += dt/m (F_p + m g), m = rho nu (spring pressure + gravity) */
int pf_fluid_forces(int64_t n, const double *x, const double *cent, const double *nu, const double *rho,
                    double *v, double dt, double eps, const double *g_host, int spring, void *stream);

/* implicit velocity update with viscosity mu (fluid graph Laplacian, P1 weights
 * |B_ij|/(2|p_j-p_i|)), wall friction mu_b (boundary weights, zero wall velocity) and
 * surface tension gamma: three Jacobi-PCG solves of (m/dt I + mu L) v = m/dt v + F_p + F_g + F_t
 * on the final evaluation of the step.  Returns the CG iteration total. */
int pf_fluid_forces_implicit(int64_t n, int smf, const double *x, const double *cent, const double *vol,
                             const int32_t *fcount, const int32_t *ftag, const double *farea, const double *nu,
                             const double *rho, double *v, double dt, double eps, const double *g_host,
                             double mu, double mu_b, double gamma, double affinity, const double *dplanes,
                             int ndom, int spring, int32_t *hcnt, int32_t *hcol, double *hval, double *diag, double *rhs,
                             double *sol, double rtol, void *stream);

/* compact per-facet CSR of an evaluation's fixed-stride facet outputs
 * (SURVEY §8(b)): row_ptr int64[n+1] (row i = the min(fcount[i], smf) facets of
 * cell i, in the fixed-stride order), then per facet tag / area / h (nnz),
 * nrm / cent (nnz*3); any output may be null.  *nnz receives the facet count;
 * more than `cap` facets -> error (call with cap 0 to size the buffers). */
int pf_facets_csr(pf_ctx *ctx, int64_t n, int64_t smf, const int64_t *fcount, const int64_t *ftag,
                  const double *farea, const double *fh, const double *fnrm, const double *fcent, int64_t cap,
                  int64_t *nnz, int64_t *row_ptr, int64_t *tag, double *area, double *h, double *nrm, double *cent,
                  void *stream);

/* ---- renderer ----------------------
 * first hit of one ray per pixel with the fluid (the union of the balls, whose
 * first point along a ray lies in the entered ball's Laguerre cell): hit_id
 * int32[h*w] (-1 miss), hit_t f64[h*w].  cam_host[14] = eye[3], forward[3],
 * right[3], up[3] (unit), tan(fov/2), aspect; rmax = largest ball radius. */
int pf_render_first_hit(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax,
                        const double *cam_host, int width, int height, int32_t *hit_id, double *hit_t,
                        void *stream);

/* Depth mode: in-fluid path length of each pixel ray (the union of the ball
 * chords, clipped to the grid box), f64[h*w]; -1 flags a pixel whose ray met
 * more than 48 ball entries inside one bucket segment (diagnostic pixel). */
int pf_render_depth(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax,
                    const double *cam_host, int width, int height, double *depth, void *stream);

/* Smooth mode: sphere tracing (<= 64 steps, surface eps) of the cubic smooth
 * union of the sphere distances with blend radius k > 0, started just before
 * the Raw hit raw_t (f64[h*w], -1 miss, from pf_render_first_hit); hit_t
 * f64[h*w] (-1 miss), normal f64[h*w*3] (central differences). */
int pf_render_smooth(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax, double k,
                     double eps, const double *cam_host, int width, int height, const double *raw_t,
                     double *hit_t, double *normal, void *stream);

/* smooth_sdf at m device points xq[m*3] -> out[m] (same field as Smooth). */
int pf_smooth_sdf(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax, double k,
                  int64_t m, const double *xq, double *out, void *stream);

/* sample_surface: sample q draws uniform points on sphere cell[q] (int64) until
 * one lies on the free-surface patch K_i -- in the current domain (pf_set_domain)
 * and strictly inside no other ball -- at most max_tries[q] draws; x[m*3],
 * outward unit normal[m*3], status[m] (0 ok, 1 tries exhausted).  Counter-based
 * RNG: the result is a function of (seed, q). */
int pf_sample_surface(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax, int64_t m,
                      const int64_t *cell, const int64_t *max_tries, uint64_t seed, double *x, double *normal,
                      int32_t *status, void *stream);

/* cell-to-cell traversal of m rays (f64[m, 6]: origin, unit direction) through the
 * unrestricted power diagram (cell_nf i32[n], planes f64[n, smf, 4] (n.x <= d), tags
 * i32[n, smf] (site >= 0, domain face < 0): pf_batch_build in full mode), SPEC.md renderer
 * `traverse` (§6): per ray up to max_seg pieces (cell, t_enter, t_exit, fluid), each
 * power-cell span split at the chord of the cell's ball; mode 0 Volume (to the domain exit),
 * 1 SurfaceOnly (up to the first exit through a sphere patch).  status: 0 ok, 1 the ray
 * misses the domain, 2 the 8n-crossing guard or max_seg was reached. */
int pf_traverse(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double psimax, int smf,
                const int32_t *cell_nf, const double *planes, const int32_t *tags, int64_t m, const double *rays,
                int mode, int max_seg, int32_t *out_cell, double *out_t0, double *out_t1, uint8_t *out_fluid,
                int32_t *count, int32_t *status, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* POTFLOW_B200_H */
