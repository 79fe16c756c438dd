// pf_dist.cu -- the row-subset kernels of the spatially partitioned Newton
// solve (SPEC.md:286-335 for the algorithm).
//
// A rank owns the cells of its slab; its local arrays hold owned + ghost
// sites in global index order (partition.py), so every kernel here works on a
// list of owned local rows.  Vectors are local-length; their ghost entries are
// filled by the host-side halo exchange (dist_solver.py) before a SpMV.  The
// scalar reductions (dots, gradient statistics) leave per-rank partial values
// in device memory for the all-reduce; every reduction is two-level over a
// fixed block count, so the per-rank partials are bitwise reproducible.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/potflow_b200.h"

extern unsigned long long pf_internal_launches_add(unsigned long long k);
extern int pf_internal_set_err(const char *msg);

namespace {

constexpr int DB = 256;   // threads per block
constexpr int DNB = 296;  // blocks (2 per SM): fixed, so the reductions are reproducible

#define DCK(x)                                                                       \
    do {                                                                             \
        cudaError_t _e = (x);                                                        \
        if (_e != cudaSuccess) {                                                     \
            char _b[256];                                                            \
            snprintf(_b, sizeof _b, "%s:%d %s: %s", __FILE__, __LINE__, #x,         \
                     cudaGetErrorString(_e));                                        \
            return pf_internal_set_err(_b);                                          \
        }                                                                            \
    } while (0)

double *g_part = nullptr;  // [4][DNB] block partials

int part_alloc() {
    if (!g_part) DCK(cudaMalloc(&g_part, 4 * DNB * sizeof(double)));
    return 0;
}

__device__ __forceinline__ double nanmax(double a, double b) { return (a != a || b != b) ? NAN : fmax(a, b); }

// block reduction of K values; op 0 = sum, 1 = NaN-propagating max
template <int K>
__device__ __forceinline__ void block_reduce(double (&v)[K], const int (&op)[K]) {
    __shared__ double sh[K][DB / 32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; k++) {
        double x = v[k];
        for (int m = 16; m > 0; m >>= 1) {
            double o = __shfl_xor_sync(0xffffffffu, x, m);
            x = op[k] ? nanmax(x, o) : x + o;
        }
        if (l == 0) sh[k][w] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) {
            double x = sh[k][0];
            for (int q = 1; q < DB / 32; q++) x = op[k] ? nanmax(x, sh[k][q]) : x + sh[k][q];
            v[k] = x;
        }
    }
}

// final pass over the block partials -> out[k]
template <int K>
__global__ void __launch_bounds__(DB) k_finish(const double *__restrict__ part, double *__restrict__ out,
                                               int o0, int o1, int o2, int o3) {
    const int op_all[4] = {o0, o1, o2, o3};
    double v[K];
    int op[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        op[k] = op_all[k];
        double x = op[k] ? -INFINITY : 0.0;
        for (int b = threadIdx.x; b < DNB; b += DB) x = op[k] ? nanmax(x, part[k * DNB + b]) : x + part[k * DNB + b];
        v[k] = x;
    }
    block_reduce<K>(v, op);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; k++) out[k] = v[k];
}

// g = nu - vol on the rows; (worst relative error, -min vol, -min nu): all MAX-reducible
__global__ void __launch_bounds__(DB) k_rows_grad(int nrows, const int *__restrict__ rows,
                                                  const double *__restrict__ nu, const double *__restrict__ vol,
                                                  double *__restrict__ g, double *__restrict__ part) {
    double v3[3] = {0.0, -INFINITY, -INFINITY};
    const int op[3] = {1, 1, 1};
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int i = rows[t];
        const double v = vol[i], n = nu[i];
        if (g) g[i] = n - v;
        const double e = fabs(v - n) / n;
        v3[0] = nanmax(v3[0], e);
        v3[1] = nanmax(v3[1], -v);
        v3[2] = fmax(v3[2], -n);
    }
    block_reduce<3>(v3, op);
    if (threadIdx.x == 0)
        for (int k = 0; k < 3; k++) part[k * DNB + blockIdx.x] = v3[k];
}

// Hessian rows (same entries as pf_newton_hessian)
__global__ void __launch_bounds__(DB) k_rows_hessian(int nrows, const int *__restrict__ rows, int smf,
                                                     const double *__restrict__ pts, const double *__restrict__ psi,
                                                     const int *__restrict__ fcount, const int *__restrict__ ftag,
                                                     const double *__restrict__ farea,
                                                     const double *__restrict__ ksur, double tau_psi,
                                                     int *__restrict__ hcnt, int *__restrict__ hcol,
                                                     double *__restrict__ hval, double *__restrict__ diag) {
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int64_t i = rows[t];
        const double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
        int c = fcount[i];
        if (c > smf) c = smf;
        double d = 0.0;
        int k = 0;
        for (int s = 0; s < c; s++) {
            const int64_t j = ftag[i * smf + s];
            if (j < 0) continue;
            const double dx = pts[3 * j] - px, dy = pts[3 * j + 1] - py, dz = pts[3 * j + 2] - pz;
            const double w = 0.5 * farea[i * smf + s] / sqrt(dx * dx + dy * dy + dz * dz);
            hcol[i * smf + k] = (int)j;
            hval[i * smf + k] = -w;
            d += w;
            k++;
        }
        const double ps = psi[i] > tau_psi ? psi[i] : tau_psi;
        d += 0.5 * ksur[i] / sqrt(ps);
        if (!(d > 0.0)) d = 2.0 * 3.141592653589793 * sqrt(ps);
        diag[i] = d;
        hcnt[i] = k;
    }
}

// x = 0, r = b, z = p = b / diag; partial (r.z, b.b)
__global__ void __launch_bounds__(DB) k_dcg_init(int nrows, const int *__restrict__ rows,
                                                 const double *__restrict__ b, const double *__restrict__ diag,
                                                 double *__restrict__ x, double *__restrict__ r,
                                                 double *__restrict__ z, double *__restrict__ p,
                                                 double *__restrict__ part) {
    double v[2] = {0.0, 0.0};
    const int op[2] = {0, 0};
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int i = rows[t];
        const double bi = b[i], zi = bi / diag[i];
        x[i] = 0.0; r[i] = bi; z[i] = zi; p[i] = zi;
        v[0] += bi * zi;
        v[1] += bi * bi;
    }
    block_reduce<2>(v, op);
    if (threadIdx.x == 0) { part[blockIdx.x] = v[0]; part[DNB + blockIdx.x] = v[1]; }
}

// Ap = H p on the rows (p's ghost entries already exchanged); partial p.Ap
__global__ void __launch_bounds__(DB) k_dcg_spmv(int nrows, const int *__restrict__ rows, int smf,
                                                 const int *__restrict__ hcnt, const int *__restrict__ hcol,
                                                 const double *__restrict__ hval, const double *__restrict__ diag,
                                                 const double *__restrict__ p, double *__restrict__ Ap,
                                                 double *__restrict__ part) {
    double v[1] = {0.0};
    const int op[1] = {0};
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int64_t i = rows[t];
        double s = diag[i] * p[i];
        const int c = hcnt[i];
        const int *col = hcol + i * smf;
        const double *val = hval + i * smf;
        for (int k = 0; k < c; k++) s += val[k] * p[col[k]];
        Ap[i] = s;
        v[0] += p[i] * s;
    }
    block_reduce<1>(v, op);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// alpha = rz / pAp (global scalars); x += alpha p, r -= alpha Ap, z = r / diag;
// partial (r.z, r.r)
__global__ void __launch_bounds__(DB) k_dcg_update(int nrows, const int *__restrict__ rows,
                                                   const double *__restrict__ diag, double *__restrict__ x,
                                                   double *__restrict__ r, double *__restrict__ z,
                                                   const double *__restrict__ p, const double *__restrict__ Ap,
                                                   const double *__restrict__ rz, const double *__restrict__ pAp,
                                                   double *__restrict__ part) {
    const double alpha = *pAp != 0.0 ? *rz / *pAp : 0.0;
    double v[2] = {0.0, 0.0};
    const int op[2] = {0, 0};
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int i = rows[t];
        const double xi = x[i] + alpha * p[i];
        const double ri = r[i] - alpha * Ap[i];
        const double zi = ri / diag[i];
        x[i] = xi; r[i] = ri; z[i] = zi;
        v[0] += ri * zi;
        v[1] += ri * ri;
    }
    block_reduce<2>(v, op);
    if (threadIdx.x == 0) { part[blockIdx.x] = v[0]; part[DNB + blockIdx.x] = v[1]; }
}

// p = z + (rz_new / rz_old) p
__global__ void __launch_bounds__(DB) k_dcg_pdir(int nrows, const int *__restrict__ rows,
                                                 const double *__restrict__ z, double *__restrict__ p,
                                                 const double *__restrict__ rz_new,
                                                 const double *__restrict__ rz_old) {
    const double beta = *rz_old != 0.0 ? *rz_new / *rz_old : 0.0;
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int i = rows[t];
        p[i] = z[i] + beta * p[i];
    }
}

// ---- single-reduction PCG (Chronopoulos & Gear): one all-reduce per iteration ----
// sc (device, caller-owned, 8 doubles): [0] gamma = r.u, [1] alpha, [2] beta
// w = A u and partial (r.u, w.u, r.r) -> part, to be all-reduced by the caller
__global__ void __launch_bounds__(DB) k_cg1_spmv_dots(int nrows, const int *__restrict__ rows, int smf,
                                                      const int *__restrict__ hcnt, const int *__restrict__ hcol,
                                                      const double *__restrict__ hval,
                                                      const double *__restrict__ diag, const double *__restrict__ u,
                                                      const double *__restrict__ r, double *__restrict__ w,
                                                      double *__restrict__ part,
                                                      const double *__restrict__ sc = nullptr) {
    double v[3] = {0.0, 0.0, 0.0};
    if (sc && sc[4] != 0.0) {  // converged (device-side test): partials of zero, no work
        if (threadIdx.x == 0)
            for (int k = 0; k < 3; k++) part[k * DNB + blockIdx.x] = 0.0;
        return;
    }
    const int op[3] = {0, 0, 0};
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int64_t i = rows[t];
        double s = diag[i] * u[i];
        const int c = hcnt[i];
        const int *col = hcol + i * smf;
        const double *val = hval + i * smf;
        for (int k = 0; k < c; k++) s += val[k] * u[col[k]];
        w[i] = s;
        v[0] += r[i] * u[i];
        v[1] += s * u[i];
        v[2] += r[i] * r[i];
    }
    block_reduce<3>(v, op);
    if (threadIdx.x == 0)
        for (int k = 0; k < 3; k++) part[k * DNB + blockIdx.x] = v[k];
}

// scalars from the reduced (gamma_new, delta): first iteration alpha = gamma/delta,
// then beta = gamma_new/gamma, alpha = gamma_new / (delta - beta gamma_new / alpha)
__global__ void k_cg1_scalars(const double *__restrict__ red, double *__restrict__ sc, int first) {
    const double g = red[0], dl = red[1];
    double beta = 0.0, alpha;
    if (first) {
        alpha = dl != 0.0 ? g / dl : 0.0;
    } else {
        beta = sc[0] != 0.0 ? g / sc[0] : 0.0;
        const double den = dl - (sc[1] != 0.0 ? beta * g / sc[1] : 0.0);
        alpha = den != 0.0 ? g / den : 0.0;
    }
    sc[0] = g; sc[1] = alpha; sc[2] = beta;
}

// the same with the convergence test of pf_pcg on the device (sc[3] = b.b,
// sc[4] = done, sc[5] = iterations); red = all-reduced (r.u, w.u, r.r)
__global__ void k_cg1_scalars_conv(const double *__restrict__ red, double *__restrict__ sc, double rtol,
                                   int max_iter) {
    if (sc[4] != 0.0) return;
    const int it = (int)sc[5];
    const double rr = red[2];
    if (it == 0) {
        sc[3] = rr;
        if (!(rr > 0.0)) { sc[4] = 1.0; return; }
    } else if (sqrt(rr) <= rtol * sqrt(sc[3]) || it >= max_iter || !isfinite(rr)) {
        sc[4] = 1.0;
        return;
    }
    const double g = red[0], dl = red[1];
    double beta = 0.0, alpha;
    if (it == 0) {
        alpha = dl != 0.0 ? g / dl : 0.0;
    } else {
        beta = sc[0] != 0.0 ? g / sc[0] : 0.0;
        const double den = dl - (sc[1] != 0.0 ? beta * g / sc[1] : 0.0);
        alpha = den != 0.0 ? g / den : 0.0;
    }
    sc[0] = g; sc[1] = alpha; sc[2] = beta;
    sc[5] = it + 1;
}

// p = u + beta p; s = w + beta s; x += alpha p; r -= alpha s; u = r / diag
__global__ void __launch_bounds__(DB) k_cg1_update(int nrows, const int *__restrict__ rows,
                                                   const double *__restrict__ diag, double *__restrict__ x,
                                                   double *__restrict__ r, double *__restrict__ u,
                                                   const double *__restrict__ w, double *__restrict__ p,
                                                   double *__restrict__ s, const double *__restrict__ sc,
                                                   int conv = 0) {
    if (conv && sc[4] != 0.0) return;
    const double alpha = sc[1], beta = sc[2];
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int i = rows[t];
        const double pi = u[i] + beta * p[i];
        const double si = w[i] + beta * s[i];
        p[i] = pi;
        s[i] = si;
        x[i] += alpha * pi;
        const double ri = r[i] - alpha * si;
        r[i] = ri;
        u[i] = ri / diag[i];
    }
}

// x = 0, r = b, u = b / diag, p = s = 0
__global__ void __launch_bounds__(DB) k_cg1_init(int nrows, const int *__restrict__ rows,
                                                 const double *__restrict__ b, const double *__restrict__ diag,
                                                 double *__restrict__ x, double *__restrict__ r,
                                                 double *__restrict__ u, double *__restrict__ p,
                                                 double *__restrict__ s) {
    for (int t = blockIdx.x * DB + threadIdx.x; t < nrows; t += DNB * DB) {
        const int i = rows[t];
        x[i] = 0.0; r[i] = b[i]; u[i] = b[i] / diag[i]; p[i] = 0.0; s[i] = 0.0;
    }
}

// out = a + s b on all n local entries
__global__ void __launch_bounds__(DB) k_daxpy(int64_t n, const double *__restrict__ a, double s,
                                              const double *__restrict__ b, double *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)DB + threadIdx.x; i < n; i += (int64_t)DNB * DB) out[i] = a[i] + s * b[i];
}

}  // namespace

extern "C" {

int pf_rows_gradient(int nrows, const int32_t *rows, const double *nu, const double *vol, double *g,
                     double *stats_dev, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (part_alloc()) return -1;
    pf_internal_launches_add(2);
    k_rows_grad<<<DNB, DB, 0, st>>>(nrows, rows, nu, vol, g, g_part);
    k_finish<3><<<1, DB, 0, st>>>(g_part, stats_dev, 1, 1, 1, 1);
    DCK(cudaGetLastError());
    return 0;
}

int pf_rows_hessian(int nrows, const int32_t *rows, int smf, const double *pts, const double *psi,
                    const int32_t *fcount, const int32_t *ftag, const double *farea, const double *ksur,
                    double tau_psi, int32_t *hcnt, int32_t *hcol, double *hval, double *diag, void *stream) {
    pf_internal_launches_add(1);
    k_rows_hessian<<<DNB, DB, 0, (cudaStream_t)stream>>>(nrows, rows, smf, pts, psi, fcount, ftag, farea, ksur,
                                                         tau_psi, hcnt, hcol, hval, diag);
    DCK(cudaGetLastError());
    return 0;
}

int pf_dcg_init(int nrows, const int32_t *rows, const double *b, const double *diag, double *x, double *r,
                double *z, double *p, double *out2_dev, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (part_alloc()) return -1;
    pf_internal_launches_add(2);
    k_dcg_init<<<DNB, DB, 0, st>>>(nrows, rows, b, diag, x, r, z, p, g_part);
    k_finish<2><<<1, DB, 0, st>>>(g_part, out2_dev, 0, 0, 0, 0);
    DCK(cudaGetLastError());
    return 0;
}

int pf_dcg_spmv(int nrows, const int32_t *rows, int smf, const int32_t *hcnt, const int32_t *hcol,
                const double *hval, const double *diag, const double *p, double *Ap, double *out1_dev,
                void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (part_alloc()) return -1;
    pf_internal_launches_add(2);
    k_dcg_spmv<<<DNB, DB, 0, st>>>(nrows, rows, smf, hcnt, hcol, hval, diag, p, Ap, g_part);
    k_finish<1><<<1, DB, 0, st>>>(g_part, out1_dev, 0, 0, 0, 0);
    DCK(cudaGetLastError());
    return 0;
}

int pf_dcg_update(int nrows, const int32_t *rows, const double *diag, double *x, double *r, double *z,
                  const double *p, const double *Ap, const double *rz_dev, const double *pAp_dev,
                  double *out2_dev, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (part_alloc()) return -1;
    pf_internal_launches_add(2);
    k_dcg_update<<<DNB, DB, 0, st>>>(nrows, rows, diag, x, r, z, p, Ap, rz_dev, pAp_dev, g_part);
    k_finish<2><<<1, DB, 0, st>>>(g_part, out2_dev, 0, 0, 0, 0);
    DCK(cudaGetLastError());
    return 0;
}

int pf_dcg_pdir(int nrows, const int32_t *rows, const double *z, double *p, const double *rz_new_dev,
                const double *rz_old_dev, void *stream) {
    pf_internal_launches_add(1);
    k_dcg_pdir<<<DNB, DB, 0, (cudaStream_t)stream>>>(nrows, rows, z, p, rz_new_dev, rz_old_dev);
    DCK(cudaGetLastError());
    return 0;
}

int pf_cg1_init(int nrows, const int32_t *rows, const double *b, const double *diag, double *x, double *r,
                double *u, double *p, double *s, void *stream) {
    pf_internal_launches_add(1);
    k_cg1_init<<<DNB, DB, 0, (cudaStream_t)stream>>>(nrows, rows, b, diag, x, r, u, p, s);
    DCK(cudaGetLastError());
    return 0;
}

int pf_cg1_spmv_dots(int nrows, const int32_t *rows, int smf, const int32_t *hcnt, const int32_t *hcol,
                     const double *hval, const double *diag, const double *u, const double *r, double *w,
                     double *out3_dev, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (part_alloc()) return -1;
    pf_internal_launches_add(2);
    k_cg1_spmv_dots<<<DNB, DB, 0, st>>>(nrows, rows, smf, hcnt, hcol, hval, diag, u, r, w, g_part);
    k_finish<3><<<1, DB, 0, st>>>(g_part, out3_dev, 0, 0, 0, 0);
    DCK(cudaGetLastError());
    return 0;
}

int pf_cg1_step(int nrows, const int32_t *rows, const double *diag, double *x, double *r, double *u,
                const double *w, double *p, double *s, const double *red_dev, double *sc_dev, int first,
                void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    pf_internal_launches_add(2);
    k_cg1_scalars<<<1, 1, 0, st>>>(red_dev, sc_dev, first);
    k_cg1_update<<<DNB, DB, 0, st>>>(nrows, rows, diag, x, r, u, w, p, s, sc_dev);
    DCK(cudaGetLastError());
    return 0;
}

int pf_cg1_spmv_dots_c(int nrows, const int32_t *rows, int smf, const int32_t *hcnt, const int32_t *hcol,
                       const double *hval, const double *diag, const double *u, const double *r, double *w,
                       double *out3_dev, const double *sc_dev, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (part_alloc()) return -1;
    pf_internal_launches_add(2);
    k_cg1_spmv_dots<<<DNB, DB, 0, st>>>(nrows, rows, smf, hcnt, hcol, hval, diag, u, r, w, g_part, sc_dev);
    k_finish<3><<<1, DB, 0, st>>>(g_part, out3_dev, 0, 0, 0, 0);
    DCK(cudaGetLastError());
    return 0;
}

int pf_cg1_step_conv(int nrows, const int32_t *rows, const double *diag, double *x, double *r, double *u,
                     const double *w, double *p, double *s, const double *red_dev, double *sc_dev, double rtol,
                     int max_iter, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    pf_internal_launches_add(2);
    k_cg1_scalars_conv<<<1, 1, 0, st>>>(red_dev, sc_dev, rtol, max_iter);
    k_cg1_update<<<DNB, DB, 0, st>>>(nrows, rows, diag, x, r, u, w, p, s, sc_dev, 1);
    DCK(cudaGetLastError());
    return 0;
}

int pf_daxpy(int64_t n, const double *a, double s, const double *b, double *out, void *stream) {
    pf_internal_launches_add(1);
    k_daxpy<<<DNB, DB, 0, (cudaStream_t)stream>>>(n, a, s, b, out);
    DCK(cudaGetLastError());
    return 0;
}

}  // extern "C"
