// pf_newton.cu -- damped Newton (KMT) solve for the Laguerre weights on the
// device (the reference ships the
// algorithm only as specification).
//
//   g_i  = nu_i - |V_i|
//   H    = -grad^2 K:  H_ij = -1/2 |B_ij| / |p_j - p_i|        (PAPER Eq. 2)
//          H_ii = sum_j 1/2 |B_ij| / |p_j - p_i| + 1/2 |K_i| / sqrt(max(psi_i, tau_psi))
//   H u = g by Jacobi-preconditioned CG, rtol 1e-3 (1e-4 once worst < 10 eps)
//   psi <- psi + alpha u, alpha halved until min_i |V_i| >= 1/2 min(min nu, min |V(psi0)|)
//
// Matrix layout: the cell kernel's restricted-facet list is an ELL matrix
// (row = cell, stride smf, int32 columns, f64 values); assembly compacts each
// row to its site facets.  All reductions are two-level with a fixed block
// count, so every number is bitwise reproducible run to run.
#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/potflow_b200.h"

extern unsigned long long pf_internal_launches_add(unsigned long long k);
extern int pf_internal_set_err(const char *msg);

namespace {

constexpr int RB = 256;      // threads per block for vector kernels
constexpr int NPART = 1024;  // fixed number of partial sums (deterministic reductions)

#define NCK(x)                                                                       \
    do {                                                                             \
        cudaError_t _e = (x);                                                        \
        if (_e != cudaSuccess) {                                                     \
            char _b[256];                                                            \
            snprintf(_b, sizeof _b, "%s:%d %s: %s", __FILE__, __LINE__, #x,         \
                     cudaGetErrorString(_e));                                        \
            return pf_internal_set_err(_b);                                          \
        }                                                                            \
    } while (0)

__device__ __forceinline__ double block_sum(double v, double *sh) {
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) s += sh[k];
    __syncthreads();
    return s;
}
__device__ __forceinline__ double nanmax(double a, double b) { return (a != a || b != b) ? NAN : fmax(a, b); }
__device__ __forceinline__ double block_max(double v, double *sh) {
    for (int m = 16; m > 0; m >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, m));
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = -INFINITY;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) s = nanmax(s, sh[k]);
    __syncthreads();
    return s;
}
__device__ __forceinline__ double block_min(double v, double *sh) {
    return -block_max(-v, sh);
}

// gradient, worst relative volume error, min volume (partials per block)
__global__ void __launch_bounds__(RB) k_grad(int64_t n, const double *__restrict__ nu,
                                            const double *__restrict__ vol, double *__restrict__ g,
                                            double *__restrict__ part) {
    __shared__ double sh[32];
    double worst = 0.0, vmin = INFINITY, nmin = INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        double v = vol[i], t = nu[i];
        if (g) g[i] = t - v;
        double e = fabs(v - t) / t;
        if (!(e <= worst)) worst = e;  // NaN-propagating max / min
        if (!(v >= vmin)) vmin = v;
        nmin = fmin(nmin, t);
    }
    double a = block_max(worst, sh), b = block_min(vmin, sh), c = block_min(nmin, sh);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = a;
        part[NPART + blockIdx.x] = b;
        part[2 * NPART + blockIdx.x] = c;
    }
}

// final reduce of the three partial arrays -> out[0]=worst, out[1]=min vol, out[2]=min nu
__global__ void k_grad_fin(const double *__restrict__ part, int nb, double *out) {
    __shared__ double sh[32];
    double a = 0.0, b = INFINITY, c = INFINITY;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        a = nanmax(a, part[k]);
        b = -nanmax(-b, -part[NPART + k]);
        c = fmin(c, part[2 * NPART + k]);
    }
    a = block_max(a, sh);
    b = block_min(b, sh);
    c = block_min(c, sh);
    if (threadIdx.x == 0) { out[0] = a; out[1] = b; out[2] = c; }
}

// Hessian rows: compact site facets of each cell's restricted-facet list
__global__ void __launch_bounds__(RB) k_hessian(int64_t n, int smf, const double *__restrict__ pts,
                                               const double *__restrict__ psi,
                                               const int *__restrict__ fcount,
                                               const int *__restrict__ ftag,
                                               const double *__restrict__ farea,
                                               const double *__restrict__ ksur, double tau_psi,
                                               int *__restrict__ hcnt, int *__restrict__ hcol,
                                               double *__restrict__ hval, double *__restrict__ diag) {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        const double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
        int c = fcount[i];
        if (c > smf) c = smf;
        double d = 0.0;
        int k = 0;
        for (int s = 0; s < c; s++) {
            int j = ftag[i * smf + s];
            if (j < 0) continue;
            double dx = pts[3 * j] - px, dy = pts[3 * j + 1] - py, dz = pts[3 * j + 2] - pz;
            double w = 0.5 * farea[i * smf + s] / sqrt(dx * dx + dy * dy + dz * dz);
            hcol[i * smf + k] = j;
            hval[i * smf + k] = -w;
            d += w;
            k++;
        }
        double ps = psi[i] > tau_psi ? psi[i] : tau_psi;
        d += 0.5 * ksur[i] / sqrt(ps);
        // an empty cell has no volume derivative; regularise with the free
        // ball's d|V|/dpsi = 2 pi sqrt(psi) so Jacobi/CG stay defined
        if (!(d > 0.0)) d = 2.0 * 3.141592653589793 * sqrt(ps);
        diag[i] = d;
        hcnt[i] = k;
    }
}

// ---- Jacobi-PCG: one cooperative persistent kernel on a SELL-32 copy -------
// The iterations read the Hessian as SELL-32 (Kreutzer et al.): slices of 32
// consecutive rows, each slice column-major and padded to its longest row, so
// a warp reads a slice's values and columns as fully coalesced 256 B / 128 B
// lines and every lane (= row) has its gathers for several entries in
// flight.  Matrix loads carry the evict-first (streaming) hint, so the
// vectors (x, r, z, two direction buffers, Ap, diag: 7 x 8 B per row, 112 MB
// at 2M rows) stay resident in the 126 MB L2 while the matrix streams past.
//
// Per iteration two grid-wide barriers:
//   A  p = z + beta p_old (formed where it is consumed: for the own row and
//      for every gathered column), Ap = H p, partial p.Ap        | grid.sync
//   B  x += alpha p, r -= alpha Ap, z = r / diag, partial r.z, r.r | grid.sync
// Every block reduces the per-block partials itself in one fixed order, so
// all blocks take the same (bitwise reproducible) decisions and the host is
// not involved until the solve ends.
constexpr int SELL_C = 32;
__global__ void __launch_bounds__(RB) k_sell_pack(int64_t n, int smf, const int *__restrict__ hcnt,
                                                 const int *__restrict__ hcol, const double *__restrict__ hval,
                                                 int *__restrict__ scol, double *__restrict__ sval,
                                                 int *__restrict__ swid) {
    const int l = threadIdx.x & 31;
    const int64_t ns = (n + SELL_C - 1) / SELL_C;
    const int64_t wstride = ((int64_t)gridDim.x * RB) >> 5;
    for (int64_t s = (blockIdx.x * (int64_t)RB + threadIdx.x) >> 5; s < ns; s += wstride) {
        const int64_t i = s * SELL_C + l;
        const int c = i < n ? hcnt[i] : 0;
        const int w = __reduce_max_sync(0xffffffffu, c);
        if (l == 0) swid[s] = w;
        const size_t base = (size_t)s * SELL_C * smf + l;
        const int pad = (int)(i < n ? i : s * SELL_C);  // padding gathers the own row's entry (cached)
        for (int m = 0; m < w; m++) {
            const bool on = m < c;
            scol[base + (size_t)m * SELL_C] = on ? hcol[i * smf + m] : pad;
            sval[base + (size_t)m * SELL_C] = on ? hval[i * smf + m] : 0.0;
        }
    }
}

constexpr int CG_T = 512;
__device__ __forceinline__ void all_reduce2(const double *__restrict__ part, int G, double *a_out,
                                            double *b_out, double *sh) {
    // fixed order: lane l sums part[l], part[l+32], ...; then a fixed shuffle tree
    if (threadIdx.x < 32) {
        double a = 0.0, b = 0.0;
        for (int k = threadIdx.x; k < G; k += 32) { a += __ldcg(part + k); b += __ldcg(part + G + k); }
        for (int m = 16; m > 0; m >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, m);
            b += __shfl_xor_sync(0xffffffffu, b, m);
        }
        if (threadIdx.x == 0) { sh[0] = a; sh[1] = b; }
    }
    __syncthreads();
    *a_out = sh[0];
    *b_out = sh[1];
    __syncthreads();
}
__device__ __forceinline__ double block_sum_all(double v, double *sh) {
    // block sum with the result in every thread (fixed tree)
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        double s = l < (int)(blockDim.x >> 5) ? sh[l] : 0.0;
        for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        if (l == 0) sh[32] = s;
    }
    __syncthreads();
    const double r = sh[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(CG_T, 2)
    k_pcg_sell(int64_t n, int smf, const int *__restrict__ scol, const double *__restrict__ sval,
               const int *__restrict__ swid, const double *__restrict__ diag, const double *__restrict__ b,
               double *__restrict__ x, double *__restrict__ r, double *__restrict__ z, double *__restrict__ pa,
               double *__restrict__ pb, double *__restrict__ Ap, double *__restrict__ part, double rtol,
               int max_iter, int *__restrict__ out_it) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[40];
    const int G = gridDim.x;
    const int64_t ns = (n + SELL_C - 1) / SELL_C;
    // this block's slices [s0, s1) and rows [lo, hi)
    const int64_t s0 = ns * blockIdx.x / G, s1 = ns * (blockIdx.x + 1) / G;
    const int64_t lo = s0 * SELL_C, hi = s1 * SELL_C < n ? s1 * SELL_C : n;
    const int wib = threadIdx.x >> 5, nwb = CG_T >> 5, l = threadIdx.x & 31;
    double *partA = part, *partB = part + 2 * G;
    // x = 0, r = b, z = D^-1 b, p_old = 0 (beta = 0: p_0 = z_0)
    double rz_p = 0.0, bb_p = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += CG_T) {
        const double bi = b[i], zi = bi / diag[i];
        x[i] = 0.0; r[i] = bi; z[i] = zi; pa[i] = 0.0;
        rz_p += bi * zi;
        bb_p += bi * bi;
    }
    rz_p = block_sum_all(rz_p, sh);
    bb_p = block_sum_all(bb_p, sh);
    if (threadIdx.x == 0) { partB[blockIdx.x] = rz_p; partB[G + blockIdx.x] = bb_p; }
    grid.sync();
    double rz, bb;
    all_reduce2(partB, G, &rz, &bb, sh);
    int it = 0;
    double beta = 0.0;
    double *pold = pa, *pnew = pb;
    if (bb > 0.0) {
        for (;;) {
            // A: p = z + beta p_old, Ap = H p (lane per row of a slice), partial p.Ap
            double pap = 0.0;
            for (int64_t s = s0 + wib; s < s1; s += nwb) {
                const int64_t i = s * SELL_C + l;
                const int w = swid[s];
                const int *__restrict__ cc = scol + (size_t)s * SELL_C * smf + l;
                const double *__restrict__ vv = sval + (size_t)s * SELL_C * smf + l;
                double acc = 0.0;
                int m = 0;
                for (; m + 4 <= w; m += 4) {  // four entries' loads and gathers in flight
                    const int c0 = __ldcs(cc), c1 = __ldcs(cc + SELL_C), c2 = __ldcs(cc + 2 * SELL_C),
                              c3 = __ldcs(cc + 3 * SELL_C);
                    const double v0 = __ldcs(vv), v1 = __ldcs(vv + SELL_C), v2 = __ldcs(vv + 2 * SELL_C),
                                 v3 = __ldcs(vv + 3 * SELL_C);
                    const double q0 = z[c0] + beta * pold[c0], q1 = z[c1] + beta * pold[c1];
                    const double q2 = z[c2] + beta * pold[c2], q3 = z[c3] + beta * pold[c3];
                    acc += v0 * q0; acc += v1 * q1; acc += v2 * q2; acc += v3 * q3;
                    cc += 4 * SELL_C; vv += 4 * SELL_C;
                }
                for (; m < w; m++) {
                    const int c0 = __ldcs(cc);
                    const double v0 = __ldcs(vv);
                    acc += v0 * (z[c0] + beta * pold[c0]);
                    cc += SELL_C; vv += SELL_C;
                }
                if (i < n) {
                    const double di = diag[i];
                    const double pi = z[i] + beta * pold[i];
                    pnew[i] = pi;
                    acc += di * pi;
                    Ap[i] = acc;
                    pap += pi * acc;
                }
            }
            pap = block_sum_all(pap, sh);
            if (threadIdx.x == 0) { partA[blockIdx.x] = pap; partA[G + blockIdx.x] = 0.0; }
            grid.sync();
            double pAp, dummy;
            all_reduce2(partA, G, &pAp, &dummy, sh);
            const double alpha = pAp != 0.0 ? rz / pAp : 0.0;
            // B: x += alpha p, r -= alpha Ap, z = r / diag, partial r.z and r.r
            double rzn = 0.0, rr = 0.0;
            for (int64_t i = lo + threadIdx.x; i < hi; i += CG_T) {
                const double ri = r[i] - alpha * Ap[i];
                x[i] = x[i] + alpha * pnew[i];
                r[i] = ri;
                const double zi = ri / diag[i];
                z[i] = zi;
                rzn += ri * zi;
                rr += ri * ri;
            }
            rzn = block_sum_all(rzn, sh);
            rr = block_sum_all(rr, sh);
            if (threadIdx.x == 0) { partB[blockIdx.x] = rzn; partB[G + blockIdx.x] = rr; }
            grid.sync();
            double rz_new, rr_all;
            all_reduce2(partB, G, &rz_new, &rr_all, sh);
            beta = rz != 0.0 ? rz_new / rz : 0.0;
            rz = rz_new;
            it++;
            if (sqrt(rr_all) <= rtol * sqrt(bb) || it >= max_iter || !(rz_new == rz_new)) break;
            double *t = pold; pold = pnew; pnew = t;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out_it = it;
}

__global__ void __launch_bounds__(RB) k_axpy_to(int64_t n, const double *__restrict__ a, double s,
                                               const double *__restrict__ b, double *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB)
        out[i] = a[i] + s * b[i];
}

// list of the empty cells and their positions
__global__ void __launch_bounds__(RB) k_empty_list(int64_t n, const double *__restrict__ vol,
                                                  const double *__restrict__ pts, int *__restrict__ list,
                                                  double *__restrict__ q, int *__restrict__ count) {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB)
        if (!(vol[i] > 0.0)) {
            const int k = atomicAdd(count, 1);
            list[k] = (int)i;
            q[3 * k] = pts[3 * i]; q[3 * k + 1] = pts[3 * i + 1]; q[3 * k + 2] = pts[3 * i + 2];
        }
}
// psi_i <- max(psi_i, psi_j), j the nearest other site of the empty cell i
__global__ void __launch_bounds__(RB) k_rescue_nn(int m, const int *__restrict__ list,
                                                 const int64_t *__restrict__ nn, double *__restrict__ psi) {
    for (int t = blockIdx.x * RB + threadIdx.x; t < m; t += gridDim.x * RB) {
        const int i = list[t];
        const int64_t j = nn[2 * t] == i ? nn[2 * t + 1] : nn[2 * t];
        if (j >= 0 && psi[j] > psi[i]) psi[i] = psi[j];
    }
}

// rescue of the cells a warm start leaves empty (SPEC.md init_weights)
__global__ void __launch_bounds__(RB) k_rescue(int64_t n, const double *__restrict__ nu,
                                              const double *__restrict__ vol, double kappa,
                                              double *__restrict__ psi) {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB)
        if (!(vol[i] > 0.0)) {
            const double r = kappa * pow(3.0 * nu[i] / (4.0 * 3.141592653589793), 2.0 / 3.0);
            if (!(psi[i] >= r)) psi[i] = r;
        }
}

__global__ void __launch_bounds__(RB) k_cold_psi(int64_t n, const double *__restrict__ nu, double kappa,
                                                double *__restrict__ psi) {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB)
        psi[i] = kappa * pow(3.0 * nu[i] / (4.0 * 3.141592653589793), 2.0 / 3.0);
}

template <class T>
int dalloc(T **p, size_t *cap, size_t n) {
    if (*p && *cap >= n) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    NCK(cudaMalloc((void **)p, std::max<size_t>(n, 16) * sizeof(T)));
    *cap = n;
    return 0;
}

struct NewtonWS {
    double *g = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *Ap = nullptr;
    double *diag = nullptr, *hval = nullptr, *farea = nullptr, *vol = nullptr, *ksur = nullptr;
    double *psi_t = nullptr, *vol_t = nullptr, *ksur_t = nullptr, *farea_t = nullptr;
    int *hcnt = nullptr, *hcol = nullptr, *fcount = nullptr, *ftag = nullptr;
    int *fcount_t = nullptr, *ftag_t = nullptr;
    double *cent = nullptr, *cent_t = nullptr;
    size_t ccap[2] = {0, 0};
    double *part = nullptr, *sc = nullptr, *red = nullptr;
    int *ic = nullptr;
    int64_t *flags = nullptr;
    size_t c[24] = {0};
};
NewtonWS g_ws;

int ws_alloc(int64_t n, int smf) {
    NewtonWS &w = g_ws;
    size_t N = n, E = (size_t)n * smf;
    int rc = 0;
    rc |= dalloc(&w.g, &w.c[0], N); rc |= dalloc(&w.x, &w.c[1], N); rc |= dalloc(&w.r, &w.c[2], N);
    rc |= dalloc(&w.z, &w.c[3], N); rc |= dalloc(&w.p, &w.c[4], N); rc |= dalloc(&w.Ap, &w.c[5], N);
    rc |= dalloc(&w.diag, &w.c[6], N); rc |= dalloc(&w.hval, &w.c[7], E); rc |= dalloc(&w.farea, &w.c[8], E);
    rc |= dalloc(&w.vol, &w.c[9], N); rc |= dalloc(&w.ksur, &w.c[10], N); rc |= dalloc(&w.psi_t, &w.c[11], N);
    rc |= dalloc(&w.vol_t, &w.c[12], N); rc |= dalloc(&w.ksur_t, &w.c[13], N);
    rc |= dalloc(&w.farea_t, &w.c[14], E); rc |= dalloc(&w.hcnt, &w.c[15], N);
    rc |= dalloc(&w.hcol, &w.c[16], E); rc |= dalloc(&w.fcount, &w.c[17], N); rc |= dalloc(&w.ftag, &w.c[18], E);
    rc |= dalloc(&w.fcount_t, &w.c[19], N); rc |= dalloc(&w.ftag_t, &w.c[20], E);
    rc |= dalloc(&w.part, &w.c[21], 4 * NPART); rc |= dalloc(&w.sc, &w.c[22], 16);
    rc |= dalloc(&w.red, &w.c[23], 16);
    rc |= dalloc(&w.cent, &w.ccap[0], 3 * N); rc |= dalloc(&w.cent_t, &w.ccap[1], 3 * N);
    if (!w.ic) NCK(cudaMalloc(&w.ic, 4 * sizeof(int)));
    if (!w.flags) NCK(cudaMalloc(&w.flags, sizeof(int64_t)));
    return rc;
}

int nblocks(int64_t n) { return (int)std::min<int64_t>(NPART, std::max<int64_t>(1, (n + RB - 1) / RB)); }

int rescue_nearest(pf_ctx *ctx, int64_t n, const double *pts, const double *vol, double *psi, cudaStream_t st) {
    int *list = nullptr, *cnt = nullptr;
    double *q = nullptr;
    int64_t *nn = nullptr;
    NCK(cudaMallocAsync((void **)&cnt, sizeof(int), st));
    NCK(cudaMemsetAsync(cnt, 0, sizeof(int), st));
    NCK(cudaMallocAsync((void **)&list, n * sizeof(int), st));
    NCK(cudaMallocAsync((void **)&q, 3 * n * sizeof(double), st));
    pf_internal_launches_add(1);
    k_empty_list<<<nblocks(n), RB, 0, st>>>(n, vol, pts, list, q, cnt);
    int m = 0;
    NCK(cudaMemcpyAsync(&m, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    NCK(cudaStreamSynchronize(st));
    int rc = 0;
    if (m > 0) {
        NCK(cudaMallocAsync((void **)&nn, 2 * (size_t)m * sizeof(int64_t), st));
        if (pf_knn(ctx, n, pts, m, q, 2, nn, 0, st) < 0) rc = -1;  // the solve's grid
        if (!rc) {
            pf_internal_launches_add(1);
            k_rescue_nn<<<nblocks(m), RB, 0, st>>>(m, list, nn, psi);
        }
        NCK(cudaFreeAsync(nn, st));
    }
    NCK(cudaFreeAsync(q, st));
    NCK(cudaFreeAsync(list, st));
    NCK(cudaFreeAsync(cnt, st));
    return rc;
}

// (worst, min vol, min nu) of the current evaluation
int grad_stats(int64_t n, const double *nu, const double *vol, double *g, double *out_host,
               cudaStream_t st) {
    int nb = nblocks(n);
    pf_internal_launches_add(2);
    k_grad<<<nb, RB, 0, st>>>(n, nu, vol, g, g_ws.part);
    k_grad_fin<<<1, 1024, 0, st>>>(g_ws.part, nb, g_ws.red);
    NCK(cudaMemcpyAsync(out_host, g_ws.red, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    NCK(cudaStreamSynchronize(st));
    return 0;
}

}  // namespace

extern "C" {

int pf_newton_gradient(int64_t n, const double *nu, const double *vol, double *g, double *stats_host,
                       void *stream) {
    if (ws_alloc(n, 1)) return -1;
    return grad_stats(n, nu, vol, g, stats_host, (cudaStream_t)stream);
}

int pf_newton_hessian(int64_t n, int smf, const double *pts, const double *psi, const int32_t *fcount,
                      const int32_t *ftag, const double *farea, const double *ksur, double tau_psi,
                      int32_t *hcnt, int32_t *hcol, double *hval, double *diag, void *stream) {
    pf_internal_launches_add(1);
    k_hessian<<<nblocks(n), RB, 0, (cudaStream_t)stream>>>(n, smf, pts, psi, fcount, ftag, farea, ksur,
                                                            tau_psi, hcnt, hcol, hval, diag);
    NCK(cudaGetLastError());
    return 0;
}

// Jacobi-PCG on the ELL Hessian; returns the iteration count (>= 0).  The
// matrix is repacked as SELL-32 (k_sell_pack) for the iterations, which run
// in one cooperative kernel (k_pcg_sell); one host read at the end.
int pf_pcg(int64_t n, int smf, const int32_t *hcnt, const int32_t *hcol, const double *hval,
           const double *diag, const double *b, double *x, double rtol, int max_iter, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (ws_alloc(n, smf)) return -1;
    NewtonWS &w = g_ws;
    if (n <= 0) return 0;
    static int coop_blocks = 0;
    if (!coop_blocks) {
        int dev = 0, nsm = 0, per = 0;
        NCK(cudaGetDevice(&dev));
        NCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        NCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_sell, CG_T, 0));
        coop_blocks = nsm * std::max(1, std::min(per, 4));
    }
    const int64_t ns = (n + SELL_C - 1) / SELL_C;
    static int *scol = nullptr, *swid = nullptr;
    static double *sval = nullptr, *pb = nullptr;
    static size_t scol_c = 0, sval_c = 0, swid_c = 0, pb_c = 0;
    const size_t E = (size_t)ns * SELL_C * smf;
    if (dalloc(&scol, &scol_c, E) || dalloc(&sval, &sval_c, E) || dalloc(&swid, &swid_c, (size_t)ns) ||
        dalloc(&pb, &pb_c, (size_t)n))
        return -1;
    pf_internal_launches_add(1);
    k_sell_pack<<<(int)std::min<int64_t>((ns * 32 + RB - 1) / RB, 148 * 32), RB, 0, st>>>(n, smf, hcnt, hcol, hval,
                                                                                         scol, sval, swid);
    NCK(cudaGetLastError());
    int G = (int)std::min<int64_t>(coop_blocks, ns);
    if (G > NPART) G = NPART;
    int64_t nn = n;
    int smf_ = smf, mi = max_iter;
    double rt = rtol;
    double *part = w.part;  // 4 * NPART doubles
    void *args[] = {&nn, &smf_, (void *)&scol, (void *)&sval, (void *)&swid, (void *)&diag, (void *)&b, &x,
                    &w.r, &w.z, &w.p, &pb, &w.Ap, &part, &rt, &mi, &w.ic};
    pf_internal_launches_add(1);
    NCK(cudaLaunchCooperativeKernel((const void *)k_pcg_sell, G, CG_T, args, 0, st));
    int it = 0;
    NCK(cudaMemcpyAsync(&it, w.ic, sizeof(int), cudaMemcpyDeviceToHost, st));
    NCK(cudaStreamSynchronize(st));
    return it;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// full solve
// ---------------------------------------------------------------------------
extern "C" int pf_newton_solve(pf_ctx *ctx, int64_t n, const double *pts, const double *nu, double *psi,
                               int cold_start, double eps_vol, int max_newton, int smf, double tau_psi,
                               int ball_aware, pf_newton_stats *stats, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    pf_newton_stats S;
    memset(&S, 0, sizeof S);
    if (n <= 0) { if (stats) *stats = S; return 0; }
    if (ws_alloc(n, smf)) return -1;
    NewtonWS &w = g_ws;
    if (pf_grid_build(ctx, n, pts, cold_start ? nullptr : psi, 0.0, stream)) return -1;
    auto evaluate = [&](const double *ps, double *vol, double *ksur, int *fcount, int *ftag,
                        double *farea, double *cent) -> int {
        S.evaluations++;
        return pf_evaluate_lean(ctx, n, pts, ps, ball_aware, smf, vol, ksur, fcount, ftag, farea, cent,
                                w.flags, stream);
    };
    double stats3[3];
    // init_weights: cold kappa doubling until no cell is empty
    if (cold_start) {
        double kappa = 1.0;
        for (;;) {
            pf_internal_launches_add(1);
            k_cold_psi<<<nblocks(n), RB, 0, st>>>(n, nu, kappa, psi);
            if (evaluate(psi, w.vol, w.ksur, w.fcount, w.ftag, w.farea, w.cent)) return -1;
            if (grad_stats(n, nu, w.vol, w.g, stats3, st)) return -1;
            if (stats3[1] > 0.0) break;
            kappa *= 2.0;
            S.init_doublings++;
            if (kappa > 1024.0) { S.status = 3; if (stats) *stats = S; return 0; }  // InitFailure
        }
    } else {
        if (evaluate(psi, w.vol, w.ksur, w.fcount, w.ftag, w.farea, w.cent)) return -1;
        if (grad_stats(n, nu, w.vol, w.g, stats3, st)) return -1;
        // warm start with per-cell rescue (SPEC.md init_weights).  First an
        // empty cell takes the weight of its nearest site (a near-coincident
        // pair then splits at its midpoint instead of ping-ponging through the
        // doubling below), then psi_i <- max(psi_i, kappa (3 nu_i / 4 pi)^(2/3)).
        if (!(stats3[1] > 0.0)) {
            if (rescue_nearest(ctx, n, pts, w.vol, psi, st)) return -1;
            S.init_doublings++;
            if (evaluate(psi, w.vol, w.ksur, w.fcount, w.ftag, w.farea, w.cent)) return -1;
            if (grad_stats(n, nu, w.vol, w.g, stats3, st)) return -1;
        }
        double kappa = 1.0;
        while (!(stats3[1] > 0.0)) {
            if (kappa > 1024.0) { S.status = 3; if (stats) *stats = S; return 0; }  // InitFailure
            pf_internal_launches_add(1);
            k_rescue<<<nblocks(n), RB, 0, st>>>(n, nu, w.vol, kappa, psi);
            S.init_doublings++;
            if (evaluate(psi, w.vol, w.ksur, w.fcount, w.ftag, w.farea, w.cent)) return -1;
            if (grad_stats(n, nu, w.vol, w.g, stats3, st)) return -1;
            kappa *= 2.0;
        }
    }
    const double floor_v = 0.5 * std::min(stats3[2], stats3[1]);
    const bool verbose = getenv("PF_NEWTON_VERBOSE") != nullptr;
    if (verbose)
        fprintf(stderr, "[pf_newton] n=%lld init worst=%.6e minvol=%.6e minnu=%.6e floor=%.6e\n",
                (long long)n, stats3[0], stats3[1], stats3[2], floor_v);
    S.worst_initial = stats3[0];
    double worst = stats3[0];
    for (int it = 0; it < max_newton; it++) {
        if (worst <= eps_vol) break;
        // H from the current evaluation, solve H u = g
        if (pf_newton_hessian(n, smf, pts, psi, w.fcount, w.ftag, w.farea, w.ksur, tau_psi, w.hcnt, w.hcol,
                              w.hval, w.diag, stream))
            return -1;
        double rtol = worst < 10.0 * eps_vol ? 1e-4 : 1e-3;
        int cg = pf_pcg(n, smf, w.hcnt, w.hcol, w.hval, w.diag, w.g, w.x, rtol, 10000, stream);
        if (cg < 0) return -1;
        S.cg_iterations += cg;
        // KMT damping
        double alpha = 1.0;
        bool accepted = false;
        while (alpha >= 0x1p-20) {
            pf_internal_launches_add(1);
            k_axpy_to<<<nblocks(n), RB, 0, st>>>(n, psi, alpha, w.x, w.psi_t);
            if (evaluate(w.psi_t, w.vol_t, w.ksur_t, w.fcount_t, w.ftag_t, w.farea_t, w.cent_t)) return -1;
            if (grad_stats(n, nu, w.vol_t, w.g, stats3, st)) return -1;
            if (stats3[1] >= floor_v) { accepted = true; break; }
            alpha *= 0.5;
            S.damping_halvings++;
        }
        if (!accepted) { S.status = 2; break; }  // DampingStall
        NCK(cudaMemcpyAsync(psi, w.psi_t, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        std::swap(w.vol, w.vol_t);
        std::swap(w.ksur, w.ksur_t);
        std::swap(w.fcount, w.fcount_t);
        std::swap(w.ftag, w.ftag_t);
        std::swap(w.farea, w.farea_t);
        std::swap(w.cent, w.cent_t);
        std::swap(w.ccap[0], w.ccap[1]);
        std::swap(w.c[9], w.c[12]);
        std::swap(w.c[10], w.c[13]);
        std::swap(w.c[17], w.c[19]);
        std::swap(w.c[18], w.c[20]);
        std::swap(w.c[8], w.c[14]);
        S.iterations++;
        S.last_alpha = alpha;
        worst = stats3[0];
        if (verbose)
            fprintf(stderr, "[pf_newton] it=%d worst=%.6e minvol=%.6e alpha=%g cg=%d\n", it + 1, worst,
                    stats3[1], alpha, cg);
    }
    S.worst_final = worst;
    if (S.status == 0 && worst > eps_vol) S.status = 1;  // not converged within max_newton
    int64_t fl = 0;
    NCK(cudaMemcpyAsync(&fl, w.flags, sizeof fl, cudaMemcpyDeviceToHost, st));
    NCK(cudaStreamSynchronize(st));
    S.flags = fl;
    if (stats) *stats = S;
    return 0;
}

extern "C" int pf_newton_last_state(double *vol, double *ksur, int32_t *fcount, int32_t *ftag, double *farea,
                                    int64_t n, int smf, void *stream) {
    return pf_newton_last_state_ex(vol, ksur, fcount, ftag, farea, nullptr, n, smf, stream);
}

extern "C" int pf_newton_last_state_ex(double *vol, double *ksur, int32_t *fcount, int32_t *ftag,
                                       double *farea, double *cent, int64_t n, int smf, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    NewtonWS &w = g_ws;
    if (cent) NCK(cudaMemcpyAsync(cent, w.cent, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (vol) NCK(cudaMemcpyAsync(vol, w.vol, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (ksur) NCK(cudaMemcpyAsync(ksur, w.ksur, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (fcount) NCK(cudaMemcpyAsync(fcount, w.fcount, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    if (ftag) NCK(cudaMemcpyAsync(ftag, w.ftag, (size_t)n * smf * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    if (farea) NCK(cudaMemcpyAsync(farea, w.farea, (size_t)n * smf * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return 0;
}

// ---------------------------------------------------------------------------
// fluid step pieces
// ---------------------------------------------------------------------------
namespace {
// x += dt v, then reflect into the box [lo+tau, hi-tau]
__global__ void __launch_bounds__(RB) k_advect(int64_t n, double *__restrict__ x, double *__restrict__ v,
                                              double dt, double lo0, double lo1, double lo2, double hi0,
                                              double hi1, double hi2, double tau) {
    const double lo[3] = {lo0 + tau, lo1 + tau, lo2 + tau}, hi[3] = {hi0 - tau, hi1 - tau, hi2 - tau};
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double p = x[3 * i + a] + dt * v[3 * i + a];
            if (p < lo[a]) { p = lo[a] + (lo[a] - p); v[3 * i + a] = -v[3 * i + a]; }
            if (p > hi[a]) { p = hi[a] - (p - hi[a]); v[3 * i + a] = -v[3 * i + a]; }
            p = p < lo[a] ? lo[a] : (p > hi[a] ? hi[a] : p);
            x[3 * i + a] = p;
        }
    }
}
// Gallouet-Merigot spring: pressure F_p = m (c - x) / eps^2,
// gravity F_g = m g; v += dt/m (F_p + F_g) = dt ((c - x)/eps^2 + g), m = rho nu.
// The spring is mass-proportional as in the scheme the paper follows; it is
// the form for which SPEC.md's stability guideline dt <= eps holds.
// spring coefficient of the pressure force F_p = k (c - x) / eps^2:
// PF_SPRING_SPEC (1): k = 1, SPEC.md:357-361 pressure_force as printed;
// PF_SPRING_GM (0): k = m, the Gallouet-Merigot acceleration (c - x)/eps^2
// the paper follows
__device__ __forceinline__ double spring_coef(int spring, double m) { return spring == 1 ? 1.0 : m; }

// F_p of every particle (SPEC.md pressure_force)
__global__ void __launch_bounds__(RB) k_pressure(int64_t n, const double *__restrict__ x,
                                                const double *__restrict__ c, const double *__restrict__ nu,
                                                const double *__restrict__ rho, double inv_eps2, int spring,
                                                double *__restrict__ F) {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        const double ks = spring_coef(spring, rho[i] * nu[i]) * inv_eps2;
        for (int a = 0; a < 3; a++) F[3 * i + a] = ks * (c[3 * i + a] - x[3 * i + a]);
    }
}

__global__ void __launch_bounds__(RB) k_forces(int64_t n, const double *__restrict__ x,
                                              const double *__restrict__ c, const double *__restrict__ nu,
                                              const double *__restrict__ rho, double *__restrict__ v,
                                              double dt, double inv_eps2, double g0, double g1, double g2,
                                              int spring) {
    const double g[3] = {g0, g1, g2};
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        const double m = rho[i] * nu[i];
        const double ks = spring_coef(spring, m) * inv_eps2;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double f = ks * (c[3 * i + a] - x[3 * i + a]) + m * g[a];
            v[3 * i + a] += dt * f / m;
        }
    }
}
// ---- full fluid forces ----
// P1 Laplacian weights from the restricted facets: w_ij = |B_ij| / (2 |p_j - p_i|)
// (PAPER Eq. 3); boundary weights w_iOmega = mu_b |B_iOmega| / (2 d(p_i, Omega) |V_i|)
// (SPEC laplacian_weights, as printed).  One row per cell:
//   A = m/dt I + mu L (+ boundary weights on the diagonal: zero wall velocity)
//   rhs_a = m/dt v_a + F_p + F_g + F_t,
//   F_t = gamma (sum_j w_ij (x_j - x_i) + sum_b affinity w^g_b (g_b - x_i)),
// g_b = orthogonal projection of x_i on the wall plane, moved |V_i|^(1/3) to the
// fluid side (SPEC surface_tension_force), w^g_b = |B_b| / (2 |g_b - x_i|).
__global__ void __launch_bounds__(RB) k_fluid_system(
    int64_t n, int smf, const double *__restrict__ x, const double *__restrict__ cent,
    const double *__restrict__ vol, const int *__restrict__ fcount, const int *__restrict__ ftag,
    const double *__restrict__ farea, const double *__restrict__ nu, const double *__restrict__ rho,
    const double *__restrict__ v, double dt, double inv_eps2, double g0, double g1, double g2, double mu,
    double mu_b, double gamma, double affinity, const double *__restrict__ dplanes, int ndom, int spring,
    int *__restrict__ hcnt, int *__restrict__ hcol, double *__restrict__ hval, double *__restrict__ diag,
    double *__restrict__ rhs) {
    const double g[3] = {g0, g1, g2};
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        const double m = rho[i] * nu[i];
        const double px = x[3 * i], py = x[3 * i + 1], pz = x[3 * i + 2];
        int c = fcount[i];
        if (c > smf) c = smf;
        double d = m / dt, ft[3] = {0.0, 0.0, 0.0};
        int k = 0;
        const double vi = vol[i] > 0.0 ? vol[i] : nu[i];
        for (int s = 0; s < c; s++) {
            const int64_t j = ftag[i * smf + s];
            const double A = farea[i * smf + s];
            if (j >= 0) {
                const double dx = x[3 * j] - px, dy = x[3 * j + 1] - py, dz = x[3 * j + 2] - pz;
                const double w = 0.5 * A / sqrt(dx * dx + dy * dy + dz * dz);
                hcol[i * smf + k] = (int)j;
                hval[i * smf + k] = -mu * w;
                d += mu * w;
                k++;
                ft[0] += w * dx; ft[1] += w * dy; ft[2] += w * dz;
            } else {
                const int b = (int)(-j - 1);
                if (b >= ndom) continue;
                const double nx = dplanes[4 * b], ny = dplanes[4 * b + 1], nz = dplanes[4 * b + 2];
                const double dist = dplanes[4 * b + 3] - (nx * px + ny * py + nz * pz);  // >= 0 inside
                const double dd = dist > 1e-300 ? dist : 1e-300;
                d += mu_b * 0.5 * A / (dd * vi);
                // ghost: projection on the wall, |V_i|^(1/3) back toward the fluid
                const double off = dist - cbrt(vi);
                const double gx = off * nx, gy = off * ny, gz = off * nz;  // g - x
                const double gl = sqrt(gx * gx + gy * gy + gz * gz);
                if (gl > 0.0) {
                    const double wg = affinity * 0.5 * A / gl;
                    ft[0] += wg * gx; ft[1] += wg * gy; ft[2] += wg * gz;
                }
            }
        }
        hcnt[i] = k;
        diag[i] = d;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const double fp = spring_coef(spring, m) * (cent[3 * i + a] - x[3 * i + a]) * inv_eps2;
            rhs[a * n + i] = m / dt * v[3 * i + a] + fp + m * g[a] + gamma * ft[a];
        }
    }
}
__global__ void __launch_bounds__(RB) k_scatter_v(int64_t n, const double *__restrict__ sol, int a,
                                                 double *__restrict__ v) {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB)
        v[3 * i + a] = sol[i];
}
}  // namespace

extern "C" int pf_fluid_advect(int64_t n, double *x, double *v, double dt, const double *lo_host,
                               const double *hi_host, double tau, void *stream) {
    pf_internal_launches_add(1);
    k_advect<<<nblocks(n), RB, 0, (cudaStream_t)stream>>>(n, x, v, dt, lo_host[0], lo_host[1], lo_host[2],
                                                          hi_host[0], hi_host[1], hi_host[2], tau);
    NCK(cudaGetLastError());
    return 0;
}

extern "C" int pf_fluid_forces(int64_t n, const double *x, const double *cent, const double *nu,
                               const double *rho, double *v, double dt, double eps, const double *g_host,
                               int spring, void *stream) {
    pf_internal_launches_add(1);
    k_forces<<<nblocks(n), RB, 0, (cudaStream_t)stream>>>(n, x, cent, nu, rho, v, dt, 1.0 / (eps * eps),
                                                          g_host[0], g_host[1], g_host[2], spring);
    NCK(cudaGetLastError());
    return 0;
}

extern "C" int pf_pressure_force(int64_t n, const double *x, const double *cent, const double *nu,
                                 const double *rho, double eps, int spring, double *F, void *stream) {
    pf_internal_launches_add(1);
    k_pressure<<<nblocks(n), RB, 0, (cudaStream_t)stream>>>(n, x, cent, nu, rho, 1.0 / (eps * eps), spring, F);
    NCK(cudaGetLastError());
    return 0;
}

// implicit velocity update with viscosity, boundary friction and surface
// tension (SPEC.md fluid_sim assemble_viscosity_system / surface_tension_force):
// three Jacobi-PCG solves (one per axis) on (m/dt I + mu L); returns the total
// CG iteration count.  Scratch: hcnt i32[n], hcol i32[n,smf], hval f64[n,smf],
// diag f64[n], rhs f64[3n], sol f64[n].
extern "C" int pf_fluid_forces_implicit(int64_t n, int smf, const double *x, const double *cent,
                                        const double *vol, const int32_t *fcount, const int32_t *ftag,
                                        const double *farea, const double *nu, const double *rho, double *v,
                                        double dt, double eps, const double *g_host, double mu, double mu_b,
                                        double gamma, double affinity, const double *dplanes, int ndom,
                                        int spring, int32_t *hcnt, int32_t *hcol, double *hval, double *diag, double *rhs,
                                        double *sol, double rtol, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    pf_internal_launches_add(1);
    k_fluid_system<<<nblocks(n), RB, 0, st>>>(n, smf, x, cent, vol, fcount, ftag, farea, nu, rho, v, dt,
                                               1.0 / (eps * eps), g_host[0], g_host[1], g_host[2], mu, mu_b,
                                               gamma, affinity, dplanes, ndom, spring, hcnt, hcol, hval, diag, rhs);
    NCK(cudaGetLastError());
    int total = 0;
    for (int a = 0; a < 3; a++) {
        int it = pf_pcg(n, smf, hcnt, hcol, hval, diag, rhs + a * n, sol, rtol, 10000, stream);
        if (it < 0) return -1;
        total += it;
        pf_internal_launches_add(1);
        k_scatter_v<<<nblocks(n), RB, 0, st>>>(n, sol, a, v);
        NCK(cudaGetLastError());
    }
    return total;
}
