// pf_runtime.cu -- device runtime of the partial-OT hot path for sm_100a:
// grid build (counting sort), weight reductions, the two-tier warp-per-cell
// evaluation kernels, batched kNN, and the C ABI of include/potflow_b200.h.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <array>
#include <vector>

#include "pf_tiers.cuh"
#include "../../include/potflow_b200.h"

using namespace pf;

// the cell kernels read their CellIn / CellOut parameters in place (param
// space) instead of from a local-memory copy (C4: 103.4 -> 100.4 ms)
#define PF_KPARAM const __grid_constant__

// the block-synchronous evaluation kernel lives in pf_eval.cu
int pf_internal_eval_sync_attr();
int pf_internal_eval_sync(const CellIn &in, const CellOut &out, int count, const Poly<FastCaps> *gpoly,
                          const uint8_t *stage, int *retry_list, int *counters, unsigned long long *err, int nsm,
                          cudaStream_t st);

namespace {

thread_local std::string g_err;
unsigned long long g_launches = 0;  // kernels launched by this library (bench evidence)

int set_err(const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return -1;
}

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t _e = (x);                                                       \
        if (_e != cudaSuccess)                                                      \
            return set_err("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(_e)); \
    } while (0)

inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

template <class T>
int ensure(T **p, size_t *cap, size_t count) {
    if (*cap >= count && *p) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    size_t c = count < 16 ? 16 : count + count / 4;
    CK(cudaMalloc((void **)p, c * sizeof(T)));
    *cap = c;
    return 0;
}

}  // namespace

struct pf_ctx {
    int device = 0;
    int nsm = 148;
    // domain (device copies, reference layout with int32 indices)
    double *dv = nullptr, *dp = nullptr;
    int *dt = nullptr, *dlp = nullptr, *dlv = nullptr;
    int dnv = 0, dnf = 0, dnl = 0;
    double tol = 0.0;
    double dlo[3] = {0, 0, 0}, dhi[3] = {1, 1, 1};
    double dvol = 1.0;
    bool has_domain = false;
    // grid
    double *sx = nullptr, *sy = nullptr, *sz = nullptr;
    size_t sx_cap = 0, sy_cap = 0, sz_cap = 0;
    int *sid = nullptr, *bid = nullptr;
    size_t sid_cap = 0, bid_cap = 0;
    int *bcount = nullptr, *bstart = nullptr;
    size_t bcount_cap = 0, bstart_cap = 0;
    double *smax = nullptr;  // per super-bucket max weight (build_cell's local slack)
    size_t smax_cap = 0;
    // a caller evaluating one (grid, psi) in several cell subsets (the host
    // drop-in's index ranges) computes the weight range and the super-bucket
    // maxima once: pf_internal_keep_weights
    bool keep_w = false, have_dpsi = false, have_smax = false;
    // full mode: the heaviest sites by one descending radix sort of (psi, index)
    double *hv_keys = nullptr;  // [n + 1]: sorted weights, then -1e300
    int *hv_iota = nullptr, *hv_vals = nullptr;
    size_t hv_cap = 0;
    void *hv_tmp = nullptr;
    size_t hv_tmp_cap = 0;
    int *csr_cnt = nullptr, *csr_off = nullptr;  // pf_facets_csr scratch
    size_t csr_cnt_cap = 0, csr_off_cap = 0;
    double *cslack = nullptr;  // per-site weight slack
    size_t cslack_cap = 0;
    int *scan_tmp = nullptr;
    size_t scan_tmp_cap = 0;
    int64_t grid_n = -1;
    const double *grid_pts = nullptr;
    int gn[3] = {1, 1, 1};
    double glo[3] = {0, 0, 0}, gh[3] = {1, 1, 1}, gih[3] = {1, 1, 1};
    // reductions / scalars (device): [0] dpsi, [1..2] ordered min/max, [3] sum
    double *dscal = nullptr;
    unsigned long long *mm = nullptr;
    // evaluation scratch
    int *retry_list = nullptr;
    size_t retry_cap = 0;
    int *retry_list2 = nullptr;  // the mid tier's overflow
    size_t retry2_cap = 0;
    bool mid = true;
    int *counters = nullptr;  // [0] retry count
    unsigned long long *err = nullptr;
    int *census = nullptr;
    size_t census_cap = 0;
    WS<ExactCaps> *exact_ws = nullptr;
    int exact_warps = 0;
    Poly<FastCaps> *gpoly = nullptr;
    size_t gpoly_cap = 0;
    uint8_t *stage = nullptr;
    size_t stage_cap = 0;
    int split = 1;  // split build/evaluate kernels (PF_FUSED=1 selects the fused kernel)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool ev_valid = false;
    // per-stage timing (cmd_bench): build / evaluation event triples of every
    // evaluation since pf_stage_timing(ctx, 1)
    bool stage_on = false;
    std::vector<std::array<cudaEvent_t, 3>> stage_ev;
    size_t stage_n = 0;
    int fast_blocks = 0, build_blocks = 0, eval_blocks = 0, eval_sync = 1;
    bool attr_set = false;
    // parity mode: restrict the facets exactly as the reference does, including
    // its spurious-entry and long-arc outcomes; 0 = robust default
    int strict = 0;
    // grid build: bucket size cached across calls (the cell results do not depend
    // on the bucket layout), refreshed from an asynchronous read of the mean ball
    // radius; bucket counts known to be zero (the scatter consumes them)
    double h_cache = 0.0;
    int64_t h_cache_n = -1;
    double *h_pinned = nullptr;
    cudaEvent_t h_ev = nullptr;
    bool h_pending = false;
    int64_t bcount_zero = -1;  // bcount[0..bcount_zero] is all zeros
    int grid_coop_blocks = 0;
    int *grid_part = nullptr;
    // evaluation order sorted by polytope size (PF_EVAL_SORT, default on)
    int eval_sort = -1;
    uint8_t *ekey = nullptr, *ekey2 = nullptr;
    int *eidx = nullptr, *eidx2 = nullptr;
    size_t ekey_cap = 0, ekey2_cap = 0, eidx_cap = 0, eidx2_cap = 0;
    void *esort_tmp = nullptr;
    size_t esort_cap = 0;
};

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
namespace {

constexpr int FAST_WARPS = 4;
constexpr int EXACT_WARPS = 2;
constexpr int MID_WARPS = 4;

__device__ __forceinline__ unsigned long long ord_bits(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long o) {
    unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    return __longlong_as_double((long long)b);
}

__global__ void k_minmax(const double *__restrict__ v, int64_t n, unsigned long long *mm) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x = v[i];
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
    }
    for (int m = 16; m > 0; m >>= 1) {
        double a = __shfl_xor_sync(0xffffffffu, lo, m), b = __shfl_xor_sync(0xffffffffu, hi, m);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], ord_bits(lo));
        atomicMax(&mm[1], ord_bits(hi));
    }
}

// dpsi = max(hi - lo, 0) (laguerre.py:142-145); empty -> 0
__global__ void k_dpsi_finish(const unsigned long long *mm, int64_t n, double *dscal) {
    double lo = ord_val(mm[0]), hi = ord_val(mm[1]);
    double d = n > 0 ? hi - lo : 0.0;
    dscal[0] = d > 0.0 ? d : 0.0;
    dscal[1] = lo;
    dscal[2] = hi;
}

__global__ void k_sum_sqrt(const double *__restrict__ v, int64_t n, double *out) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += v[i] > 0.0 ? sqrt(v[i]) : 0.0;
    for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void k_grid_bucket(const double *__restrict__ pts, int64_t n, double lo0, double lo1,
                              double lo2, double ih0, double ih1, double ih2, int g0, int g1, int g2,
                              int *__restrict__ bid, int *__restrict__ bcount) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int a = bucket_coord(pts[3 * i], lo0, ih0, g0);
        int b = bucket_coord(pts[3 * i + 1], lo1, ih1, g1);
        int c = bucket_coord(pts[3 * i + 2], lo2, ih2, g2);
        int l = (a * g1 + b) * g2 + c;
        bid[i] = l;
        atomicAdd(&bcount[l], 1);
    }
}

// exclusive scan, block-local (1024 threads x 4 items); block sums to `sums`
constexpr int SCAN_T = 1024, SCAN_I = 4, SCAN_B = SCAN_T * SCAN_I;

__device__ __forceinline__ int block_excl_scan(int v, int *total) {
    __shared__ int wsum[32];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        wsum[lane] = s;
    }
    __syncthreads();
    int base = w > 0 ? wsum[w - 1] : 0;
    *total = wsum[31];
    __syncthreads();
    return base + x - v;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_blocks(const int *__restrict__ in, int *__restrict__ out,
                                                        int64_t n, int *__restrict__ sums) {
    int64_t b0 = (int64_t)blockIdx.x * SCAN_B + (int64_t)threadIdx.x * SCAN_I;
    int v[SCAN_I], s = 0;
    for (int k = 0; k < SCAN_I; k++) {
        v[k] = b0 + k < n ? in[b0 + k] : 0;
        s += v[k];
    }
    int tot;
    int off = block_excl_scan(s, &tot);
    for (int k = 0; k < SCAN_I; k++) {
        if (b0 + k < n) out[b0 + k] = off;
        off += v[k];
    }
    if (threadIdx.x == 0 && sums) sums[blockIdx.x] = tot;
}

__global__ void k_scan_add(int *__restrict__ out, int64_t n, const int *__restrict__ sums) {
    int64_t b0 = (int64_t)blockIdx.x * SCAN_B;
    int add = sums[blockIdx.x];
    for (int64_t k = threadIdx.x; k < SCAN_B && b0 + k < n; k += blockDim.x) out[b0 + k] += add;
}

__global__ void k_grid_scatter(const int *__restrict__ bid, int64_t n, const int *__restrict__ bstart,
                               int *__restrict__ fill, int *__restrict__ sid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int l = bid[i];
        int s = bstart[l] + atomicAdd(&fill[l], 1);
        sid[s] = (int)i;
    }
}

// order each bucket by site index (== numpy's stable argsort) and lay out SoA
__global__ void k_grid_finish(int ncell, const int *__restrict__ bstart, int *__restrict__ sid,
                              const double *__restrict__ pts, double *__restrict__ sx,
                              double *__restrict__ sy, double *__restrict__ sz) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        int a = bstart[c], b = bstart[c + 1];
        for (int k = a + 1; k < b; k++) {
            int v = sid[k], j = k - 1;
            while (j >= a && sid[j] > v) { sid[j + 1] = sid[j]; j--; }
            sid[j + 1] = v;
        }
        for (int k = a; k < b; k++) {
            int i = sid[k];
            sx[k] = pts[3 * i];
            sy[k] = pts[3 * i + 1];
            sz[k] = pts[3 * i + 2];
        }
    }
}

__global__ void k_grid_export(const int *__restrict__ bstart, int ncell, const int *__restrict__ sid,
                              int64_t n, int64_t *__restrict__ bs64, int64_t *__restrict__ sid64) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = t; c <= ncell; c += st) bs64[c] = bstart[c];
    for (int64_t i = t; i < n; i += st) sid64[i] = sid[i];
}

// The whole counting sort as ONE cooperative kernel (four grid barriers):
//   1. bucket id of every site, histogram (shared counts start at zero)
//   2. exclusive scan of the counts: per-block chunk sums, every block adds the
//      sums of the blocks before it, then scans its chunk
//   3. scatter, the counts serving as decrementing cursors (they end at zero,
//      so the next build needs no memset)
//   4. per bucket (by its first slot: work ~ n, not ~ the bucket count): order
//      by site index (== numpy's stable argsort); then the SoA copy
constexpr int GRID_T = 1024;
__global__ void __launch_bounds__(GRID_T, 1) k_grid_coop(const double *__restrict__ pts, int64_t n, double lo0,
                                                       double lo1, double lo2, double ih0, double ih1, double ih2,
                                                       int g0, int g1, int g2, int64_t ncell, int *__restrict__ bid,
                                                       int *__restrict__ bcount, int *__restrict__ bstart,
                                                       int *__restrict__ sid, double *__restrict__ sx,
                                                       double *__restrict__ sy, double *__restrict__ sz,
                                                       int *__restrict__ part) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int sh[33];
    const int64_t T = (int64_t)gridDim.x * GRID_T, t0 = blockIdx.x * (int64_t)GRID_T + threadIdx.x;
    for (int64_t i = t0; i < n; i += T) {
        const int a = bucket_coord(pts[3 * i], lo0, ih0, g0);
        const int b = bucket_coord(pts[3 * i + 1], lo1, ih1, g1);
        const int c = bucket_coord(pts[3 * i + 2], lo2, ih2, g2);
        const int l = (a * g1 + b) * g2 + c;
        bid[i] = l;
        atomicAdd(&bcount[l], 1);
    }
    grid.sync();
    // chunk of this block over the ncell + 1 counts (bcount[ncell] == 0), in
    // tiles of GRID_T x 8 counts read as two int4 per thread (enough loads in
    // flight to stream the counts; the arrays carry 16 ints of padding)
    const int64_t m = ncell + 1, G = gridDim.x;
    const int64_t C8 = ((m + G - 1) / G + 7) & ~(int64_t)7;
    const int64_t c0 = C8 * blockIdx.x < m ? C8 * blockIdx.x : m, c1 = c0 + C8 < m ? c0 + C8 : m;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int TILE = GRID_T * 8;
    int loc = 0;
    for (int64_t base = c0; base < c1; base += TILE) {
        const int64_t k = base + 8 * (int64_t)threadIdx.x;
        if (k < c1) {
            const int4 u0 = *(const int4 *)(bcount + k), u1 = *(const int4 *)(bcount + k + 4);
            const int v[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
            for (int e = 0; e < 8; e++) loc += k + e < c1 ? v[e] : 0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, o);
    if (lane == 0) sh[w] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int k = 0; k < GRID_T / 32; k++) s += sh[k];
        part[blockIdx.x] = s;
    }
    grid.sync();
    // offset of this chunk: sum of the preceding blocks' chunk sums
    int off = 0;
    for (int k = threadIdx.x; k < blockIdx.x; k += GRID_T) off += __ldcg(part + k);
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
    __syncthreads();
    if (lane == 0) sh[w] = off;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int k = 0; k < GRID_T / 32; k++) s += sh[k];
        sh[32] = s;
    }
    __syncthreads();
    int run = sh[32];
    __syncthreads();
    for (int64_t base = c0; base < c1; base += TILE) {
        const int64_t k = base + 8 * (int64_t)threadIdx.x;
        int v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (k < c1) {
            const int4 u0 = *(const int4 *)(bcount + k), u1 = *(const int4 *)(bcount + k + 4);
            v[0] = u0.x; v[1] = u0.y; v[2] = u0.z; v[3] = u0.w; v[4] = u1.x; v[5] = u1.y; v[6] = u1.z; v[7] = u1.w;
#pragma unroll
            for (int e = 0; e < 8; e++) v[e] = k + e < c1 ? v[e] : 0;
        }
        int tsum = 0;
#pragma unroll
        for (int e = 0; e < 8; e++) { const int t = v[e]; v[e] = tsum; tsum += t; }
        int x = tsum;  // inclusive warp scan of the thread sums
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sh[w] = x;
        __syncthreads();
        if (w == 0) {
            int s2 = sh[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, s2, o);
                if (lane >= o) s2 += y;
            }
            sh[lane] = s2;
        }
        __syncthreads();
        const int tb = run + (w > 0 ? sh[w - 1] : 0) + x - tsum;
        if (k < c1) {
            if (k + 8 <= c1) {
                *(int4 *)(bstart + k) = make_int4(tb + v[0], tb + v[1], tb + v[2], tb + v[3]);
                *(int4 *)(bstart + k + 4) = make_int4(tb + v[4], tb + v[5], tb + v[6], tb + v[7]);
            } else {
#pragma unroll
                for (int e = 0; e < 8; e++)
                    if (k + e < c1) bstart[k + e] = tb + v[e];
            }
        }
        run += sh[31];
        __syncthreads();
    }
    grid.sync();
    // scatter, four sites per thread in flight
    for (int64_t i0 = t0; i0 < n; i0 += 4 * T) {
        int l[4], st[4];
#pragma unroll
        for (int u = 0; u < 4; u++) l[u] = i0 + u * T < n ? bid[i0 + u * T] : -1;
#pragma unroll
        for (int u = 0; u < 4; u++) st[u] = l[u] >= 0 ? bstart[l[u]] : 0;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (l[u] >= 0) sid[st[u] + atomicSub(&bcount[l[u]], 1) - 1] = (int)(i0 + u * T);
    }
    grid.sync();
    // order each bucket by site index (its first slot's thread; most buckets
    // hold one or two sites)
    for (int64_t k = t0; k < n; k += T) {
        const int l = bid[sid[k]];
        const int a = bstart[l];
        if (k != a) continue;
        const int b = bstart[l + 1];
        for (int q = a + 1; q < b; q++) {
            const int v = sid[q];
            int j = q - 1;
            while (j >= a && sid[j] > v) { sid[j + 1] = sid[j]; j--; }
            sid[j + 1] = v;
        }
    }
    grid.sync();
    // SoA copy of the positions in bucket order, four slots per thread in flight
    for (int64_t k0 = t0; k0 < n; k0 += 4 * T) {
        int i[4];
#pragma unroll
        for (int u = 0; u < 4; u++) i[u] = k0 + u * T < n ? sid[k0 + u * T] : -1;
        double px[4], py[4], pz[4];
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (i[u] >= 0) { px[u] = pts[3 * i[u]]; py[u] = pts[3 * i[u] + 1]; pz[u] = pts[3 * i[u] + 2]; }
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (i[u] >= 0) { sx[k0 + u * T] = px[u]; sy[k0 + u * T] = py[u]; sz[k0 + u * T] = pz[u]; }
    }
}

// cells of the fast tier: shared-memory workspace, one warp per cell, cells
// visited in bucket order (neighbouring warps share candidates through L1/L2)
__global__ void __launch_bounds__(FAST_WARPS * 32, 4)
    k_cells_fast(CellIn in, CellOut out, int count, int *__restrict__ retry_list,
                 int *__restrict__ counters, unsigned long long *__restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WS<FastCaps> *ws = (WS<FastCaps> *)(smem + (size_t)wid * sizeof(WS<FastCaps>));
    const int nw = gridDim.x * FAST_WARPS;
    int fl = 0;
    for (int t = blockIdx.x * FAST_WARPS + wid; t < count; t += nw) {
        const int i = in.cells ? in.cells[t] : in.g.sid[t];
        int r = run_cell(ws, in, out, i);
        if (r & FLAG_RETRY) {
            if (lane == 0) retry_list[atomicAdd(&counters[0], 1)] = i;
        } else {
            fl |= r & 7;
        }
    }
    if (lane == 0 && fl) atomicOr(err, (unsigned long long)fl);
}

// Split pipeline (fast tier).  One fused kernel touches ~130 KB of SASS per
// cell and stalls on instruction fetch; building in one kernel and
// evaluating in another halves the hot code each SM cycles through.  The
// finished polytope travels through global memory (Poly<FastCaps>, ~3 KB).
#ifndef PF_NO_TMA_LOAD
#define PF_NO_TMA_LOAD 0  // 1: the evaluation loads the polytope with lane loads instead of a bulk copy
#endif
#ifndef PF_BUILD_WARPS
#define PF_BUILD_WARPS 8
#endif
constexpr int BUILD_WARPS = PF_BUILD_WARPS;
#ifndef PF_DYN_BUILD
#define PF_DYN_BUILD 1
#endif
#ifndef PF_BUILD_MINB
#define PF_BUILD_MINB 3
#endif
// BW: BWSN<FastCaps> (timed: no census code) or BWS<FastCaps> (the census pass);
// HV: the general build (full mode, packed outputs) or the ball-aware evaluation build
template <class BW, bool HV>
__global__ void __launch_bounds__(BUILD_WARPS * 32, PF_BUILD_MINB)
    k_cells_build(PF_KPARAM CellIn in, PF_KPARAM CellOut out, int count, Poly<FastCaps> *__restrict__ gpoly,
                  uint8_t *__restrict__ stage, int *__restrict__ retry_list, int *__restrict__ counters,
                  unsigned long long *__restrict__ err, uint8_t *__restrict__ ekey, int *__restrict__ eidx) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    BW *ws = (BW *)(smem + (size_t)wid * sizeof(BW));
    int fl = 0;
    // cells handed out one at a time from a global counter (counters[2]): the
    // kernel ends when the last cell does, not when the unluckiest of the
    // warps' fixed shares does (PF_DYN_BUILD=0: grid stride)
    const int nw = gridDim.x * BUILD_WARPS;
    int t = PF_DYN_BUILD ? 0 : blockIdx.x * BUILD_WARPS + wid;
    for (;;) {
        if (PF_DYN_BUILD) {
            int tt = 0;
            if (lane == 0) tt = atomicAdd(&counters[2], 1);
            t = __shfl_sync(0xffffffffu, tt, 0);
        }
        if (t >= count) break;
        const int i = in.cells ? in.cells[t] : in.g.sid[t];
        int which = 0;
        poly_store_tma_wait();  // the previous cell's bulk store has read its buffer
        int r = cell_phase_build<BW, HV>(ws, in, out, i, &which);
        if (r < 0) {
            poly_store_tma(ws->P[which], gpoly + i);
            if (lane == 0) {
                stage[i] = 1;
                if (ekey) {  // evaluation order: larger polytopes first (sort key ascending)
                    const int nl = ws->P[which].nl;
                    ekey[t] = (uint8_t)(254 - (nl < 254 ? nl : 254));
                    eidx[t] = i;
                }
                if (BW::CEN && out.census16)
                    for (int k = 0; k < 16; k++) out.census16[(size_t)i * 16 + k] = ws->cen[k];
            }
        } else {
            if (lane == 0) {
                stage[i] = 0;
                if (ekey) { ekey[t] = 255; eidx[t] = i; }  // nothing to evaluate: last
            }
            if (r & FLAG_RETRY) {
                if (lane == 0) retry_list[atomicAdd(&counters[0], 1)] = i;
            } else {
                cell_finish(ws, out, i, r);
                fl |= r & 7;
            }
        }
        __syncwarp();
        if (!PF_DYN_BUILD) t += nw;
    }
    // drain the last bulk store: it still reads this warp's shared memory
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
    if (lane == 0 && fl) atomicOr(err, (unsigned long long)fl);
}

__global__ void __launch_bounds__(FAST_WARPS * 32, 4)
    k_cells_eval(CellIn in, CellOut out, int count, const Poly<FastCaps> *__restrict__ gpoly,
                 const uint8_t *__restrict__ stage, int *__restrict__ retry_list, int *__restrict__ counters,
                 unsigned long long *__restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    EWS<FastCaps> *ws = (EWS<FastCaps> *)(smem + (size_t)wid * sizeof(EWS<FastCaps>));
    const int nw = gridDim.x * FAST_WARPS;
    int fl = 0;
    for (int t = blockIdx.x * FAST_WARPS + wid; t < count; t += nw) {
        const int i = in.cells ? in.cells[t] : in.g.sid[t];
        if (stage[i] != 1) continue;
        poly_load(gpoly + i, ws->P[0]);
        if (lane == 0) {
            ws->oflow = 0;
            ws->strict = in.strict;
            ws->cen_on = out.census16 != nullptr;
            for (int k = 0; k < 16; k++) ws->cen[k] = out.census16 ? out.census16[(size_t)i * 16 + k] : 0;
        }
        __syncwarp();
        int r = cell_phase_eval(ws, in, out, i, 0);
        if (r & FLAG_RETRY) {
            if (lane == 0) retry_list[atomicAdd(&counters[0], 1)] = i;
        } else {
            cell_finish(ws, out, i, r);
            fl |= r & 7;
        }
        __syncwarp();
    }
    if (lane == 0 && fl) atomicOr(err, (unsigned long long)fl);
}

// Block-synchronous evaluation kernel: pf_eval.cu (its own translation unit,
// launched through pf_internal_eval_sync).

// cells that overflowed the fast tier: larger capacities, still in shared memory;
// their own overflow is queued for the exact tier
__global__ void __launch_bounds__(MID_WARPS * 32, 1)
    k_cells_mid(CellIn in, CellOut out, const int *__restrict__ list, int *__restrict__ counters,
                int *__restrict__ list2, unsigned long long *__restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WS<MidCaps> *ws = (WS<MidCaps> *)(smem + (size_t)wid * sizeof(WS<MidCaps>));
    const int count = counters[0];
    const int nw = gridDim.x * MID_WARPS;
    int fl = 0;
    for (int t = blockIdx.x * MID_WARPS + wid; t < count; t += nw) {
        const int i = list[t];
        int r = run_cell(ws, in, out, i);
        if (r & FLAG_RETRY) {
            if (lane == 0) list2[atomicAdd(&counters[1], 1)] = i;
        } else {
            fl |= r & 7;
        }
    }
    if (lane == 0 && fl) atomicOr(err, (unsigned long long)fl);
}

// cells that overflowed the mid tier, with the reference's capacities
__global__ void __launch_bounds__(EXACT_WARPS * 32)
    k_cells_exact(CellIn in, CellOut out, const int *__restrict__ list, const int *__restrict__ counters,
                  WS<ExactCaps> *__restrict__ wsbase, unsigned long long *__restrict__ err) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WS<ExactCaps> *ws = wsbase + (size_t)blockIdx.x * EXACT_WARPS + wid;
    const int count = counters[0];
    const int nw = gridDim.x * EXACT_WARPS;
    int fl = 0;
    for (int t = blockIdx.x * EXACT_WARPS + wid; t < count; t += nw) {
        int r = run_cell(ws, in, out, list[t]);
        fl |= r & 7;
    }
    if (lane == 0 && fl) atomicOr(err, (unsigned long long)fl);
}

// exact k nearest of each query by (d^2, j) (_kernels.py:1562-1620), warp per query
__global__ void __launch_bounds__(EXACT_WARPS * 32)
    k_knn(CellIn in, int64_t nq, const double *__restrict__ q, int k, double t0,
          WS<ExactCaps> *__restrict__ wsbase, int64_t *__restrict__ out_idx) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WS<ExactCaps> *ws = wsbase + (size_t)blockIdx.x * EXACT_WARPS + wid;
    const int nw = gridDim.x * EXACT_WARPS;
    for (int64_t t = blockIdx.x * EXACT_WARPS + wid; t < nq; t += nw) {
        const double qx = q[3 * t], qy = q[3 * t + 1], qz = q[3 * t + 2];
        double tlo = -1.0, thi = t0;
        int got = 0;
        for (;;) {
            bool all = false;
            int nc = gather_shell<true>(ws, in, -1, qx, qy, qz, tlo, thi, &all);
            if (nc > ExactCaps::CC) {
                double base = tlo > 0.0 ? tlo : 0.0;
                double nt = base + (thi - base) * 0.25;
                if (!(nt > base) || !(nt < thi)) {  // > CC sites tied at one distance
                    for (int c = got + lane; c < k; c += 32) out_idx[t * k + c] = -1;
                    break;
                }
                thi = nt;
                continue;
            }
            sort_candidates(ws, nc);
            // emit the shell's candidates in order
            int take = nc < k - got ? nc : k - got;
            for (int c = lane; c < take; c += 32) out_idx[t * k + got + c] = ws->u.b.cj[c];
            got += take;
            __syncwarp();
            if (got >= k || all) break;
            tlo = thi;
            thi = thi * 4.0;
        }
    }
}

// kNN with a shared-memory workspace (k <= 64): warp per query, 8 warps per
// block, all SMs busy; the query's shells are gathered and (d^2, j)-sorted as
// in the cell build.  k > 64 (or a shell of > 64 candidates tied at one
// distance) falls back to k_knn's reference-capacity workspace.
using KnnCaps = Caps<8, 8, 8, 64, 8, 8, false>;
using KnnWS = BWS<KnnCaps>;
constexpr int KNN_WARPS = 8;
__global__ void __launch_bounds__(KNN_WARPS * 32)
    k_knn_fast(CellIn in, int64_t nq, const double *__restrict__ q, int k, double t0,
               int64_t *__restrict__ out_idx, int *__restrict__ fallback, int *__restrict__ nfall) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    KnnWS *ws = (KnnWS *)(smem + (size_t)wid * sizeof(KnnWS));
    const int64_t nw = (int64_t)gridDim.x * KNN_WARPS;
    for (int64_t t = blockIdx.x * (int64_t)KNN_WARPS + wid; t < nq; t += nw) {
        const double qx = q[3 * t], qy = q[3 * t + 1], qz = q[3 * t + 2];
        // first shell sized from the local site density (the 3x3x3 buckets
        // around q) for ~2k candidates: one gather for most queries
        double thi = t0;
        {
            const GridView &g = in.g;
            const int bx = bucket_coord(qx, g.lo[0], g.ih[0], g.gn[0]);
            const int by = bucket_coord(qy, g.lo[1], g.ih[1], g.gn[1]);
            const int bz = bucket_coord(qz, g.lo[2], g.ih[2], g.gn[2]);
            int cnt = 0, nb = 0;
            if (lane < 27) {
                const int x = bx + lane / 9 - 1, y = by + (lane / 3) % 3 - 1, z = bz + lane % 3 - 1;
                if (x >= 0 && y >= 0 && z >= 0 && x < g.gn[0] && y < g.gn[1] && z < g.gn[2]) {
                    const int l = (x * g.gn[1] + y) * g.gn[2] + z;
                    cnt = g.bstart[l + 1] - g.bstart[l];
                    nb = 1;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                nb += __shfl_xor_sync(0xffffffffu, nb, o);
            }
            if (cnt > 0) {
                const double vb = 1.0 / (g.ih[0] * g.ih[1] * g.ih[2]);  // bucket volume
                const double rho = cnt / (nb * vb);
                const double r3 = 2.0 * k / (4.1887902047863905 * rho);
                thi = cbrt(r3 * r3);
            }
        }
        double tlo = -1.0;
        int got = 0;
        bool fail = false;
        for (;;) {
            bool all = false;
            const int nc = gather_shell<true>(ws, in, -1, qx, qy, qz, tlo, thi, &all);
            if (nc > KnnCaps::CC) {
                const double base = tlo > 0.0 ? tlo : 0.0;
                const double nt = base + (thi - base) * 0.25;
                if (!(nt > base) || !(nt < thi)) { fail = true; break; }
                thi = nt;
                continue;
            }
            sort_candidates(ws, nc);
            const int take = nc < k - got ? nc : k - got;
            for (int c = lane; c < take; c += 32) out_idx[t * k + got + c] = ws->u.b.cj[c];
            got += take;
            __syncwarp();
            if (got >= k || all) break;
            tlo = thi;
            thi = thi * 4.0;
        }
        if (fail && lane == 0) fallback[atomicAdd(nfall, 1)] = (int)t;
        if (!fail && got < k)
            for (int c = got + lane; c < k; c += 32) out_idx[t * k + c] = -1;
        __syncwarp();
    }
}

// queries that overflowed the fast kNN workspace, with the exact-tier workspace
__global__ void __launch_bounds__(EXACT_WARPS * 32)
    k_knn_list(CellIn in, const int *__restrict__ list, const int *__restrict__ nlist, const double *__restrict__ q,
               int k, double t0, WS<ExactCaps> *__restrict__ wsbase, int64_t *__restrict__ out_idx) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WS<ExactCaps> *ws = wsbase + (size_t)blockIdx.x * EXACT_WARPS + wid;
    const int nw = gridDim.x * EXACT_WARPS;
    for (int u = blockIdx.x * EXACT_WARPS + wid; u < *nlist; u += nw) {
        const int64_t t = list[u];
        const double qx = q[3 * t], qy = q[3 * t + 1], qz = q[3 * t + 2];
        double tlo = -1.0, thi = t0;
        int got = 0;
        for (;;) {
            bool all = false;
            int nc = gather_shell<true>(ws, in, -1, qx, qy, qz, tlo, thi, &all);
            if (nc > ExactCaps::CC) {
                double base = tlo > 0.0 ? tlo : 0.0;
                double nt = base + (thi - base) * 0.25;
                if (!(nt > base) || !(nt < thi)) {
                    for (int c = got + lane; c < k; c += 32) out_idx[t * k + c] = -1;
                    break;
                }
                thi = nt;
                continue;
            }
            sort_candidates(ws, nc);
            int take = nc < k - got ? nc : k - got;
            for (int c = lane; c < take; c += 32) out_idx[t * k + got + c] = ws->u.b.cj[c];
            got += take;
            __syncwarp();
            if (got >= k || all) {
                for (int c = got + lane; c < k; c += 32) out_idx[t * k + c] = -1;
                break;
            }
            tlo = thi;
            thi = thi * 4.0;
        }
    }
}

void fill_cellin(pf_ctx *c, CellIn &in, int64_t n, const double *pts, const double *psi, double tol,
                 double dpsi, int ball_aware, int want_m2) {
    memset(&in, 0, sizeof in);
    in.pts = pts;
    in.psi = psi;
    in.n = (int)n;
    in.g.sx = c->sx; in.g.sy = c->sy; in.g.sz = c->sz; in.g.sid = c->sid; in.g.bstart = c->bstart;
    for (int a = 0; a < 3; a++) { in.g.lo[a] = c->glo[a]; in.g.ih[a] = c->gih[a]; in.g.gn[a] = c->gn[a]; }
    in.dv = c->dv; in.dp = c->dp; in.dt = c->dt; in.dlp = c->dlp; in.dlv = c->dlv;
    in.dnv = c->dnv; in.dnf = c->dnf; in.dnl = c->dnl;
    in.tol = tol;
    in.dpsi = dpsi >= 0.0 ? dpsi : 0.0;
    in.dpsi_ptr = dpsi >= 0.0 ? nullptr : c->dscal;
    in.ball_aware = ball_aware;
    in.want_m2 = want_m2;
    in.strict = c->strict;
    // first shell of the non-ball-aware search: a few bucket edges
    double h = std::max(c->gh[0], std::max(c->gh[1], c->gh[2]));
    in.t_init = (3.0 * h) * (3.0 * h);
}

// max weight per super-bucket (PF_SUPER^3 buckets), thread per super-bucket over
// its columns' contiguous bucket runs
enum { PF_SUPER = 4 };
__global__ void k_super_max(GridView g, const double *__restrict__ psi, double *__restrict__ smax) {
    const int ns = g.sgn[0] * g.sgn[1] * g.sgn[2];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ns; t += gridDim.x * blockDim.x) {
        const int a = t / (g.sgn[1] * g.sgn[2]), b = (t / g.sgn[2]) % g.sgn[1], cz = t % g.sgn[2];
        const int f = g.sf;
        const int k0 = cz * f, k1 = min(k0 + f, g.gn[2]) - 1;
        double m = -1e300;
        for (int ix = a * f; ix < min(a * f + f, g.gn[0]); ix++)
            for (int iy = b * f; iy < min(b * f + f, g.gn[1]); iy++) {
                const int base = (ix * g.gn[1] + iy) * g.gn[2];
                for (int s = g.bstart[base + k0]; s < g.bstart[base + k1 + 1]; s++) m = fmax(m, psi[g.sid[s]]);
            }
        smax[t] = m;
    }
}

// 0..n-1 and the sentinel weight after the sorted ones (the heavy-site list)
enum { PF_HEAVY = 8 };
__global__ void k_iota_tail(int *__restrict__ iota, int64_t n, double *__restrict__ tail) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        iota[t] = (int)t;
    if (blockIdx.x == 0 && threadIdx.x == 0) *tail = -1e300;
}

// per-site weight slack (pf_cell.cuh cell_slack), thread per evaluated cell
// (the cells of a subset call only: chunked callers pay it once in total)
__global__ void k_cell_slack(CellIn in, int64_t count, double *__restrict__ slack) {
    const double dpsi = in.dpsi_ptr ? *in.dpsi_ptr : in.dpsi;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = in.cells ? in.cells[t] : t;
        slack[i] = cell_slack(in.g, in.pts[3 * i], in.pts[3 * i + 1], in.pts[3 * i + 2], in.psi[i], dpsi);
    }
}

int launch_cells(pf_ctx *c, const CellIn &in_, const CellOut &out, int64_t n, cudaStream_t st) {
    CellIn in = in_;
    if (!c->attr_set) {
        CK(cudaFuncSetAttribute(k_cells_fast, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(FAST_WARPS * sizeof(WS<FastCaps>))));
        CK(cudaFuncSetAttribute(k_cells_fast, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        static_assert(sizeof(BWSN<FastCaps>) == sizeof(BWS<FastCaps>), "one launch shape for both build kernels");
        for (const void *kf : {(const void *)k_cells_build<BWSN<FastCaps>, false>,
                               (const void *)k_cells_build<BWS<FastCaps>, false>,
                               (const void *)k_cells_build<BWSN<FastCaps>, true>,
                               (const void *)k_cells_build<BWS<FastCaps>, true>})
            CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(BUILD_WARPS * sizeof(BWS<FastCaps>))));
        CK(cudaFuncSetAttribute(k_cells_eval, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(FAST_WARPS * sizeof(EWS<FastCaps>))));
        if (pf_internal_eval_sync_attr()) return -1;
        CK(cudaFuncSetAttribute(k_cells_mid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(MID_WARPS * sizeof(WS<MidCaps>))));
        c->mid = !getenv("PF_NO_MID");
        {
            const char *e = getenv("PF_EVAL_SYNC");
            c->eval_sync = !(e && e[0] == '0');
        }
        for (const void *kf : {(const void *)k_cells_build<BWSN<FastCaps>, false>,
                               (const void *)k_cells_build<BWS<FastCaps>, false>,
                               (const void *)k_cells_build<BWSN<FastCaps>, true>,
                               (const void *)k_cells_build<BWS<FastCaps>, true>, (const void *)k_cells_eval})
            CK(cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        c->split = getenv("PF_FUSED") ? 0 : 1;
        int nb = 0, nbb = 0, nbe = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_cells_fast, FAST_WARPS * 32,
                                                         FAST_WARPS * sizeof(WS<FastCaps>)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbb, k_cells_build<BWSN<FastCaps>, false>, BUILD_WARPS * 32,
                                                         BUILD_WARPS * sizeof(BWS<FastCaps>)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbe, k_cells_eval, FAST_WARPS * 32,
                                                         FAST_WARPS * sizeof(EWS<FastCaps>)));
        if (nb < 1 || nbb < 1 || nbe < 1) return set_err("fast cell kernels cannot be resident");
        c->fast_blocks = nb * c->nsm;
        c->build_blocks = nbb * c->nsm;
        c->eval_blocks = nbe * c->nsm;
        c->exact_warps = c->nsm * EXACT_WARPS;
        CK(cudaMalloc(&c->exact_ws, (size_t)c->exact_warps * sizeof(WS<ExactCaps>)));
        c->attr_set = true;
    }
    if (ensure(&c->retry_list, &c->retry_cap, (size_t)n + 1)) return -1;
    CK(cudaMemsetAsync(c->counters, 0, 4 * sizeof(int), st));
    CK(cudaMemsetAsync(c->err, 0, sizeof(unsigned long long), st));
    const int64_t count = in.cells ? in.ncells : n;
    const int64_t want = std::max<int64_t>(1, (count + FAST_WARPS - 1) / FAST_WARPS);
    const int64_t blocks = std::min<int64_t>(c->fast_blocks, want);
    const int64_t bblocks = std::min<int64_t>(c->build_blocks, std::max<int64_t>(1, (count + BUILD_WARPS - 1) / BUILD_WARPS));
    int64_t eblocks = std::min<int64_t>(c->eval_blocks, want);
    if (const char *e = getenv("PF_EVAL_BPSM"))  // development experiment: cap eval blocks per SM
        eblocks = std::min<int64_t>(eblocks, (int64_t)atoi(e) * c->nsm);
    if (!c->ev[0]) {
        CK(cudaEventCreate(&c->ev[0]));
        CK(cudaEventCreate(&c->ev[1]));
    }
    CK(cudaEventRecord(c->ev[0], st));
    if (in.ball_aware && count > 0 && !getenv("PF_GLOBAL_SLACK")) {
        in.g.sf = PF_SUPER;
        if (const char *e = getenv("PF_SUPER_F")) in.g.sf = std::max(1, atoi(e));  // development experiment
        for (int a = 0; a < 3; a++) in.g.sgn[a] = (in.g.gn[a] + in.g.sf - 1) / in.g.sf;
        const size_t ns = (size_t)in.g.sgn[0] * in.g.sgn[1] * in.g.sgn[2];
        if (!(c->keep_w && c->have_smax)) {
            if (ensure(&c->smax, &c->smax_cap, ns)) return -1;
            g_launches++;
            k_super_max<<<(int)std::min<size_t>((ns + 255) / 256, (size_t)c->nsm * 8), 256, 0, st>>>(in.g, in.psi,
                                                                                                      c->smax);
            CK(cudaGetLastError());
            c->have_smax = c->keep_w;
        }
        in.g.smax = c->smax;
        if (ensure(&c->cslack, &c->cslack_cap, (size_t)n)) return -1;
        g_launches++;
        k_cell_slack<<<(int)std::min<int64_t>((count + 255) / 256, (int64_t)c->nsm * 16), 256, 0, st>>>(in, count,
                                                                                                          c->cslack);
        CK(cudaGetLastError());
        in.cslack = c->cslack;
    }
    if (!in.ball_aware && count > 0 && !getenv("PF_NO_HEAVY")) {
        // full mode: the PF_HEAVY heaviest sites for build_cell's heavy-site phase
        const size_t nn = (size_t)n;
        if (c->hv_cap < nn + 1) {
            for (void *p : {(void *)c->hv_keys, (void *)c->hv_iota, (void *)c->hv_vals})
                if (p) cudaFree(p);
            CK(cudaMalloc(&c->hv_keys, (nn + 1) * sizeof(double)));
            CK(cudaMalloc(&c->hv_iota, nn * sizeof(int)));
            CK(cudaMalloc(&c->hv_vals, nn * sizeof(int)));
            c->hv_cap = nn + 1;
        }
        g_launches++;
        k_iota_tail<<<(int)std::min<int64_t>((n + 255) / 256, (int64_t)c->nsm * 8), 256, 0, st>>>(c->hv_iota, n,
                                                                                                 c->hv_keys + n);
        size_t need = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, need, in.psi, c->hv_keys, c->hv_iota, c->hv_vals, (int)n,
                                                  0, 64, st);
        if (need > c->hv_tmp_cap) {
            if (c->hv_tmp) cudaFree(c->hv_tmp);
            CK(cudaMalloc(&c->hv_tmp, need));
            c->hv_tmp_cap = need;
        }
        CK(cub::DeviceRadixSort::SortPairsDescending(c->hv_tmp, need, in.psi, c->hv_keys, c->hv_iota, c->hv_vals,
                                                     (int)n, 0, 64, st));
        g_launches += 4;
        in.heavy_idx = c->hv_vals;
        in.heavy_psi = c->hv_keys;
        in.nheavy = (int)std::min<int64_t>(PF_HEAVY, n);
    }
    cudaEvent_t *sev = nullptr;
    if (c->stage_on && c->split && count > 0) {
        if (c->stage_n == c->stage_ev.size()) {
            std::array<cudaEvent_t, 3> t;
            for (auto &e : t) CK(cudaEventCreate(&e));
            c->stage_ev.push_back(t);
        }
        sev = c->stage_ev[c->stage_n++].data();
        CK(cudaEventRecord(sev[0], st));
    }
    if (c->split && count > 0) {
        if (ensure(&c->gpoly, &c->gpoly_cap, (size_t)n) || ensure(&c->stage, &c->stage_cap, (size_t)n))
            return -1;
        if (c->eval_sort < 0) {
            const char *e = getenv("PF_EVAL_SORT");
            c->eval_sort = !(e && e[0] == '0');
        }
        const bool sorted = c->eval_sort && c->eval_sync && count > 4096;
        if (sorted && (ensure(&c->ekey, &c->ekey_cap, (size_t)count) || ensure(&c->ekey2, &c->ekey2_cap, (size_t)count) ||
                       ensure(&c->eidx, &c->eidx_cap, (size_t)count) || ensure(&c->eidx2, &c->eidx2_cap, (size_t)count)))
            return -1;
        g_launches++;
        auto kb = (in.ball_aware && !out.pk_status) ? (out.census16 ? k_cells_build<BWS<FastCaps>, false> : k_cells_build<BWSN<FastCaps>, false>)
                                : (out.census16 ? k_cells_build<BWS<FastCaps>, true> : k_cells_build<BWSN<FastCaps>, true>);
        kb<<<(int)bblocks, BUILD_WARPS * 32, BUILD_WARPS * sizeof(BWS<FastCaps>), st>>>(
            in, out, (int)count, c->gpoly, c->stage, c->retry_list, c->counters, c->err,
            sorted ? c->ekey : nullptr, sorted ? c->eidx : nullptr);
        CK(cudaGetLastError());
        if (sev) CK(cudaEventRecord(sev[1], st));
        g_launches++;
        if (c->eval_sync) {
            CellIn ein = in;
            int ecount = (int)count;
            if (sorted) {
                // The 8 warps of an evaluation block run every phase in lockstep,
                // so a round costs its largest cell: similar cells share rounds.
                size_t need = 0;
                cub::DeviceRadixSort::SortPairs(nullptr, need, c->ekey, c->ekey2, c->eidx, c->eidx2, ecount, 0, 8, st);
                if (need > c->esort_cap) {
                    if (c->esort_tmp) cudaFree(c->esort_tmp);
                    CK(cudaMalloc(&c->esort_tmp, need));
                    c->esort_cap = need;
                }
                CK(cub::DeviceRadixSort::SortPairs(c->esort_tmp, need, c->ekey, c->ekey2, c->eidx, c->eidx2, ecount,
                                                   0, 8, st));
                g_launches += 2;
                ein.cells = c->eidx2;
                ein.ncells = ecount;
            }
            if (pf_internal_eval_sync(ein, out, ecount, c->gpoly, c->stage, c->retry_list, c->counters, c->err,
                                      c->nsm, st))
                return -1;
        } else {
            k_cells_eval<<<(int)eblocks, FAST_WARPS * 32, FAST_WARPS * sizeof(EWS<FastCaps>), st>>>(
                in, out, (int)count, c->gpoly, c->stage, c->retry_list, c->counters, c->err);
        }
        CK(cudaGetLastError());
    } else {
        g_launches++;
        k_cells_fast<<<(int)blocks, FAST_WARPS * 32, FAST_WARPS * sizeof(WS<FastCaps>), st>>>(
            in, out, (int)count, c->retry_list, c->counters, c->err);
        CK(cudaGetLastError());
    }
    if (c->mid) {
        if (ensure(&c->retry_list2, &c->retry2_cap, (size_t)n + 1)) return -1;
        g_launches++;
        k_cells_mid<<<c->nsm, MID_WARPS * 32, MID_WARPS * sizeof(WS<MidCaps>), st>>>(
            in, out, c->retry_list, c->counters, c->retry_list2, c->err);
        CK(cudaGetLastError());
    }
    g_launches++;
    k_cells_exact<<<c->exact_warps / EXACT_WARPS, EXACT_WARPS * 32, 0, st>>>(
        in, out, c->mid ? c->retry_list2 : c->retry_list, c->mid ? c->counters + 1 : c->counters, c->exact_ws,
        c->err);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[1], st));
    if (sev) CK(cudaEventRecord(sev[2], st));
    c->ev_valid = true;
    return 0;
}

int grid_build(pf_ctx *c, int64_t n, const double *pts, const double *psi, double cell_size,
               cudaStream_t st, const int *dims = nullptr) {
    if (!c->has_domain) return set_err("pf_grid_build: no domain set");
    double ext[3];
    for (int a = 0; a < 3; a++) ext[a] = std::max(c->dhi[a] - c->dlo[a], 1e-300);
    double H = cell_size;
    if (!(H > 0.0)) {
        // bucket edge = mean ball radius (~ half the ball-aware search radius).
        // The cell results do not depend on the bucket layout, so
        // the edge is cached per site count and refreshed from an asynchronous
        // read: only the first build of a run waits for the device.
        H = 0.0;
        if (psi && n > 0) {
            if (!c->h_pinned) {
                CK(cudaMallocHost(&c->h_pinned, sizeof(double)));
                CK(cudaEventCreateWithFlags(&c->h_ev, cudaEventDisableTiming));
            }
            if (c->h_pending && c->h_cache_n == n && cudaEventQuery(c->h_ev) == cudaSuccess) {
                c->h_cache = *c->h_pinned / (double)n;
                c->h_pending = false;
            }
            const bool have = c->h_cache_n == n && c->h_cache > 0.0;
            if (!c->h_pending || !have) {
                CK(cudaMemsetAsync(c->dscal + 3, 0, sizeof(double), st));
                g_launches++;
                k_sum_sqrt<<<c->nsm * 4, 256, 0, st>>>(psi, n, c->dscal + 3);
                CK(cudaMemcpyAsync(c->h_pinned, c->dscal + 3, sizeof(double), cudaMemcpyDeviceToHost, st));
                CK(cudaEventRecord(c->h_ev, st));
                c->h_pending = true;
            }
            if (!have) {
                CK(cudaEventSynchronize(c->h_ev));
                c->h_cache = *c->h_pinned / (double)n;
                c->h_cache_n = n;
                c->h_pending = false;
            }
            H = c->h_cache;
        }
        if (!(H > 0.0)) H = 0.5 * std::cbrt(c->dvol / (double)std::max<int64_t>(n, 1));
    }
    // bound the bucket count (memory and scan cost): <= 512 per axis, <= 2^24 total
    int g[3];
    for (;;) {
        for (int a = 0; a < 3; a++) g[a] = (int)std::min(512.0, std::max(1.0, std::ceil(ext[a] / H)));
        if ((double)g[0] * g[1] * g[2] <= 16777216.0) break;
        H *= 1.25;
    }
    if (dims)
        for (int a = 0; a < 3; a++) g[a] = std::max(1, dims[a]);
    for (int a = 0; a < 3; a++) {
        c->gn[a] = g[a];
        c->glo[a] = c->dlo[a];
        c->gh[a] = ext[a] / g[a];
        c->gih[a] = 1.0 / c->gh[a];
    }
    const int64_t ncell = (int64_t)g[0] * g[1] * g[2];
    const size_t bcap0 = c->bcount_cap;
    if (ensure(&c->sx, &c->sx_cap, n) || ensure(&c->sy, &c->sy_cap, n) || ensure(&c->sz, &c->sz_cap, n) ||
        ensure(&c->sid, &c->sid_cap, n) || ensure(&c->bid, &c->bid_cap, n) ||
        ensure(&c->bcount, &c->bcount_cap, ncell + 17) || ensure(&c->bstart, &c->bstart_cap, ncell + 17))
        return -1;
    if (c->bcount_cap != bcap0) c->bcount_zero = -1;  // reallocated
    if (!c->grid_coop_blocks) {
        int per = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_grid_coop, GRID_T, 0));
        c->grid_coop_blocks = c->nsm * std::max(1, std::min(per, 2));
        CK(cudaMalloc(&c->grid_part, sizeof(int) * c->grid_coop_blocks));
    }
    if (c->bcount_zero < ncell) {  // first build on this buffer (later builds leave it zeroed)
        CK(cudaMemsetAsync(c->bcount, 0, (ncell + 1) * sizeof(int), st));
        c->bcount_zero = ncell;
    }
    int64_t nn = n, nc = ncell;
    double lo0 = c->glo[0], lo1 = c->glo[1], lo2 = c->glo[2], ih0 = c->gih[0], ih1 = c->gih[1], ih2 = c->gih[2];
    int g0 = g[0], g1 = g[1], g2 = g[2];
    void *args[] = {(void *)&pts, &nn, &lo0, &lo1, &lo2, &ih0, &ih1, &ih2, &g0, &g1, &g2, &nc,
                    &c->bid, &c->bcount, &c->bstart, &c->sid, &c->sx, &c->sy, &c->sz, &c->grid_part};
    g_launches++;
    CK(cudaLaunchCooperativeKernel((const void *)k_grid_coop, c->grid_coop_blocks, GRID_T, args, 0, st));
    c->grid_n = n;
    c->grid_pts = pts;
    return 0;
}

int dpsi_dev(pf_ctx *c, int64_t n, const double *psi, cudaStream_t st) {
    unsigned long long init[2] = {~0ull, 0ull};
    CK(cudaMemcpyAsync(c->mm, init, sizeof init, cudaMemcpyHostToDevice, st));
    g_launches++;
    if (n > 0) k_minmax<<<c->nsm * 4, 256, 0, st>>>(psi, n, c->mm);
    g_launches++;
    k_dpsi_finish<<<1, 1, 0, st>>>(c->mm, n, c->dscal);
    CK(cudaGetLastError());
    return 0;
}

// FP64 pipe peak: independent DFMA chains, 8 per thread, no memory traffic
__global__ void __launch_bounds__(256) k_dfma_peak(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
    double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (r == 1234.5) out[0] = r;  // keep the chains alive
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char *pf_version(void) { return "potflow-b200 0.1.0 (sm_100a)"; }

unsigned long long pf_launch_count(void) { return g_launches; }

// measured FP64 FMA throughput of this device (TFLOP/s, FMA = 2 flops)
int pf_fp64_peak(double *tflops_host, double *ms_host) {
    const int iters = 4096, threads = 256;
    int dev = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int blocks = nsm * 8;
    double *buf = nullptr;
    CK(cudaMalloc(&buf, sizeof(double)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    g_launches++;
    k_dfma_peak<<<blocks, threads>>>(buf, 64, 0.999999, 1e-7);  // warm
    CK(cudaEventRecord(e0));
    g_launches++;
    k_dfma_peak<<<blocks, threads>>>(buf, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    if (tflops_host) *tflops_host = flops / (ms * 1e-3) / 1e12;
    if (ms_host) *ms_host = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    return 0;
}
const char *pf_last_error(void) { return g_err.c_str(); }

int pf_ctx_create(pf_ctx **out, int device) {
    if (!out) return set_err("pf_ctx_create: null out");
    CK(cudaSetDevice(device));
    pf_ctx *c = new pf_ctx();
    c->device = device;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        delete c;
        return set_err("pf_ctx_create: device %d is sm_%d%d, this build targets sm_100a", device,
                       prop.major, prop.minor);
    }
    c->nsm = prop.multiProcessorCount;
    CK(cudaMalloc(&c->dscal, 8 * sizeof(double)));
    CK(cudaMalloc(&c->mm, 2 * sizeof(unsigned long long)));
    CK(cudaMalloc(&c->counters, 4 * sizeof(int)));
    CK(cudaMalloc(&c->err, sizeof(unsigned long long)));
    CK(cudaMemset(c->dscal, 0, 8 * sizeof(double)));
    if (const char *e = getenv("PF_PARITY_MODE")) c->strict = e[0] == '1';
    *out = c;
    return 0;
}

int pf_set_parity_mode(pf_ctx *c, int on) {
    if (!c) return set_err("pf_set_parity_mode: null context");
    c->strict = on != 0;
    return 0;
}

int pf_get_parity_mode(pf_ctx *c) { return c ? c->strict : 0; }

int pf_ctx_destroy(pf_ctx *c) {
    if (!c) return 0;
    void *ptrs[] = {c->dv, c->dp, c->dt, c->dlp, c->dlv, c->sx, c->sy, c->sz, c->sid, c->bid,
                    c->bcount, c->bstart, c->scan_tmp, c->dscal, c->mm, c->retry_list, c->counters,
                    c->err, c->census, c->exact_ws, c->gpoly, c->stage, c->smax, c->cslack, c->retry_list2, c->csr_cnt, c->csr_off, c->grid_part,
                    c->ekey, c->ekey2, c->eidx, c->eidx2, c->esort_tmp, c->hv_keys, c->hv_iota, c->hv_vals,
                    c->hv_tmp};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->h_ev) cudaEventDestroy(c->h_ev);
    delete c;
    return 0;
}

int pf_set_domain(pf_ctx *c, const double *dv, const int64_t *dc, const double *dp, const int64_t *dt,
                  const int64_t *dlp, const int64_t *dlv, double tol) {
    int nv = (int)dc[0], nf = (int)dc[1], nl = (int)dc[2];
    if (nv <= 0 || nf <= 0 || nl <= 0 || nv > FastCaps::CV || nf > FastCaps::CF || nl > FastCaps::CL)
        return set_err("pf_set_domain: domain (%d verts, %d facets, %d loop entries) exceeds the "
                       "shared-memory cell capacity", nv, nf, nl);
    int dti[REF_MAX_F], dlpi[REF_MAX_F + 1], dlvi[REF_MAX_L];
    for (int f = 0; f < nf; f++) dti[f] = (int)dt[f];
    for (int f = 0; f <= nf; f++) dlpi[f] = (int)dlp[f];
    for (int k = 0; k < nl; k++) dlvi[k] = (int)dlv[k];
    void *ptrs[] = {c->dv, c->dp, c->dt, c->dlp, c->dlv};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    CK(cudaMalloc(&c->dv, 3 * nv * sizeof(double)));
    CK(cudaMalloc(&c->dp, 4 * nf * sizeof(double)));
    CK(cudaMalloc(&c->dt, nf * sizeof(int)));
    CK(cudaMalloc(&c->dlp, (nf + 1) * sizeof(int)));
    CK(cudaMalloc(&c->dlv, nl * sizeof(int)));
    CK(cudaMemcpy(c->dv, dv, 3 * nv * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dp, dp, 4 * nf * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dt, dti, nf * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dlp, dlpi, (nf + 1) * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dlv, dlvi, nl * sizeof(int), cudaMemcpyHostToDevice));
    c->dnv = nv; c->dnf = nf; c->dnl = nl;
    c->tol = tol;
    for (int a = 0; a < 3; a++) { c->dlo[a] = INFINITY; c->dhi[a] = -INFINITY; }
    for (int v = 0; v < nv; v++)
        for (int a = 0; a < 3; a++) {
            c->dlo[a] = std::min(c->dlo[a], dv[3 * v + a]);
            c->dhi[a] = std::max(c->dhi[a], dv[3 * v + a]);
        }
    // polytope volume by apex fan (geom.cell_volume_convex, geom.py:506-518)
    double ap[3] = {0, 0, 0};
    for (int v = 0; v < nv; v++)
        for (int a = 0; a < 3; a++) ap[a] += dv[3 * v + a] / nv;
    double vol = 0.0;
    for (int f = 0; f < nf; f++) {
        const double *p0 = dv + 3 * dlv[dlp[f]];
        for (int k = (int)dlp[f] + 1; k + 1 < (int)dlp[f + 1]; k++) {
            const double *p1 = dv + 3 * dlv[k], *p2 = dv + 3 * dlv[k + 1];
            double u[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
            double w[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
            double cr[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]};
            vol += cr[0] * (p0[0] - ap[0]) + cr[1] * (p0[1] - ap[1]) + cr[2] * (p0[2] - ap[2]);
        }
    }
    c->dvol = std::fabs(vol) / 6.0;
    c->has_domain = true;
    c->grid_n = -1;  // the grid's origin and edge come from the domain bbox
    c->grid_pts = nullptr;
    return 0;
}

int pf_grid_build(pf_ctx *c, int64_t n, const double *pts, const double *psi, double cell_size,
                  void *stream) {
    return grid_build(c, n, pts, psi, cell_size, S(stream));
}

int pf_grid_build_dims(pf_ctx *c, int64_t n, const double *pts, const int *dims_host, void *stream) {
    return grid_build(c, n, pts, nullptr, 1.0, S(stream), dims_host);
}

}  // extern "C"
// device view of the current bucket grid (renderer)
int pf_internal_grid_view(pf_ctx *c, const double **sx, const double **sy, const double **sz, const int **sid,
                          const int **bstart, int *gn, double *lo, double *h) {
    if (c->grid_n < 0 || !c->sid) return set_err("grid view: no grid");
    *sx = c->sx; *sy = c->sy; *sz = c->sz; *sid = c->sid; *bstart = c->bstart;
    for (int a = 0; a < 3; a++) { gn[a] = c->gn[a]; lo[a] = c->glo[a]; h[a] = c->gh[a]; }
    return 0;
}
int pf_internal_domain_view(pf_ctx *c, const double **dp, int *nf, double *tol) {
    if (!c->has_domain) return set_err("domain view: no domain set");
    *dp = c->dp; *nf = c->dnf; *tol = c->tol;
    return 0;
}
// compact per-facet CSR of the fixed-stride outputs:
// count per cell, two-level exclusive scan, then a thread-per-cell copy
__global__ void k_facet_count(int64_t n, int64_t smf, const int64_t *__restrict__ fcount, int *__restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = i < n ? fcount[i] : 0;
        cnt[i] = (int)(k < 0 ? 0 : (k > smf ? smf : k));
    }
}
__global__ void k_facet_fill(int64_t n, int64_t smf, const int *__restrict__ off, const int64_t *__restrict__ ftag,
                             const double *__restrict__ farea, const double *__restrict__ fh,
                             const double *__restrict__ fnrm, const double *__restrict__ fcent,
                             int64_t *__restrict__ row_ptr, int64_t *__restrict__ tag_o, double *__restrict__ area_o,
                             double *__restrict__ h_o, double *__restrict__ nrm_o, double *__restrict__ cent_o) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = off[i];
        if (row_ptr) row_ptr[i] = o;
        if (i == n) continue;
        const int64_t m = off[i + 1] - o;
        for (int64_t s = 0; s < m; s++) {
            const int64_t a = i * smf + s, b = o + s;
            if (tag_o) tag_o[b] = ftag[a];
            if (area_o) area_o[b] = farea[a];
            if (h_o) h_o[b] = fh[a];
            for (int d = 0; d < 3; d++) {
                if (nrm_o) nrm_o[3 * b + d] = fnrm[3 * a + d];
                if (cent_o) cent_o[3 * b + d] = fcent[3 * a + d];
            }
        }
    }
}

extern "C" {
int pf_grid_info(pf_ctx *c, int *dims, double *lo, double *h) {
    for (int a = 0; a < 3; a++) {
        if (dims) dims[a] = c->gn[a];
        if (lo) lo[a] = c->glo[a];
        if (h) h[a] = c->gh[a];
    }
    return 0;
}

int pf_grid_export(pf_ctx *c, int64_t *bucket_start, int64_t *bucket_sites, void *stream) {
    if (c->grid_n < 0) return set_err("pf_grid_export: no grid");
    int ncell = c->gn[0] * c->gn[1] * c->gn[2];
    g_launches++;
    k_grid_export<<<c->nsm * 4, 256, 0, S(stream)>>>(c->bstart, ncell, c->sid, c->grid_n, bucket_start,
                                                     bucket_sites);
    CK(cudaGetLastError());
    return 0;
}

int pf_dpsi_max(pf_ctx *c, int64_t n, const double *psi, double *dpsi_host, void *stream) {
    if (dpsi_dev(c, n, psi, S(stream))) return -1;
    if (dpsi_host) {
        CK(cudaMemcpyAsync(dpsi_host, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
        CK(cudaStreamSynchronize(S(stream)));
    }
    return 0;
}

int64_t pf_batch_evaluate(pf_ctx *c, int64_t n, const double *pts, const double *psi, double tol,
                          double dpsi_max, int ball_aware, int want_m2, int64_t smf, int64_t *status,
                          double *vol, double *ksur, double *cent, double *ipt, double *m2,
                          int64_t *fcount, int64_t *ftag, double *farea, double *fh, double *fnrm,
                          double *fcent, int rebuild_grid, void *stream) {
    return pf_batch_evaluate_ex(c, n, pts, psi, tol, dpsi_max, ball_aware, want_m2, smf, status, vol,
                                ksur, cent, ipt, m2, fcount, ftag, farea, fh, fnrm, fcent, nullptr, 0,
                                nullptr, nullptr, rebuild_grid, stream);
}

int64_t pf_batch_evaluate_ex(pf_ctx *c, int64_t n, const double *pts, const double *psi, double tol,
                             double dpsi_max, int ball_aware, int want_m2, int64_t smf, int64_t *status,
                             double *vol, double *ksur, double *cent, double *ipt, double *m2,
                             int64_t *fcount, int64_t *ftag, double *farea, double *fh, double *fnrm,
                             double *fcent, const int32_t *cells, int64_t ncells, int32_t *cell_flags,
                             int32_t *census16, int rebuild_grid, void *stream) {
    cudaStream_t st = S(stream);
    if (!c->has_domain) return set_err("pf_batch_evaluate: no domain set");
    if (n < 0 || n > 0x7fffffff) return set_err("pf_batch_evaluate: bad n");
    if (rebuild_grid || c->grid_n != n || c->grid_pts != pts) {
        if (grid_build(c, n, pts, psi, 0.0, st)) return -1;
    }
    if (dpsi_max < 0.0 && !(c->keep_w && c->have_dpsi)) {
        if (dpsi_dev(c, n, psi, st)) return -1;
        c->have_dpsi = c->keep_w;
    }
    if (ensure(&c->census, &c->census_cap, (size_t)n + 1)) return -1;
    CellIn in;
    fill_cellin(c, in, n, pts, psi, tol, dpsi_max, ball_aware, want_m2);
    CellOut out;
    memset(&out, 0, sizeof out);
    out.status = status; out.vol = vol; out.ksur = ksur; out.cent = cent; out.ipt = ipt; out.m2 = m2;
    out.fcount = fcount; out.ftag = ftag; out.farea = farea; out.fh = fh; out.fnrm = fnrm;
    out.fcent = fcent; out.smf = (int)smf; out.census = c->census;
    out.flags = cell_flags;
    out.census16 = census16;
    in.cells = cells;
    in.ncells = (int)ncells;
    if (n > 0 && (!cells || ncells > 0) && launch_cells(c, in, out, n, st)) return -1;
    unsigned long long e = 0;
    if (n > 0) {
        CK(cudaMemcpyAsync(&e, c->err, sizeof e, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    return (int64_t)e;
}

int pf_evaluate_lean(pf_ctx *c, int64_t n, const double *pts, const double *psi, int ball_aware,
                     int64_t smf, double *vol, double *ksur, int32_t *fcount, int32_t *ftag,
                     double *farea, double *cent, int64_t *flags, void *stream) {
    cudaStream_t st = S(stream);
    if (!c->has_domain) return set_err("pf_evaluate_lean: no domain set");
    if (c->grid_n != n || c->grid_pts != pts) return set_err("pf_evaluate_lean: build the grid first");
    if (dpsi_dev(c, n, psi, st)) return -1;
    CellIn in;
    fill_cellin(c, in, n, pts, psi, c->tol, -1.0, ball_aware, 0);
    CellOut out;
    memset(&out, 0, sizeof out);
    out.vol = vol; out.ksur = ksur; out.cent = cent; out.fcount32 = fcount; out.ftag32 = ftag;
    out.farea = farea; out.smf = (int)smf;
    if (n > 0 && launch_cells(c, in, out, n, st)) return -1;
    if (flags) {
        CK(cudaMemcpyAsync(flags, c->err, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    }
    return 0;
}

// _kernels._batch_build (_kernels.py:1481-1559): every unrestricted Laguerre
// cell (ball-aware or full security-radius mode) into the caller's
// fixed-stride packed arrays; returns the OR of the cells' flags
int64_t pf_batch_build(pf_ctx *c, int64_t n, const double *pts, const double *psi, double tol,
                       double dpsi_max, int ball_aware, int64_t smv, int64_t smf, int64_t sml,
                       int64_t *status, int64_t *nv, int64_t *nf, int64_t *nl, double *verts, double *planes,
                       int64_t *tags, int64_t *lp, int64_t *lv, int rebuild_grid, void *stream) {
    cudaStream_t st = S(stream);
    if (!c->has_domain) return set_err("pf_batch_build: no domain set");
    if (n < 0 || n > 0x7fffffff) return set_err("pf_batch_build: bad n");
    if (rebuild_grid || c->grid_n != n || c->grid_pts != pts) {
        if (grid_build(c, n, pts, psi, 0.0, st)) return -1;
    }
    if (dpsi_max < 0.0 && dpsi_dev(c, n, psi, st)) return -1;
    if (ensure(&c->census, &c->census_cap, (size_t)n + 1)) return -1;
    CellIn in;
    fill_cellin(c, in, n, pts, psi, tol, dpsi_max, ball_aware, 0);
    CellOut out;
    memset(&out, 0, sizeof out);
    out.census = c->census;
    out.pk_status = status; out.pk_nv = nv; out.pk_nf = nf; out.pk_nl = nl;
    out.pk_verts = verts; out.pk_planes = planes; out.pk_tags = tags; out.pk_lp = lp; out.pk_lv = lv;
    out.smv = (int)smv; out.smfb = (int)smf; out.sml = (int)sml;
    if (n > 0 && launch_cells(c, in, out, n, st)) return -1;
    unsigned long long e = 0;
    if (n > 0) {
        CK(cudaMemcpyAsync(&e, c->err, sizeof e, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    return (int64_t)e;
}

// lean evaluation of a subset of the cells with a given weight slack dpsi
// (the partitioned solve: owned cells of a slab, all-reduced dpsi)
int pf_evaluate_lean_cells(pf_ctx *c, int64_t n, const double *pts, const double *psi, double dpsi,
                           int ball_aware, int64_t smf, const int32_t *cells, int64_t ncells, double *vol,
                           double *ksur, int32_t *fcount, int32_t *ftag, double *farea, double *cent,
                           int64_t *flags, int rebuild_grid, void *stream) {
    cudaStream_t st = S(stream);
    if (!c->has_domain) return set_err("pf_evaluate_lean_cells: no domain set");
    if (!(dpsi >= 0.0)) return set_err("pf_evaluate_lean_cells: dpsi must be >= 0");
    if (rebuild_grid || c->grid_n != n || c->grid_pts != pts) {
        if (grid_build(c, n, pts, psi, 0.0, st)) return -1;
    }
    CellIn in;
    fill_cellin(c, in, n, pts, psi, c->tol, dpsi, ball_aware, 0);
    in.cells = cells;
    in.ncells = (int)ncells;
    CellOut out;
    memset(&out, 0, sizeof out);
    out.vol = vol; out.ksur = ksur; out.cent = cent; out.fcount32 = fcount; out.ftag32 = ftag;
    out.farea = farea; out.smf = (int)smf;
    if (n > 0 && ncells > 0 && launch_cells(c, in, out, n, st)) return -1;
    if (flags) {
        CK(cudaMemcpyAsync(flags, c->err, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    }
    return 0;
}

__global__ void k_or_flags(unsigned long long *acc, const unsigned long long *err) { *acc |= *err; }

// asynchronous evaluation of a cell subset: the flag word is OR-ed into a
// device accumulator, no host synchronisation (pipelined host round trips)
int pf_batch_evaluate_async(pf_ctx *c, int64_t n, const double *pts, const double *psi, double tol,
                            double dpsi_max, int ball_aware, int want_m2, int64_t smf, int64_t *status,
                            double *vol, double *ksur, double *cent, double *ipt, double *m2,
                            int64_t *fcount, int64_t *ftag, double *farea, double *fh, double *fnrm,
                            double *fcent, const int32_t *cells, int64_t ncells, int32_t *cell_flags,
                            int64_t *err_accum, int rebuild_grid, void *stream) {
    cudaStream_t st = S(stream);
    if (!c->has_domain) return set_err("pf_batch_evaluate_async: no domain set");
    if (n < 0 || n > 0x7fffffff) return set_err("pf_batch_evaluate_async: bad n");
    if (rebuild_grid || c->grid_n != n || c->grid_pts != pts) {
        if (grid_build(c, n, pts, psi, 0.0, st)) return -1;
    }
    if (dpsi_max < 0.0 && !(c->keep_w && c->have_dpsi)) {
        if (dpsi_dev(c, n, psi, st)) return -1;
        c->have_dpsi = c->keep_w;
    }
    if (ensure(&c->census, &c->census_cap, (size_t)n + 1)) return -1;
    CellIn in;
    fill_cellin(c, in, n, pts, psi, tol, dpsi_max, ball_aware, want_m2);
    CellOut out;
    memset(&out, 0, sizeof out);
    out.status = status; out.vol = vol; out.ksur = ksur; out.cent = cent; out.ipt = ipt; out.m2 = m2;
    out.fcount = fcount; out.ftag = ftag; out.farea = farea; out.fh = fh; out.fnrm = fnrm;
    out.fcent = fcent; out.smf = (int)smf; out.census = c->census;
    out.flags = cell_flags;
    in.cells = cells;
    in.ncells = (int)ncells;
    if (n > 0 && (!cells || ncells > 0)) {
        if (launch_cells(c, in, out, n, st)) return -1;
        if (err_accum) {
            g_launches++;
            k_or_flags<<<1, 1, 0, st>>>((unsigned long long *)err_accum, c->err);
            CK(cudaGetLastError());
        }
    }
    return 0;
}

// the bucket-ordered site permutation of the current grid (int32[n])
int pf_grid_order(pf_ctx *c, int32_t *order, void *stream) {
    if (c->grid_n < 0 || !c->sid) return set_err("pf_grid_order: no grid");
    CK(cudaMemcpyAsync(order, c->sid, (size_t)c->grid_n * sizeof(int32_t), cudaMemcpyDeviceToDevice, S(stream)));
    return 0;
}

int pf_last_census(pf_ctx *c, int32_t *census, void *stream) {
    if (!c->census || c->grid_n < 0) return set_err("pf_last_census: nothing evaluated");
    CK(cudaMemcpyAsync(census, c->census, c->grid_n * sizeof(int32_t), cudaMemcpyDeviceToDevice, S(stream)));
    return 0;
}

int pf_last_cells_ms(pf_ctx *c, double *ms) {
    if (!c->ev_valid) return set_err("pf_last_cells_ms: no evaluation recorded");
    CK(cudaEventSynchronize(c->ev[1]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, c->ev[0], c->ev[1]));
    *ms = f;
    return 0;
}

int pf_stage_timing(pf_ctx *c, int enable) {
    c->stage_on = enable != 0;
    c->stage_n = 0;
    return 0;
}

int pf_stage_times(pf_ctx *c, double *build_ms, double *eval_ms, int64_t *evaluations) {
    double b = 0.0, e = 0.0;
    for (size_t k = 0; k < c->stage_n; k++) {
        auto &t = c->stage_ev[k];
        CK(cudaEventSynchronize(t[2]));
        float x = 0.f, y = 0.f;
        CK(cudaEventElapsedTime(&x, t[0], t[1]));
        CK(cudaEventElapsedTime(&y, t[1], t[2]));
        b += x;
        e += y;
    }
    *build_ms = b;
    *eval_ms = e;
    *evaluations = (int64_t)c->stage_n;
    return 0;
}

int pf_last_retry_count(pf_ctx *c, int64_t *count) {
    int v = 0;
    CK(cudaMemcpy(&v, c->counters, sizeof(int), cudaMemcpyDeviceToHost));
    *count = v;
    return 0;
}

int64_t pf_knn(pf_ctx *c, int64_t n, const double *pts, int64_t nq, const double *queries, int64_t k,
               int64_t *out_idx, int rebuild_grid, void *stream) {
    cudaStream_t st = S(stream);
    if (!c->has_domain) return set_err("pf_knn: no domain set");
    if (k > n) k = n;
    if (k <= 0 || nq <= 0) return k > 0 ? k : 0;
    if (rebuild_grid || c->grid_n != n || c->grid_pts != pts) {
        if (grid_build(c, n, pts, nullptr, 0.0, st)) return -1;
    }
    if (!c->attr_set) {
        CellIn dummy;
        CellOut dout;
        memset(&dummy, 0, sizeof dummy);
        memset(&dout, 0, sizeof dout);
        // allocates the exact-tier workspace (no cells launched)
        if (launch_cells(c, dummy, dout, 0, st)) return -1;
    }
    CellIn in;
    fill_cellin(c, in, n, pts, nullptr, c->tol, 0.0, 1, 0);
    double h = std::max(c->gh[0], std::max(c->gh[1], c->gh[2]));
    double r0 = h * std::cbrt((double)k);
    if (k > KnnCaps::CC) {
        g_launches++;
        k_knn<<<c->exact_warps / EXACT_WARPS, EXACT_WARPS * 32, 0, st>>>(in, nq, queries, (int)k, r0 * r0,
                                                                       c->exact_ws, out_idx);
    } else {
        static int knn_blocks = 0;
        const int smem = (int)(KNN_WARPS * sizeof(KnnWS));
        if (!knn_blocks) {
            CK(cudaFuncSetAttribute(k_knn_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            int per = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_knn_fast, KNN_WARPS * 32, smem));
            knn_blocks = c->nsm * std::max(per, 1);
        }
        if (ensure(&c->retry_list, &c->retry_cap, (size_t)nq + 1)) return -1;
        CK(cudaMemsetAsync(c->counters + 2, 0, sizeof(int), st));
        const int64_t want = (nq + KNN_WARPS - 1) / KNN_WARPS;
        g_launches += 2;
        k_knn_fast<<<(int)std::min<int64_t>(knn_blocks, want), KNN_WARPS * 32, smem, st>>>(
            in, nq, queries, (int)k, r0 * r0, out_idx, c->retry_list, c->counters + 2);
        k_knn_list<<<c->exact_warps / EXACT_WARPS, EXACT_WARPS * 32, 0, st>>>(
            in, c->retry_list, c->counters + 2, queries, (int)k, r0 * r0, c->exact_ws, out_idx);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return k;
}

int pf_facets_csr(pf_ctx *c, int64_t n, int64_t smf, const int64_t *fcount, const int64_t *ftag,
                  const double *farea, const double *fh, const double *fnrm, const double *fcent, int64_t cap,
                  int64_t *nnz, int64_t *row_ptr, int64_t *tag, double *area, double *h, double *nrm, double *cent,
                  void *stream) {
    cudaStream_t st = S(stream);
    if (n < 0 || smf <= 0 || !fcount) return set_err("pf_facets_csr: bad arguments");
    if ((double)n * (double)smf > 2147483647.0) return set_err("pf_facets_csr: n * smf exceeds int32 offsets");
    const int64_t nblk = (n + 1 + SCAN_B - 1) / SCAN_B;
    if (nblk > SCAN_B) return set_err("pf_facets_csr: too many cells for the two-level scan");
    if (ensure(&c->csr_cnt, &c->csr_cnt_cap, (size_t)n + 1) || ensure(&c->csr_off, &c->csr_off_cap, (size_t)n + 1) ||
        ensure(&c->scan_tmp, &c->scan_tmp_cap, 2 * nblk + 2))
        return -1;
    const int gb = (int)std::min<int64_t>(c->nsm * 8, (n + 256) / 256);
    g_launches += 2;
    k_facet_count<<<gb, 256, 0, st>>>(n, smf, fcount, c->csr_cnt);
    k_scan_blocks<<<(int)nblk, SCAN_T, 0, st>>>(c->csr_cnt, c->csr_off, n + 1, c->scan_tmp);
    if (nblk > 1) {
        g_launches += 2;
        k_scan_blocks<<<1, SCAN_T, 0, st>>>(c->scan_tmp, c->scan_tmp + nblk + 1, nblk, nullptr);
        k_scan_add<<<(int)nblk, 256, 0, st>>>(c->csr_off, n + 1, c->scan_tmp + nblk + 1);
    }
    int tot = 0;
    CK(cudaMemcpyAsync(&tot, c->csr_off + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (nnz) *nnz = tot;
    if (tot > cap) return set_err("pf_facets_csr: %d facets exceed the capacity %lld", tot, (long long)cap);
    g_launches++;
    k_facet_fill<<<gb, 256, 0, st>>>(n, smf, c->csr_off, ftag, farea, fh, fnrm, fcent, row_ptr, tag, area, h, nrm,
                                      cent);
    CK(cudaGetLastError());
    return 0;
}

}  // extern "C"

unsigned long long pf_internal_launches_add(unsigned long long k) { return g_launches += k; }
int pf_internal_set_err(const char *msg) { return set_err("%s", msg); }
// between keep_weights(c, 1) and keep_weights(c, 0) the weights and the grid
// do not change: the first evaluation computes dpsi and the super-bucket
// maxima, the later ones reuse them
void pf_internal_keep_weights(pf_ctx *c, int on) {
    c->keep_w = on != 0;
    c->have_dpsi = false;
    c->have_smax = false;
}
