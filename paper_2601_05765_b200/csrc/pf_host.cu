// pf_host.cu -- the host-array drop-in of _kernels._batch_evaluate
// (_kernels.py:1362-1478) at the C ABI: pageable HOST arrays in, the
// reference's fixed-stride HOST outputs written exactly as the reference
// writes them (every cell's status / vol / ksur / fcount; cent / ipt / m2
// except on build-overflow cells; facet slots < fcount only -- slots past it
// are left untouched, as the reference leaves them).
//
// Pipeline (one call):
//   H2D pts, psi -> grid counting sort -> K index ranges of cells, each in
//   bucket order (one stable radix sort of the bucket-ordered sites by range)
//   -> per range, on the compute stream: the cell kernels, then a pack of
//   the range's outputs into compact records (96 B per cell, 72 B per
//   restricted facet instead of the 2.3 KB fixed-stride row), and its facet
//   total into pinned memory.
//   The host thread follows the ranges: as range k's total lands it queues
//   the D2H of exactly those bytes into a pinned ring slot (copy stream), and
//   a persistent worker pool scatters the slot into the caller's arrays
//   while the device computes ranges k+1..K.  Device->host bytes are ~40% of
//   the fixed-stride arrays, and the caller's arrays need not be pinned.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <deque>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/potflow_b200.h"

extern unsigned long long pf_internal_launches_add(unsigned long long k);
extern int pf_internal_set_err(const char *msg);
extern void pf_internal_keep_weights(pf_ctx *c, int on);

namespace {

#define HCK(x)                                                                       \
    do {                                                                             \
        cudaError_t _e = (x);                                                        \
        if (_e != cudaSuccess) {                                                     \
            char _b[256];                                                            \
            snprintf(_b, sizeof _b, "%s:%d %s: %s", __FILE__, __LINE__, #x,         \
                     cudaGetErrorString(_e));                                        \
            return pf_internal_set_err(_b);                                          \
        }                                                                            \
    } while (0)

constexpr int DENSE_W = 12;  // doubles per cell record
constexpr int FACET_W = 9;   // doubles per facet record
constexpr int FLAG_BUILD_OVERFLOW = 512;
constexpr int RING = 4;      // pinned staging slots in flight

// ---------------------------------------------------------------------------
// device side
// ---------------------------------------------------------------------------
// range id of every bucket-ordered site (index ranges [bnd[k], bnd[k+1]))
__global__ void k_range_id(const int32_t *__restrict__ order, int64_t n, const int64_t *__restrict__ bnd, int K,
                           uint8_t *__restrict__ rid) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = order[t];
        int lo = 0, hi = K - 1;
        while (lo < hi) {  // last k with bnd[k] <= i
            const int mid = (lo + hi + 1) >> 1;
            if (bnd[mid] <= i) lo = mid; else hi = mid - 1;
        }
        rid[t] = (uint8_t)lo;
    }
}

// facet count per cell of [i0, i1), clamped to smf; cnt[m] = 0 (the scan's total slot)
__global__ void k_pack_count(int64_t i0, int64_t m, int64_t smf, const int64_t *__restrict__ fcount,
                             int32_t *__restrict__ cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= m; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = t < m ? fcount[i0 + t] : 0;
        cnt[t] = (int32_t)(k < 0 ? 0 : (k > smf ? smf : k));
    }
}

// cell records: status, vol, ksur, cent[3], ipt[3], m2, fcount, flags (as doubles / int64 bits)
__global__ void k_pack_dense(int64_t i0, int64_t m, const int64_t *__restrict__ status, const double *__restrict__ vol,
                             const double *__restrict__ ksur, const double *__restrict__ cent,
                             const double *__restrict__ ipt, const double *__restrict__ m2,
                             const int64_t *__restrict__ fcount, const int32_t *__restrict__ flags,
                             double *__restrict__ dst) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + t;
        double r[DENSE_W];
        r[0] = __longlong_as_double(status[i]);
        r[1] = vol[i];
        r[2] = ksur[i];
        r[3] = cent[3 * i]; r[4] = cent[3 * i + 1]; r[5] = cent[3 * i + 2];
        r[6] = ipt[3 * i]; r[7] = ipt[3 * i + 1]; r[8] = ipt[3 * i + 2];
        r[9] = m2[i];
        r[10] = __longlong_as_double(fcount[i]);
        r[11] = __longlong_as_double((long long)flags[i]);
#pragma unroll
        for (int w = 0; w < DENSE_W; w++) dst[t * DENSE_W + w] = r[w];
    }
}

// facet records (warp per cell, lane per slot): tag, area, h, nrm[3], cent[3]
__global__ void k_pack_facets(int64_t i0, int64_t m, int64_t smf, const int32_t *__restrict__ off,
                              const int32_t *__restrict__ cnt, const int64_t *__restrict__ ftag,
                              const double *__restrict__ farea, const double *__restrict__ fh,
                              const double *__restrict__ fnrm, const double *__restrict__ fcent,
                              double *__restrict__ dst) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < m; t += nw) {
        const int64_t i = i0 + t;
        const int c = cnt[t];
        const int64_t o = off[t];
        for (int s = lane; s < c; s += 32) {
            const int64_t a = i * smf + s;
            double *d = dst + (o + s) * FACET_W;
            d[0] = __longlong_as_double(ftag[a]);
            d[1] = farea[a];
            d[2] = fh[a];
            d[3] = fnrm[3 * a]; d[4] = fnrm[3 * a + 1]; d[5] = fnrm[3 * a + 2];
            d[6] = fcent[3 * a]; d[7] = fcent[3 * a + 1]; d[8] = fcent[3 * a + 2];
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// persistent worker pool (scatter of the staged records into the caller's arrays)
class Pool {
  public:
    explicit Pool(int n) {
        for (int t = 0; t < n; t++) th_.emplace_back([this] { run(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    int size() const { return (int)th_.size(); }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> g(m_);
            q_.push_back(std::move(f));
        }
        cv_.notify_one();
    }

  private:
    void run() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [this] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                f = std::move(q_.front());
                q_.pop_front();
            }
            f();
        }
    }
    std::vector<std::thread> th_;
    std::deque<std::function<void()>> q_;
    std::mutex m_;
    std::condition_variable cv_;
    bool stop_ = false;
};

// host timeline of one call (PF_HOST_TRACE=1: printed to stderr; dev tool)
double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// completion count of one range's scatter tasks
struct Job {
    std::mutex m;
    std::condition_variable cv;
    int left = 0;
    double t_copied = 0.0, t_done = 0.0;  // trace
    void done() {
        std::lock_guard<std::mutex> g(m);
        if (--left == 0) {
            t_done = now_ms();
            cv.notify_all();
        }
    }
    void wait() {
        std::unique_lock<std::mutex> l(m);
        cv.wait(l, [this] { return left == 0; });
    }
};

template <class T>
int dev_ensure(T **p, size_t *cap, size_t count) {
    if (*cap >= count && *p) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    const size_t c = std::max<size_t>(count + count / 8, 16);
    HCK(cudaMalloc((void **)p, c * sizeof(T)));
    *cap = c;
    return 0;
}

struct HostPath {
    // device copies of the inputs, the fixed-stride outputs, and the staging
    double *pts = nullptr, *psi = nullptr;
    size_t pts_c = 0, psi_c = 0;
    int64_t *status = nullptr, *fcount = nullptr, *ftag = nullptr;
    size_t status_c = 0, fcount_c = 0, ftag_c = 0;
    double *vol = nullptr, *ksur = nullptr, *cent = nullptr, *ipt = nullptr, *m2 = nullptr;
    size_t vol_c = 0, ksur_c = 0, cent_c = 0, ipt_c = 0, m2_c = 0;
    double *farea = nullptr, *fh = nullptr, *fnrm = nullptr, *fcent = nullptr;
    size_t farea_c = 0, fh_c = 0, fnrm_c = 0, fcent_c = 0;
    int32_t *flags = nullptr, *order = nullptr, *cells = nullptr, *cnt = nullptr, *off = nullptr;
    size_t flags_c = 0, order_c = 0, cells_c = 0, cnt_c = 0, off_c = 0;
    uint8_t *rid = nullptr, *rid2 = nullptr;
    size_t rid_c = 0, rid2_c = 0;
    int64_t *bnd = nullptr;
    size_t bnd_c = 0;
    double *sdense = nullptr, *sfac = nullptr;  // device staging (whole call)
    size_t sdense_c = 0, sfac_c = 0;
    void *cub_tmp = nullptr;
    size_t cub_c = 0;
    int64_t *err = nullptr;
    // pinned
    double *in_stage = nullptr;  // inputs (pts, psi) staged by the worker pool
    size_t in_stage_c = 0;
    double *ring[RING] = {};
    size_t ring_c[RING] = {};
    int32_t *totals = nullptr;  // per-range facet totals (pinned)
    int totals_c = 0;
    cudaStream_t comp = nullptr, copy = nullptr;
    std::vector<cudaEvent_t> ev_tot, ev_copy;
    Pool *pool = nullptr;
    int64_t last_h2d = 0, last_d2h = 0;
    int device = 0;
};

std::mutex g_hp_m;
std::map<pf_ctx *, HostPath *> g_hp;

HostPath *host_path(pf_ctx *c) {
    std::lock_guard<std::mutex> g(g_hp_m);
    HostPath *&h = g_hp[c];
    if (!h) h = new HostPath();
    return h;
}

int ensure_events(HostPath *h, int K) {
    while ((int)h->ev_tot.size() < K) {
        cudaEvent_t a, b;
        HCK(cudaEventCreate(&a));  // timed: PF_HOST_TRACE reads it
        HCK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        h->ev_tot.push_back(a);
        h->ev_copy.push_back(b);
    }
    return 0;
}

int ensure_pinned(double **p, size_t *cap, size_t count) {
    if (*cap >= count && *p) return 0;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    const size_t c = count + count / 4 + 1024;
    HCK(cudaHostAlloc((void **)p, c * sizeof(double), cudaHostAllocDefault));
    *cap = c;
    return 0;
}

// index-range boundaries: equal ranges, the last three shrinking (1/2, 1/4,
// 1/8 of one) so the work left after the last kernel is short, and with
// K >= 10 the first two (1/4, 1/2) so the host's scatter -- host-memory
// bound, about as fast as the device produces -- starts early
std::vector<int64_t> range_bounds(int64_t n, int K) {
    std::vector<double> w(K, 1.0);
    if (K >= 6) { w[K - 3] = 0.5; w[K - 2] = 0.25; w[K - 1] = 0.125; }
    if (K >= 10) { w[0] = 0.25; w[1] = 0.5; }  // the first copy (and the host's scatter) starts early
    double tot = 0.0;
    for (double x : w) tot += x;
    std::vector<int64_t> b(K + 1, 0);
    double acc = 0.0;
    for (int k = 0; k < K; k++) {
        acc += w[k];
        b[k + 1] = (int64_t)std::llround(acc / tot * (double)n);
    }
    b[0] = 0;
    b[K] = n;
    return b;
}

// scatter rows [r0, r1) of range (i0, staged records) into the caller's arrays
void scatter_rows(int64_t i0, int64_t r0, int64_t r1, const double *dense, const double *fac, const int32_t *cell_off,
                  int64_t smf, int64_t *status, double *vol, double *ksur, double *cent, double *ipt, double *m2,
                  int64_t *fcount, int64_t *ftag, double *farea, double *fh, double *fnrm, double *fcent) {
    int64_t fo = cell_off[r0];
    for (int64_t t = r0; t < r1; t++) {
        const int64_t i = i0 + t;
        const double *r = dense + t * DENSE_W;
        int64_t st, fc, fl;
        memcpy(&st, &r[0], 8);
        memcpy(&fc, &r[10], 8);
        memcpy(&fl, &r[11], 8);
        if (status) status[i] = st;
        if (vol) vol[i] = r[1];
        if (ksur) ksur[i] = r[2];
        if (fcount) fcount[i] = fc;
        if (!(fl & FLAG_BUILD_OVERFLOW)) {  // the reference leaves them untouched (_kernels.py:1393-1399)
            if (cent) { cent[3 * i] = r[3]; cent[3 * i + 1] = r[4]; cent[3 * i + 2] = r[5]; }
            if (ipt) { ipt[3 * i] = r[6]; ipt[3 * i + 1] = r[7]; ipt[3 * i + 2] = r[8]; }
            if (m2) m2[i] = r[9];
        }
        const int64_t nk = fc < 0 ? 0 : (fc > smf ? smf : fc);
        // one contiguous run per output array (five write streams at a time
        // instead of interleaving them per facet)
        const double *f = fac + fo * FACET_W;
        const int64_t a0 = i * smf;
        if (ftag)
            for (int64_t s = 0; s < nk; s++) memcpy(&ftag[a0 + s], &f[s * FACET_W], 8);
        if (farea)
            for (int64_t s = 0; s < nk; s++) farea[a0 + s] = f[s * FACET_W + 1];
        if (fh)
            for (int64_t s = 0; s < nk; s++) fh[a0 + s] = f[s * FACET_W + 2];
        if (fnrm)
            for (int64_t s = 0; s < nk; s++) {
                fnrm[3 * (a0 + s)] = f[s * FACET_W + 3];
                fnrm[3 * (a0 + s) + 1] = f[s * FACET_W + 4];
                fnrm[3 * (a0 + s) + 2] = f[s * FACET_W + 5];
            }
        if (fcent)
            for (int64_t s = 0; s < nk; s++) {
                fcent[3 * (a0 + s)] = f[s * FACET_W + 6];
                fcent[3 * (a0 + s) + 1] = f[s * FACET_W + 7];
                fcent[3 * (a0 + s) + 2] = f[s * FACET_W + 8];
            }
        fo += nk;
    }
}

// Transparent huge pages for the caller's output arrays (a hint; the
// scatter writes ~1 KB per cell spread over five 0.5-1.5 GB arrays, so 4 KB
// pages make it TLB bound).  Pages already faulted in keep their size until
// khugepaged merges them; np.zeros arrays are faulted by our first call.
void advise_huge(const void *p, size_t bytes) {
    static const bool on = [] {
        const char *e = getenv("PF_HOST_THP");
        return !(e && e[0] == '0');
    }();
    if (!on || !p || bytes < ((size_t)8 << 20)) return;
    const uintptr_t pg = (uintptr_t)sysconf(_SC_PAGESIZE);
    const uintptr_t a = ((uintptr_t)p + pg - 1) & ~(pg - 1), b = ((uintptr_t)p + bytes) & ~(pg - 1);
    if (b > a) madvise((void *)a, b - a, MADV_HUGEPAGE);
}

}  // namespace

extern "C" {

int64_t pf_batch_evaluate_host(pf_ctx *ctx, int64_t n, const double *pts_h, const double *psi_h, double tol,
                               double dpsi_max, int ball_aware, int want_m2, int64_t smf, int64_t *status,
                               double *vol, double *ksur, double *cent, double *ipt, double *m2, int64_t *fcount,
                               int64_t *ftag, double *farea, double *fh, double *fnrm, double *fcent, int chunks,
                               int64_t *h2d_bytes, int64_t *d2h_bytes) {
    if (!ctx) return pf_internal_set_err("pf_batch_evaluate_host: null context");
    if (n < 0 || n > 0x7fffffff || smf <= 0) return pf_internal_set_err("pf_batch_evaluate_host: bad n / smf");
    HostPath *h = host_path(ctx);
    if (n == 0) return 0;
    if (!h->comp) {
        HCK(cudaStreamCreateWithFlags(&h->comp, cudaStreamNonBlocking));
        HCK(cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking));
        HCK(cudaMalloc(&h->err, sizeof(int64_t)));
        HCK(cudaGetDevice(&h->device));
        const unsigned hw = std::thread::hardware_concurrency();
        // one core left to the thread that follows the ranges and queues the
        // copies (with every core scattering it was descheduled for ms at a time)
        h->pool = new Pool((int)std::max(1u, std::min(hw ? hw - 1 : 4u, 16u)));
    }
    // chunks <= 0: ~12k+ cells per range, 4 to 16 (_kernels.default_chunks)
    const int64_t kdef = std::min<int64_t>(16, std::max<int64_t>(4, n / 12000));
    const int K = (int)std::max<int64_t>(1, std::min<int64_t>(chunks > 0 ? chunks : kdef, std::min<int64_t>(n, 64)));
    const size_t n3 = 3 * (size_t)n, nf = (size_t)n * smf;
    if (dev_ensure(&h->pts, &h->pts_c, n3) || dev_ensure(&h->psi, &h->psi_c, n) ||
        dev_ensure(&h->status, &h->status_c, n) || dev_ensure(&h->vol, &h->vol_c, n) ||
        dev_ensure(&h->ksur, &h->ksur_c, n) || dev_ensure(&h->cent, &h->cent_c, n3) ||
        dev_ensure(&h->ipt, &h->ipt_c, n3) || dev_ensure(&h->m2, &h->m2_c, n) ||
        dev_ensure(&h->fcount, &h->fcount_c, n) || dev_ensure(&h->ftag, &h->ftag_c, nf) ||
        dev_ensure(&h->farea, &h->farea_c, nf) || dev_ensure(&h->fh, &h->fh_c, nf) ||
        dev_ensure(&h->fnrm, &h->fnrm_c, 3 * nf) || dev_ensure(&h->fcent, &h->fcent_c, 3 * nf) ||
        dev_ensure(&h->flags, &h->flags_c, n) || dev_ensure(&h->order, &h->order_c, n) ||
        dev_ensure(&h->cells, &h->cells_c, n) || dev_ensure(&h->cnt, &h->cnt_c, (size_t)n + K + 1) ||
        dev_ensure(&h->off, &h->off_c, (size_t)n + K + 1) || dev_ensure(&h->rid, &h->rid_c, n) ||
        dev_ensure(&h->rid2, &h->rid2_c, n) || dev_ensure(&h->bnd, &h->bnd_c, (size_t)K + 1) ||
        dev_ensure(&h->sdense, &h->sdense_c, (size_t)n * DENSE_W) ||
        dev_ensure(&h->sfac, &h->sfac_c, nf * FACET_W) || ensure_events(h, K))
        return -1;
    if (h->totals_c < K) {
        if (h->totals) cudaFreeHost(h->totals);
        HCK(cudaHostAlloc((void **)&h->totals, K * sizeof(int32_t), cudaHostAllocDefault));
        h->totals_c = K;
    }
    {
        const size_t n1 = (size_t)n * 8, nf8 = (size_t)n * smf * 8;
        advise_huge(status, n1); advise_huge(vol, n1); advise_huge(ksur, n1); advise_huge(m2, n1);
        advise_huge(fcount, n1); advise_huge(cent, 3 * n1); advise_huge(ipt, 3 * n1); advise_huge(ftag, nf8);
        advise_huge(farea, nf8); advise_huge(fh, nf8); advise_huge(fnrm, 3 * nf8); advise_huge(fcent, 3 * nf8);
    }
    cudaStream_t st = h->comp;
    void *sv = (void *)st;
    static const bool trace = getenv("PF_HOST_TRACE") != nullptr;
    const double t_start = trace ? now_ms() : 0.0;
    std::vector<double> t_kern(K, 0.0);
    double t_staged = 0.0, t_queued = 0.0;
    cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};  // trace: stream start, inputs on device, grid + ranges sorted
    if (trace) {
        for (auto &e : tev) HCK(cudaEventCreate(&e));
        HCK(cudaEventRecord(tev[0], st));
    }
    const std::vector<int64_t> bnd = range_bounds(n, K);
    int64_t h2d = 0, d2h = 0;
    // inputs (the caller's pageable arrays): the worker pool copies pieces into
    // pinned staging, each piece's H2D is queued as soon as it is staged
    // (a pageable cudaMemcpy stages through one driver buffer: C4 ~5 ms -> ~1.5 ms)
    {
        if (ensure_pinned(&h->in_stage, &h->in_stage_c, n3 + n)) return -1;
        constexpr int PIECES = 16;
        const size_t tot = n3 + n;
        std::vector<Job> staged(PIECES);
        double *stg = h->in_stage;
        for (int q = 0; q < PIECES; q++) {
            const size_t a = tot * q / PIECES, b = tot * (q + 1) / PIECES;
            staged[q].left = 1;
            Job *job = &staged[q];
            h->pool->submit([=]() {
                // [0, n3) = pts, [n3, n3 + n) = psi
                if (a < n3) memcpy(stg + a, pts_h + a, (std::min(b, n3) - a) * sizeof(double));
                if (b > n3) {
                    const size_t a2 = std::max(a, n3);
                    memcpy(stg + a2, psi_h + (a2 - n3), (b - a2) * sizeof(double));
                }
                job->done();
            });
        }
        for (int q = 0; q < PIECES; q++) {
            const size_t a = tot * q / PIECES, b = tot * (q + 1) / PIECES;
            staged[q].wait();
            if (a < n3)
                HCK(cudaMemcpyAsync(h->pts + a, stg + a, (std::min(b, n3) - a) * sizeof(double),
                                    cudaMemcpyHostToDevice, st));
            if (b > n3) {
                const size_t a2 = std::max(a, n3);
                HCK(cudaMemcpyAsync(h->psi + (a2 - n3), stg + a2, (b - a2) * sizeof(double), cudaMemcpyHostToDevice,
                                    st));
            }
        }
    }
    HCK(cudaMemcpyAsync(h->bnd, bnd.data(), (K + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    h2d += (int64_t)((n3 + n) * sizeof(double));
    HCK(cudaMemsetAsync(h->err, 0, sizeof(int64_t), st));
    if (trace) {
        t_staged = now_ms();
        HCK(cudaEventRecord(tev[1], st));
    }
    if (pf_grid_build(ctx, n, h->pts, h->psi, 0.0, sv)) return -1;
    if (pf_grid_order(ctx, h->order, sv)) return -1;
    // cells of each index range in bucket order: stable radix sort by range id
    if (K > 1) {
        pf_internal_launches_add(1);
        k_range_id<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(h->order, n, h->bnd, K, h->rid);
        int bits = 1;
        while ((1 << bits) < K) bits++;
        size_t need = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, need, h->rid, h->rid2, h->order, h->cells, (int)n, 0, bits, st);
        if (need > h->cub_c) {
            if (h->cub_tmp) cudaFree(h->cub_tmp);
            HCK(cudaMalloc(&h->cub_tmp, need));
            h->cub_c = need;
        }
        HCK(cub::DeviceRadixSort::SortPairs(h->cub_tmp, h->cub_c, h->rid, h->rid2, h->order, h->cells, (int)n, 0,
                                            bits, st));
        pf_internal_launches_add(4);
    } else {
        HCK(cudaMemcpyAsync(h->cells, h->order, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    }
    if (trace) HCK(cudaEventRecord(tev[2], st));
    // per range: cell kernels, pack, facet total
    size_t scan_need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_need, h->cnt, h->off, (int)n + 1, st);
    if (scan_need > h->cub_c) {
        if (h->cub_tmp) cudaFree(h->cub_tmp);
        HCK(cudaMalloc(&h->cub_tmp, scan_need));
        h->cub_c = scan_need;
    }
    // one (grid, psi) for all ranges: dpsi and the slack bounds computed by the first
    struct KeepWeights {
        pf_ctx *c;
        explicit KeepWeights(pf_ctx *c_) : c(c_) { pf_internal_keep_weights(c, 1); }
        ~KeepWeights() { pf_internal_keep_weights(c, 0); }
    } keep(ctx);
    for (int k = 0; k < K; k++) {
        const int64_t i0 = bnd[k], m = bnd[k + 1] - bnd[k];
        if (m <= 0) { h->totals[k] = 0; continue; }
        if (pf_batch_evaluate_async(ctx, n, h->pts, h->psi, tol, dpsi_max, ball_aware, want_m2, smf, h->status,
                                    h->vol, h->ksur, h->cent, h->ipt, h->m2, h->fcount, h->ftag, h->farea, h->fh,
                                    h->fnrm, h->fcent, h->cells + i0, m, h->flags, h->err, 0, sv))
            return -1;
        const int gb = (int)std::min<int64_t>((m + 256) / 256, 148 * 8);
        int32_t *cnt = h->cnt + i0 + k, *off = h->off + i0 + k;  // m + 1 entries per range
        k_pack_count<<<gb, 256, 0, st>>>(i0, m, smf, h->fcount, cnt);
        HCK(cub::DeviceScan::ExclusiveSum(h->cub_tmp, h->cub_c, cnt, off, (int)m + 1, st));
        k_pack_dense<<<gb, 256, 0, st>>>(i0, m, h->status, h->vol, h->ksur, h->cent, h->ipt, h->m2, h->fcount,
                                         h->flags, h->sdense + i0 * DENSE_W);
        k_pack_facets<<<(int)std::min<int64_t>((m + 7) / 8, 148 * 16), 256, 0, st>>>(
            i0, m, smf, off, cnt, h->ftag, h->farea, h->fh, h->fnrm, h->fcent, h->sfac + i0 * smf * FACET_W);
        pf_internal_launches_add(4);
        HCK(cudaGetLastError());
        HCK(cudaMemcpyAsync(h->totals + k, off + m, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HCK(cudaEventRecord(h->ev_tot[k], st));
    }
    if (trace) t_queued = now_ms();
    // host: follow the ranges -- D2H of exactly the staged bytes into a pinned
    // ring slot, then the worker pool scatters it into the caller's arrays
    std::vector<Job> jobs(K);
    std::vector<std::vector<int32_t>> offs(K);
    const int T = h->pool->size();
    for (int k = 0; k < K; k++) {
        const int64_t i0 = bnd[k], m = bnd[k + 1] - bnd[k];
        if (m <= 0) continue;
        const int slot = k % RING;
        if (k >= RING) jobs[k - RING].wait();  // slot free
        HCK(cudaEventSynchronize(h->ev_tot[k]));
        if (trace) t_kern[k] = now_ms();
        const int64_t F = h->totals[k];
        const size_t dn = (size_t)m * DENSE_W, fn = (size_t)F * FACET_W;
        if (ensure_pinned(&h->ring[slot], &h->ring_c[slot], dn + fn)) return -1;
        double *hd = h->ring[slot], *hf = h->ring[slot] + dn;
        HCK(cudaStreamWaitEvent(h->copy, h->ev_tot[k], 0));
        HCK(cudaMemcpyAsync(hd, h->sdense + i0 * DENSE_W, dn * sizeof(double), cudaMemcpyDeviceToHost, h->copy));
        if (fn)
            HCK(cudaMemcpyAsync(hf, h->sfac + i0 * smf * FACET_W, fn * sizeof(double), cudaMemcpyDeviceToHost,
                                h->copy));
        HCK(cudaEventRecord(h->ev_copy[k], h->copy));
        d2h += (int64_t)((dn + fn) * sizeof(double) + sizeof(int32_t));
        // per-row facet offsets for the split of the scatter (host, from the dense records)
        std::vector<int32_t> &o = offs[k];
        o.assign(m + 1, 0);
        Job *job = &jobs[k];
        cudaEvent_t ev = h->ev_copy[k];
        // the offsets need the staged fcounts: one task computes them, then the row tasks run
        const int ntask = (int)std::min<int64_t>(T, std::max<int64_t>(1, m / 2048));
        job->left = ntask;
        const int dev = h->device;
        h->pool->submit([=, &o]() {
            cudaSetDevice(dev);
            cudaEventSynchronize(ev);
            if (trace) job->t_copied = now_ms();
            int64_t acc = 0;
            for (int64_t t = 0; t < m; t++) {
                o[t] = (int32_t)acc;
                int64_t fc;
                memcpy(&fc, &hd[t * DENSE_W + 10], 8);
                acc += fc < 0 ? 0 : (fc > smf ? smf : fc);
            }
            o[m] = (int32_t)acc;
            for (int q = 1; q < ntask; q++)
                h->pool->submit([=, &o]() {
                    const int64_t r0 = m * q / ntask, r1 = m * (q + 1) / ntask;
                    scatter_rows(i0, r0, r1, hd, hf, o.data(), smf, status, vol, ksur, cent, ipt, m2, fcount, ftag,
                                 farea, fh, fnrm, fcent);
                    job->done();
                });
            scatter_rows(i0, 0, m / ntask, hd, hf, o.data(), smf, status, vol, ksur, cent, ipt, m2, fcount, ftag,
                         farea, fh, fnrm, fcent);
            job->done();
        });
    }
    for (int k = 0; k < K; k++)
        if (bnd[k + 1] > bnd[k]) jobs[k].wait();
    int64_t e = 0;
    HCK(cudaMemcpyAsync(&e, h->err, sizeof e, cudaMemcpyDeviceToHost, st));
    HCK(cudaStreamSynchronize(st));
    HCK(cudaStreamSynchronize(h->copy));
    d2h += (int64_t)sizeof e;
    if (trace) {
        float g_in = 0.f, g_grid = 0.f, g_r0 = 0.f;
        cudaEventElapsedTime(&g_in, tev[0], tev[1]);
        cudaEventElapsedTime(&g_grid, tev[1], tev[2]);
        cudaEventElapsedTime(&g_r0, tev[2], h->ev_tot[0]);
        fprintf(stderr, "[pf_host] K=%d threads=%d total %.2f ms; host: inputs staged %.2f, all queued %.2f; "
                "device: inputs %.2f, grid+sort %.2f, range 0 %.2f\n", K, T, now_ms() - t_start, t_staged - t_start,
                t_queued - t_start, g_in, g_grid, g_r0);
        for (auto &e : tev) cudaEventDestroy(e);
        fprintf(stderr, "[pf_host] per range (ms from start): kernels+pack done / copied / scattered\n");
        for (int k = 0; k < K; k++)
            fprintf(stderr, "[pf_host] %2d %8.2f %8.2f %8.2f\n", k, t_kern[k] - t_start, jobs[k].t_copied - t_start,
                    jobs[k].t_done - t_start);
    }
    h->last_h2d = h2d;
    h->last_d2h = d2h;
    if (h2d_bytes) *h2d_bytes = h2d;
    if (d2h_bytes) *d2h_bytes = d2h;
    return e;
}

}  // extern "C"
