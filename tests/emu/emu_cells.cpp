// emu_cells.cpp -- TEST INFRASTRUCTURE ONLY: runs the device cell algorithm
// (paper_2601_05765_b200/csrc/pf_cell.cuh) on the host under the lock-step
// warp emulator of emu_warp.h.  Loaded only by tests/test_emu_cells.py to
// check the warp-cooperative logic against the oracle on CPU.  It is never
// loaded by the product package, bench.py or smoke().
#define PF_EMU 1
#include "emu_warp.h"
#include "pf_tiers.cuh"

#include <algorithm>
#include <vector>

asm(R"(
.text
.globl emu_swap
.type emu_swap,@function
emu_swap:
    pushq %rbp
    pushq %rbx
    pushq %r12
    pushq %r13
    pushq %r14
    pushq %r15
    movq %rsp, (%rdi)
    movq %rsi, %rsp
    popq %r15
    popq %r14
    popq %r13
    popq %r12
    popq %rbx
    popq %rbp
    ret
)");

namespace pfw {
thread_local EmuWarp *g_w = nullptr;
thread_local int g_lane = 0;

static void fiber_entry() {
    EmuWarp *w = g_w;
    int l = g_lane;
    w->fn(w->ctx, l);
    w = g_w;  // same warp; re-read after the user function
    w->done[g_lane] = true;
    w->kind[g_lane] = K_NONE;
    emu_swap(&w->lane_sp[g_lane], w->sched_sp);
    abort();  // never resumed
}

EmuWarp *emu_new_warp(size_t stack_size) {
    EmuWarp *w = (EmuWarp *)calloc(1, sizeof(EmuWarp));
    w->stack_size = stack_size;
    w->stacks = (char *)malloc(stack_size * 32);
    return w;
}

void emu_free_warp(EmuWarp *w) {
    free(w->stacks);
    free(w);
}

static inline uint64_t xs(uint64_t &s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

int emu_run_warp(EmuWarp *w, void (*fn)(void *, int), void *ctx, uint64_t seed) {
    w->fn = fn;
    w->ctx = ctx;
    w->rng = seed ? seed : 88172645463325252ull;
    w->error = 0;
    for (int l = 0; l < 32; l++) {
        w->done[l] = false;
        w->kind[l] = K_NONE;
        w->epoch[l] = 0;
        uintptr_t sp = (uintptr_t)(w->stacks + (size_t)(l + 1) * w->stack_size);
        sp &= ~(uintptr_t)15;
        sp -= 8;
        *(uint64_t *)sp = 0;
        sp -= 8;
        *(void **)sp = (void *)&fiber_entry;
        for (int r = 0; r < 6; r++) {
            sp -= 8;
            *(uint64_t *)sp = 0;
        }
        w->lane_sp[l] = (void *)sp;
    }
    EmuWarp *saved_w = g_w;
    int saved_lane = g_lane;
    int order[32];
    for (int l = 0; l < 32; l++) order[l] = l;
    for (;;) {
        // shuffled resume order per epoch
        for (int l = 31; l > 0; l--) {
            int r = (int)(xs(w->rng) % (uint64_t)(l + 1));
            std::swap(order[l], order[r]);
        }
        int alive = 0;
        for (int t = 0; t < 32; t++) {
            int l = order[t];
            if (w->done[l]) continue;
            g_w = w;
            g_lane = l;
            emu_swap(&w->sched_sp, w->lane_sp[l]);
        }
        int kind0 = -1;
        long ep0 = -1;
        int ndone = 0;
        for (int l = 0; l < 32; l++) {
            if (w->done[l]) { ndone++; continue; }
            alive++;
            if (kind0 < 0) { kind0 = w->kind[l]; ep0 = w->epoch[l]; }
            else if (w->kind[l] != kind0 || w->epoch[l] != ep0) w->error = 2;  // divergent collectives
        }
        if (alive == 0) break;
        if (ndone > 0) { w->error = 3; break; }  // some lanes exited while others wait at a collective
        if (w->error) break;
        w->n_collectives++;
    }
    g_w = saved_w;
    g_lane = saved_lane;
    return w->error;
}
}  // namespace pfw

namespace {

template <class C>
struct Job {
    pf::WS<C> *ws;
    const pf::CellIn *in;
    const pf::CellOut *out;
    int cell;
    int result;
};

template <class C>
void lane_fn(void *ctx, int lane) {
    Job<C> *j = (Job<C> *)ctx;
    int r = pf::run_cell(j->ws, *j->in, *j->out, j->cell);
    if (lane == 0) j->result = r;
}

}  // namespace

static const int *g_only = nullptr;  // optional cell subset (debugging)
static int g_nonly = 0;
static int g_strict = 0;  // parity mode (CellIn::strict)

extern "C" {

void pfemu_set_strict(int on) { g_strict = on != 0; }

void pfemu_set_cells(const int *cells, int ncells) {
    g_only = cells;
    g_nonly = ncells;
}

// Build the bucket-sorted SoA grid exactly as the device grid build does
// (stable counting sort by bucket id) and run every cell through the fast
// tier, then the mid and exact tiers for retries.  tier: 0 = fast->mid->exact,
// 1 = exact only, 2 = mid->exact.
int64_t pfemu_evaluate(int n, const double *pts, const double *psi,
                       const double *dv, int dnv, const double *dp, const int *dt, int dnf,
                       const int *dlp, const int *dlv, int dnl,
                       double glo0, double glo1, double glo2, double gih0, double gih1, double gih2,
                       int gn0, int gn1, int gn2, double tol, double dpsi, int ball_aware,
                       int want_m2, int smf, double t_init,
                       int64_t *status, double *vol, double *ksur, double *cent, double *ipt,
                       double *m2, int64_t *fcount, int64_t *ftag, double *farea, double *fh,
                       double *fnrm, double *fcent, int *flags, int *census, int tier,
                       uint64_t seed, int *n_retry, long *n_coll) {
    using namespace pf;
    const double lo[3] = {glo0, glo1, glo2}, ih[3] = {gih0, gih1, gih2};
    const int gn[3] = {gn0, gn1, gn2};
    const int ncell = gn0 * gn1 * gn2;
    std::vector<int> bid(n), bstart(ncell + 1, 0), sid(n);
    std::vector<double> sx(n), sy(n), sz(n);
    for (int i = 0; i < n; i++) {
        int b[3];
        for (int a = 0; a < 3; a++) b[a] = bucket_coord(pts[3 * i + a], lo[a], ih[a], gn[a]);
        bid[i] = (b[0] * gn1 + b[1]) * gn2 + b[2];
        bstart[bid[i] + 1]++;
    }
    for (int c = 0; c < ncell; c++) bstart[c + 1] += bstart[c];
    {
        std::vector<int> fill(bstart.begin(), bstart.end() - 1);
        for (int i = 0; i < n; i++) {
            int s = fill[bid[i]]++;
            sid[s] = i;
            sx[s] = pts[3 * i];
            sy[s] = pts[3 * i + 1];
            sz[s] = pts[3 * i + 2];
        }
    }
    CellIn in;
    memset(&in, 0, sizeof(in));
    in.pts = pts; in.psi = psi; in.n = n;
    in.g.sx = sx.data(); in.g.sy = sy.data(); in.g.sz = sz.data(); in.g.sid = sid.data();
    in.g.bstart = bstart.data();
    for (int a = 0; a < 3; a++) { in.g.lo[a] = lo[a]; in.g.ih[a] = ih[a]; in.g.gn[a] = gn[a]; }
    in.dv = dv; in.dp = dp; in.dt = dt; in.dlp = dlp; in.dlv = dlv;
    in.dnv = dnv; in.dnf = dnf; in.dnl = dnl;
    in.tol = tol; in.dpsi = dpsi; in.ball_aware = ball_aware; in.want_m2 = want_m2;
    in.t_init = t_init;
    in.strict = g_strict;
    // per super-bucket max weight, as pf_runtime.cu's k_super_max (PF_SUPER = 4)
    std::vector<double> smax, cslack;
    if (ball_aware && !getenv("PF_GLOBAL_SLACK")) {
        const int f = 4, G[3] = {gn0, gn1, gn2};
        for (int a = 0; a < 3; a++) in.g.sgn[a] = (G[a] + f - 1) / f;
        in.g.sf = f;
        smax.assign((size_t)in.g.sgn[0] * in.g.sgn[1] * in.g.sgn[2], -1e300);
        for (int ix = 0; ix < gn0; ix++)
            for (int iy = 0; iy < gn1; iy++)
                for (int iz = 0; iz < gn2; iz++) {
                    const int b = (ix * gn1 + iy) * gn2 + iz;
                    double &m = smax[((ix / f) * in.g.sgn[1] + iy / f) * in.g.sgn[2] + iz / f];
                    for (int s = bstart[b]; s < bstart[b + 1]; s++) m = std::max(m, psi[sid[s]]);
                }
        in.g.smax = smax.data();
        cslack.resize(n);
        for (int i = 0; i < n; i++) cslack[i] = cell_slack(in.g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], psi[i], dpsi);
        in.cslack = cslack.data();
    }
    // full mode: the heaviest sites (pf_runtime.cu launch_cells, PF_HEAVY = 8)
    std::vector<int> hv_idx;
    std::vector<double> hv_psi;
    if (!ball_aware && n > 0 && !getenv("PF_NO_HEAVY")) {
        std::vector<int> o(n);
        for (int i = 0; i < n; i++) o[i] = i;
        std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return psi[a] > psi[b]; });
        const int nh = std::min(8, n);
        hv_idx.assign(o.begin(), o.begin() + nh);
        for (int k = 0; k < nh; k++) hv_psi.push_back(psi[o[k]]);
        hv_psi.push_back(n > nh ? psi[o[nh]] : -1e300);
        in.heavy_idx = hv_idx.data();
        in.heavy_psi = hv_psi.data();
        in.nheavy = nh;
    }
    CellOut out;
    memset(&out, 0, sizeof(out));
    out.status = status; out.vol = vol; out.ksur = ksur; out.cent = cent; out.ipt = ipt; out.m2 = m2;
    out.fcount = fcount; out.ftag = ftag; out.farea = farea; out.fh = fh; out.fnrm = fnrm;
    out.fcent = fcent; out.smf = smf; out.flags = flags; out.census = census;

    int64_t err_all = 0;
    int retries = 0;
    long ncoll = 0;
    int emu_error = 0;
#pragma omp parallel reduction(| : err_all) reduction(+ : retries, ncoll) reduction(max : emu_error)
    {
        pfw::EmuWarp *w = pfw::emu_new_warp(1 << 18);
        WS<FastCaps> *wsf = (WS<FastCaps> *)aligned_alloc(64, (sizeof(WS<FastCaps>) + 63) / 64 * 64);
        WS<ExactCaps> *wse = (WS<ExactCaps> *)aligned_alloc(64, (sizeof(WS<ExactCaps>) + 63) / 64 * 64);
        WS<MidCaps> *wsm = (WS<MidCaps> *)aligned_alloc(64, (sizeof(WS<MidCaps>) + 63) / 64 * 64);
        const int nk = g_only ? g_nonly : n;
#pragma omp for schedule(dynamic, 4)
        for (int k = 0; k < nk; k++) {
            int i = g_only ? g_only[k] : sid[k];  // cells processed in bucket order, as on the device
            int r = FLAG_RETRY;
            if (tier == 0) {
                Job<FastCaps> job{wsf, &in, &out, i, 0};
                int e = pfw::emu_run_warp(w, lane_fn<FastCaps>, &job, seed + (uint64_t)i * 7919u);
                if (e > emu_error) emu_error = e;
                r = job.result;
            }
            if (tier == 0 && (r & FLAG_RETRY)) retries++;
            if ((r & FLAG_RETRY) && tier != 1) {
                Job<MidCaps> job{wsm, &in, &out, i, 0};
                int e = pfw::emu_run_warp(w, lane_fn<MidCaps>, &job, seed + (uint64_t)i * 31337u);
                if (e > emu_error) emu_error = e;
                r = job.result;
            }
            if (r & FLAG_RETRY) {
                Job<ExactCaps> job{wse, &in, &out, i, 0};
                int e = pfw::emu_run_warp(w, lane_fn<ExactCaps>, &job, seed + (uint64_t)i * 104729u);
                if (e > emu_error) emu_error = e;
                r = job.result;
            }
            err_all |= (r & 7);
        }
        ncoll += w->n_collectives;
        free(wsf);
        free(wse);
        free(wsm);
        pfw::emu_free_warp(w);
    }
    if (n_retry) *n_retry = retries;
    if (n_coll) *n_coll = ncoll;
    if (emu_error) return -1000 - emu_error;
    return err_all;
}

int pfemu_ws_bytes(int tier) {
    return tier == 0 ? (int)sizeof(pf::WS<pf::FastCaps>) : (int)sizeof(pf::WS<pf::ExactCaps>);
}
}
