// pf_eval.cu -- the block-synchronous evaluation kernel of the fast tier
// (restricted facets, generalized-polygon integrals, interior point, patch
// areas: pf_cell.cuh's eval_* phases), in its own translation unit so that it
// can be compiled with its own floating-point contraction setting (Makefile
// EVAL_FMAD; the build kernels and every tolerance predicate of the clip stay
// in pf_runtime.cu without FMA).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>

#include "pf_tiers.cuh"

using namespace pf;

// the cell kernels read their CellIn / CellOut parameters in place (param
// space) instead of from a local-memory copy (C4: 103.4 -> 100.4 ms)
#define PF_KPARAM const __grid_constant__

extern int pf_internal_set_err(const char *msg);
extern unsigned long long pf_internal_launches_add(unsigned long long k);

#ifndef PF_NO_TMA_LOAD
#define PF_NO_TMA_LOAD 0  // 1: the evaluation loads the polytope with lane loads instead of a bulk copy
#endif

namespace {
// Block-synchronous evaluation: blocks of SYNC_WARPS warps (2 per SM), one
// cell per warp per round; the warps run each phase of the evaluation
// together (__syncthreads between phases), so the SM's instruction caches
// hold one phase at a time instead of the whole ~90 KB of evaluation code
// (measured: the unsynchronised kernel spends half its stall samples on
// instruction fetch).
#ifndef PF_SYNC_WARPS
#define PF_SYNC_WARPS 8
#endif
#ifndef PF_SYNC_BLOCKS
#define PF_SYNC_BLOCKS 2
#endif
constexpr int SYNC_WARPS = PF_SYNC_WARPS;
constexpr int SYNC_BLOCKS = PF_SYNC_BLOCKS;  // blocks per SM
// EW: EWSN<FastCaps> (timed: no census code) or EWS<FastCaps> (the census pass)
template <class EW>
__global__ void __launch_bounds__(SYNC_WARPS * 32, SYNC_BLOCKS)
    k_cells_eval_sync(PF_KPARAM CellIn in, PF_KPARAM CellOut out, int count, const Poly<FastCaps> *__restrict__ gpoly,
                      const uint8_t *__restrict__ stage, int *__restrict__ retry_list,
                      int *__restrict__ counters, unsigned long long *__restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    EW *ws = (EW *)(smem + (size_t)wid * sizeof(EW));
    int fl = 0;
    const bool tma = !PF_NO_TMA_LOAD;
    unsigned phase = 0;
    if (tma && lane == 0) mbar_init(&ws->u.e.mbar);
    __syncwarp();
#ifndef PF_EVAL_PIPE_IDX
#define PF_EVAL_PIPE_IDX 1  // next round's cell index and stage byte loaded a round ahead
#endif
#ifndef PF_DYN_EVAL
#define PF_DYN_EVAL 1  // rounds handed out from a global counter (0: grid stride)
#endif
    // Rounds of SYNC_WARPS consecutive work items: with PF_DYN_EVAL each block
    // takes its next round from counters[3] (one round ahead, so the next
    // round's cells can be prefetched), and the kernel ends with the work, not
    // with the block whose fixed share was the heaviest.
    __shared__ int s_round;
    int base, nb;  // this round's and the next round's first work item
    if (PF_DYN_EVAL) {
        __shared__ int s_first[2];
        if (threadIdx.x == 0) {
            s_first[0] = atomicAdd(&counters[3], SYNC_WARPS);
            s_first[1] = atomicAdd(&counters[3], SYNC_WARPS);
        }
        __syncthreads();
        base = s_first[0];
        nb = s_first[1];
    } else {
        base = blockIdx.x * SYNC_WARPS;
        nb = base + gridDim.x * SYNC_WARPS;
    }
#ifndef PF_EARLY_TMA
#define PF_EARLY_TMA 1
#endif
    bool issued = false;  // this round's polytope load was issued at the end of the last round
    int i_nx = -1;  // this warp's next cell (or -1), loaded during the previous round
    if (PF_EVAL_PIPE_IDX) {
        const int t0 = base + wid;
        if (t0 < count) {
            const int i0 = in.cells ? in.cells[t0] : in.g.sid[t0];
            i_nx = stage[i0] == 1 ? i0 : -1;
        }
    }
    while (base < count) {
        const int t = base + wid;
        int i = -1;
        if (PF_EVAL_PIPE_IDX) {
            i = i_nx;
        } else if (t < count) {
            i = in.cells ? in.cells[t] : in.g.sid[t];
            if (stage[i] != 1) i = -1;
        }
        const bool act = i >= 0;
        {
            // next round's polytope into L2 while this round computes
            const int tn = nb + wid;
            i_nx = -1;
            if (tn < count) {
                const int inext = in.cells ? in.cells[tn] : in.g.sid[tn];
                const char *pp = (const char *)(gpoly + inext);
                const int nlines = (int)((sizeof(Poly<FastCaps>) + 127) / 128);
                if (lane < nlines) asm volatile("prefetch.global.L2 [%0];" ::"l"(pp + 128 * lane));
                if (PF_EVAL_PIPE_IDX) i_nx = stage[inext] == 1 ? inext : -1;
            }
        }
        double px = 0.0, py = 0.0, pz = 0.0, psi = 0.0;
        CellRes res;
        EvalState st;
        st.done = 1;
        if (act) {
            if (tma && PF_EARLY_TMA) {
                if (!issued) poly_load_tma_issue(gpoly + i, ws->P[0], &ws->u.e.mbar);
                poly_load_tma_wait(&ws->u.e.mbar, phase);
            } else if (tma) {
                poly_load_tma(gpoly + i, ws->P[0], &ws->u.e.mbar, phase);
            } else {
                poly_load(gpoly + i, ws->P[0]);
            }
            if (lane == 0) {
                ws->oflow = 0;
                ws->strict = in.strict;
                ws->cen_on = out.census16 != nullptr;
                if (EW::CEN)
                    for (int k = 0; k < 16; k++) ws->cen[k] = out.census16 ? out.census16[(size_t)i * 16 + k] : 0;
            }
            __syncwarp();
            px = in.pts[3 * i]; py = in.pts[3 * i + 1]; pz = in.pts[3 * i + 2];
            psi = in.psi[i];
            eval_setup(ws, ws->P[0], px, py, pz, psi, in.tol, &res, &st);
        }
        __syncthreads();
        if (!st.done) eval_restrict(ws, ws->P[0], px, py, pz, psi, in.tol, &res, &st);
        __syncthreads();
        if (!st.done) eval_integrals(ws, ws->P[0], px, py, pz, psi, in.tol, in.want_m2, &res, &st);
        __syncthreads();
        if (!st.done) eval_interior(ws, ws->P[0], px, py, pz, psi, in.tol, &res, &st);
        for (int a = 0; a < 4; a++) {
            const bool need = !st.done && st.attempt < 4;
            if (!__syncthreads_or(need)) break;
            if (need) eval_patch_attempt(ws, ws->P[0], px, py, pz, psi, in.tol, &res, &st);
        }
        __syncthreads();
        if (!st.done) eval_final(ws, ws->P[0], px, py, pz, psi, in.want_m2, &res, &st);
        if (act) {
            const int r = eval_write(ws, in, out, i, 0, res);
            if (r & FLAG_RETRY) {
                if (lane == 0) retry_list[atomicAdd(&counters[0], 1)] = i;
            } else {
                cell_finish(ws, out, i, r);
                fl |= r & 7;
            }
        }
        // the next round's polytope, issued as soon as this warp is done with
        // the buffer: the copy overlaps the round's barrier and the next setup
        issued = false;
        if (tma && PF_EARLY_TMA && PF_EVAL_PIPE_IDX && i_nx >= 0) {
            poly_load_tma_issue(gpoly + i_nx, ws->P[0], &ws->u.e.mbar);
            issued = true;
        }
        if (PF_DYN_EVAL && threadIdx.x == 0) s_round = atomicAdd(&counters[3], SYNC_WARPS);  // the round after next
        __syncthreads();
        base = nb;
        nb = PF_DYN_EVAL ? s_round : nb + gridDim.x * SYNC_WARPS;
    }
    if (lane == 0 && fl) atomicOr(err, (unsigned long long)fl);
}

}  // namespace

int pf_internal_eval_sync_attr() {
    static_assert(sizeof(EWSN<FastCaps>) == sizeof(EWS<FastCaps>), "one launch shape for both evaluation kernels");
    cudaError_t e = cudaSuccess;
    for (const void *kf : {(const void *)k_cells_eval_sync<EWSN<FastCaps>>, (const void *)k_cells_eval_sync<EWS<FastCaps>>}) {
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SYNC_WARPS * sizeof(EWS<FastCaps>)));
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    if (e != cudaSuccess) {
        char b[256];
        snprintf(b, sizeof b, "pf_eval.cu: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        return pf_internal_set_err(b);
    }
    return 0;
}

int pf_internal_eval_sync(const CellIn &in, const CellOut &out, int count, const Poly<FastCaps> *gpoly,
                          const uint8_t *stage, int *retry_list, int *counters, unsigned long long *err, int nsm,
                          cudaStream_t st) {
    const int64_t sb = std::min<int64_t>((int64_t)nsm * SYNC_BLOCKS, (count + SYNC_WARPS - 1) / SYNC_WARPS);
    if (sb <= 0) return 0;
    auto ke = out.census16 ? k_cells_eval_sync<EWS<FastCaps>> : k_cells_eval_sync<EWSN<FastCaps>>;
    ke<<<(int)sb, SYNC_WARPS * 32, SYNC_WARPS * sizeof(EWS<FastCaps>), st>>>(in, out, count, gpoly, stage, retry_list,
                                                                             counters, err);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        char b[256];
        snprintf(b, sizeof b, "pf_eval.cu: k_cells_eval_sync: %s", cudaGetErrorString(e));
        return pf_internal_set_err(b);
    }
    return 0;
}
