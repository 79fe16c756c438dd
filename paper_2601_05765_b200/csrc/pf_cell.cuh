// pf_cell.cuh -- warp-per-cell construction + analytic evaluation of one
// generalized Laguerre cell (power cell of site i restricted to the ball
// B(p_i, sqrt(psi_i))).
//
// One warp owns one cell.  The convex polytope lives in shared memory in the
// reference's primal packed layout (vertices, facet planes, tags, CCW vertex
// loops; _kernels.py:10-18) so that every vertex is produced by the same
// arithmetic as the reference clip (_kernels.py:188-191) and every
// tolerance-deciding predicate sees the same bits.  Compiled with
// --fmad=false, the build phase and all predicates are bit-identical to the
// reference; only the transcendentals (atan2/sin/cos) differ in the last ulp.
//
// Work distribution inside the warp:
//   * candidate gather  : lanes stride over the flattened z-runs of the grid
//                         buckets that can hold a site within the stop radius
//   * candidate order   : rank sort on the key (d^2, j) (_kernels.py:1293-1304)
//   * clip (A7)         : lane per vertex (classify / keep, ballot-prefix
//                         compaction), lane per facet (walk, crossing entries),
//                         lane per crossing entry (dedup + new vertex), lane per
//                         new-facet vertex (atan2 angle + rank sort)
//   * evaluate (A9-A13) : lane per facet (restriction walk, generalized polygon
//                         integrals, ray for the interior point, Gauss-Bonnet
//                         patch area); order-dependent sums are done by every
//                         lane redundantly over shared memory in the
//                         reference's facet order, so results are deterministic
//                         and independent of scheduling.
#pragma once
#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "pf_warp.cuh"

namespace pf {

// _kernels.py:29-50
enum { CLIP_CUT = 0, CLIP_UNTOUCHED = 1, CLIP_EMPTY = 2, CLIP_OVERFLOW = 3, CLIP_DEGENERATE = 4 };
enum { RF_OUTSIDE = 0, RF_UNTOUCHED = 1, RF_FULLCIRCLE = 2, RF_GENPOLY = 3 };
enum { CELL_EMPTY = 0, CELL_FULLBALL = 1, CELL_CLIPPED = 2 };
enum { FLAG_OVERFLOW = 1, FLAG_DEGENERATE_INTERIOR = 2, FLAG_UNSTABLE_PROJECTION = 4 };
// internal: a capacity of this (small, shared-memory) instantiation was
// exceeded; the cell is queued for the reference-capacity instantiation.
enum { FLAG_RETRY = 256 };
// per-cell flag only: the Laguerre cell itself overflowed (build status 3);
// the reference then writes status/vol/ksur/fcount but not cent/ipt/m2
enum { FLAG_BUILD_OVERFLOW = 512 };

#define PF_PI 3.141592653589793
#define PF_FOUR_PI (4.0 * PF_PI)

// reference capacities (_kernels.py:24-27)
enum { REF_MAX_V = 512, REF_MAX_F = 160, REF_MAX_L = 2048, REF_MAX_P = 256 };

// Capacity set of one instantiation.  EXACT=true means the reference's own
// capacities: overflow then reproduces the reference's CLIP_OVERFLOW outcome.
template <int CV_, int CF_, int CL_, int CC_, int CE_, int CP_, bool EXACT_>
struct Caps {
    static constexpr int CV = CV_;  // vertices
    static constexpr int CF = CF_;  // facets
    static constexpr int CL = CL_;  // loop entries
    static constexpr int CC = CC_;  // candidates per shell
    static constexpr int CE = CE_;  // crossing entries per clip
    static constexpr int CP = CP_;  // restricted boundary points per cell
    static constexpr bool EXACT = EXACT_;
};

template <class C>
struct Poly {
    double x[C::CV], y[C::CV], z[C::CV];
    double nx[C::CF], ny[C::CF], nz[C::CF], d[C::CF];
    int tag[C::CF];
    uint16_t lp[C::CF + 1];
    uint16_t lv[C::CL];
    int nv, nf, nl;
};

template <class C>
struct BuildScratch {
    double sd[C::CV];          // signed distances, reused for new-facet angles
    uint16_t vmap[C::CV];      // kept index / referenced map
    uint16_t onl[C::CV];       // new-facet vertex list (B indices, increasing)
    int fk[C::CF];             // emitted loop length per facet
    uint16_t fscan0[C::CF];    // emitted-entry scan value at the facet's first entry
    uint16_t flb[C::CF];       // output loop base per facet (0xffff = dropped)
    uint16_t fout[C::CF];      // output facet index
    uint16_t ea[C::CE], eb[C::CE], eid[C::CE];  // crossing entries (walk order)
    uint16_t emt[C::CE];       // first-occurrence entry of the same edge
    uint8_t ecls[C::CL];       // per loop entry of A: bit0 tail inside, bit1 crossing edge
    uint8_t lf[2][C::CL];      // facet of each loop entry, per polytope buffer
    union {                    // phase-disjoint scratch (shared memory is the occupancy limit)
        struct {               // clip steps 3a-3e
            uint16_t epos[C::CL];  // per loop entry of A: emitted entries before it (all facets)
            typename std::conditional<(C::CE < 256), uint8_t, uint16_t>::type cpos[C::CL];  // its crossing entry
        };
        struct {               // clip step 4
            double sy[C::CV];      // new-facet vertex ordinates (abscissae in sd)
            uint8_t half[C::CV];   // their half-plane (angle order, see ang_lt)
        };
        struct {               // gather_shell
            int run_start[32], run_off[32];  // per column: first run, offset in the batch
            int run_la[32], run_stb[32];      // length of the first run, start of the second
        };
    };
    double cd2[C::CC];         // candidates (d^2, j), sorted
    int cj[C::CC];
    uint16_t cord[C::CC];      // sorted rank -> gather slot of the candidate data below
    double cx[C::CC], cy[C::CC], cz[C::CC], cw[C::CC];  // position and weight, by gather slot
    int ncand;
};

template <class C>
struct alignas(16) EvalScratch {  // 16-byte multiple: the evaluation workspaces stay TMA-aligned
    unsigned long long mbar;  // per-warp mbarrier of the polytope's bulk (TMA) load (k_cells_eval_sync)
    // per facet
    double fh[C::CF], frc[C::CF], farea[C::CF], fcx[C::CF], fcy[C::CF], fcz[C::CF], fip[C::CF];
    double fpa[C::CF];       // Gauss-Bonnet sum, then the projected (occluded) patch area
    double fe[6][C::CF];     // facet-circle frame (perp_basis); later the interior-point rays
    int16_t fhead[C::CF + 1], fnp[C::CF];  // boundary ring = pool[fhead, fhead + fnp)
    uint8_t fkind[C::CF], fseg[C::CF], funs[C::CF], fmrg[C::CF];
    uint8_t vin[C::CV];
    // twin-facet lookup (replaces the reference's O(nf m) _edge_other_facet scan)
    uint8_t vdeg[C::CV];            // outgoing loop entries per vertex
    uint16_t vinc[C::CV * 4];       // their entry indices (first 4)
    uint8_t efac[C::CL];            // facet of each loop entry
    uint16_t esv[C::CL];            // successor vertex of each loop entry
    // point pool: the facets' boundary rings, contiguous per facet, walk order
    double ppx[C::CP], ppy[C::CP], ppz[C::CP];
    double prx[C::CP], pry[C::CP], prz[C::CP];  // central projections from the interior point
    uint8_t pfl[C::CP];   // PF_ONSPH / PF_CONN (arc to next) / PF_DEL / PF_ENTRY
    uint8_t pfac[C::CP];  // facet of the point (PF_DEAD: freed by a merge)
    int npool;
};

// per-warp workspaces.  WS: both phases (fused and reference-capacity
// kernels); BWS / EWS: what the split build / evaluate kernels need.
template <class C_, int NP, class U, bool CEN_ = true>
struct alignas(16) WSX {  // 16-byte multiple: every warp's polytope stays TMA-aligned
    using Cap = C_;
    static constexpr bool CEN = CEN_;  // census code compiled in (the timed kernels leave it out)
    Poly<C_> P[NP];
    U u;
    // one word of per-cell flags: the build workspace is sized to the byte
    // (24 warps x 9600 B fill the SM's shared memory exactly)
    uint8_t oflow;   // capacity overflow seen by any lane
    uint8_t strict;  // parity mode (CellIn::strict) for this cell
    uint8_t cen_on;  // census requested for this cell
    uint8_t pad_;
    int cen[16];  // algorithmic-work census (SURVEY.md §8(d) S_cell terms)
};
template <class C> union BEU { BuildScratch<C> b; EvalScratch<C> e; };
template <class C> struct BU { BuildScratch<C> b; };
template <class C> struct EU { EvalScratch<C> e; };
template <class C> using WS = WSX<C, 2, BEU<C>>;
template <class C> using BWS = WSX<C, 2, BU<C>>;
template <class C> using EWS = WSX<C, 1, EU<C>>;
// the same without the census code: the split kernels' timed instantiations
template <class C> using BWSN = WSX<C, 2, BU<C>, false>;
template <class C> using EWSN = WSX<C, 1, EU<C>, false>;
// census requested for this cell (never, where the workspace leaves it out)
template <class W>
PF_DEV bool cen_on(const W *ws) { return W::CEN && ws->cen_on; }


// census slots:
enum {
    CEN_CLIPS = 0, CEN_TESTS, CEN_NEWV, CEN_NFV, CEN_RFAR, CEN_CUTS, CEN_LOOP, CEN_CROSS,
    CEN_RFAC, CEN_RFAC_NF, CEN_SEG, CEN_ARC, CEN_BPTS, CEN_PROJ, CEN_FULLC, CEN_GATH, CEN_N
};

// ---------------------------------------------------------------------------
// inputs / outputs of the cell kernels
// ---------------------------------------------------------------------------
struct GridView {
    const double *sx, *sy, *sz;  // sites in bucket order (SoA)
    const int *sid;              // original index of sorted slot
    const int *bstart;           // [ncell + 1]
    double lo[3], ih[3];
    int gn[3];
    // per super-bucket (sf^3 buckets) maximum weight, or null: bounds the
    // weights near a site for its security radius (build_cell)
    const double *smax;
    int sgn[3], sf;
};

struct CellIn {
    const double *pts;  // [n, 3] original order
    const double *psi;  // [n]
    int n;
    GridView g;
    // domain pack (reference layout, int32 indices)
    const double *dv;
    const double *dp;
    const int *dt, *dlp, *dlv;
    int dnv, dnf, dnl;
    double tol, dpsi;
    const double *dpsi_ptr;  // when set, dpsi is read from device memory
    int ball_aware, want_m2;
    int strict;     // parity mode: the reference's restriction outcomes bit for bit
    double t_init;  // first shell radius^2 when not ball-aware
    const double *cslack;  // optional: per-cell weight slack (cell_slack), ball-aware only
    // optional, full (non-ball-aware) mode: the PF_HEAVY heaviest sites
    // (indices, weights in descending order) and, in heavy_psi[nheavy], the
    // largest weight of all other sites (build_cell: heavy-site phase)
    const int *heavy_idx;
    const double *heavy_psi;
    int nheavy;
    const int *cells;  // optional: evaluate only these cells (original indices)
    int ncells;
};

struct CellOut {
    // fixed-stride reference outputs (any pointer may be null)
    int64_t *status;
    double *vol, *ksur, *cent, *ipt, *m2;
    int64_t *fcount, *ftag;
    double *farea, *fh, *fnrm, *fcent;
    int smf;
    // lean outputs for the Newton solver (may be null)
    int *ftag32;    // [n, smf]
    int *fcount32;  // [n]
    int *flags;     // [n] per-cell flag word (incl. FLAG_RETRY)
    int *census;    // [n] processed candidates (clips attempted)
    int *census16;  // [n, 16] full census (CEN_*), optional
    // unrestricted packed cells (_batch_build, _kernels.py:1481-1559): when
    // pk_status is set the build writes these and no evaluation follows
    int64_t *pk_status, *pk_nv, *pk_nf, *pk_nl, *pk_tags, *pk_lp, *pk_lv;
    double *pk_verts, *pk_planes;
    int smv, smfb, sml;
};

PF_DEV double sq(double x) { return x * x; }
// the evaluation's phases and their single-call-site helpers inlined into the
// kernel (each has one call site per kernel, so the code does not grow; the
// phase-synchronous kernel keeps its instruction-cache footprint): C4
// evaluation 41.4 -> 38.0 ms.  PF_EVAL_INL=0: out of line.
#ifndef PF_EVAL_INL
#define PF_EVAL_INL 1
#endif
#if PF_EVAL_INL
#define PF_PHASE PF_DEV
#else
#define PF_PHASE PF_NOINL
#endif
// one out-of-line copy of the (long) double-precision atan2
// atan2 and the evaluation's multi-call-site helpers inline (C4 evaluation
// 34.1 -> 29.4 ms: the calls' register save/restore and the local-memory
// argument traffic cost more than the larger code)
#ifndef PF_ATAN2_INL
#define PF_ATAN2_INL 1
#endif
#if PF_ATAN2_INL
PF_DEV double atan2_ool(double y, double x) { return atan2(y, x); }
#else
PF_NOINL double atan2_ool(double y, double x) { return atan2(y, x); }
#endif
// Branch-free atan2 for the value-only angles of the evaluation (arc sweeps,
// Gauss-Bonnet turning angles): one division (the ratio, or its pi/4-reduced
// form (mn - mx) / (mn + mx) when above tan(pi/8)) and a degree-10 polynomial
// in t^2 (Chebyshev interpolant of atan(t)/t on [0, tan^2(pi/8)], 7e-17
// relative); quadrant by selects, sign from y (so t < 0 tests and -0 behave as
// atan2).  Within ~2 ulp of the library atan2, which keeps its branches for
// the lanes' different quadrants; zeros / inf / nan go to the library.  The
// wrap decisions of near-coincident arc end points keep the library atan2.
#ifndef PF_FAST_ATAN2
#define PF_FAST_ATAN2 1
#endif
PF_DEV double atan2_val(double y, double x) {
#if PF_FAST_ATAN2
    const double ax = fabs(x), ay = fabs(y);
    const double mx = fmax(ax, ay), mn = fmin(ax, ay);
    if (!(mx > 0.0) || !(mx < 1e300)) return atan2(y, x);
    const bool red = mn > 0.41421356237309503 * mx;
    const double t = (red ? mn - mx : mn) / (red ? mn + mx : mx);
    const double z = t * t;
    double p = 0.021135373157693246;
    p = fma(p, z, -0.04348052215716462);
    p = fma(p, z, 0.056883492268090106);
    p = fma(p, z, -0.06640233930429408);
    p = fma(p, z, 0.07689953496306857);
    p = fma(p, z, -0.09090773074808414);
    p = fma(p, z, 0.11111106180455946);
    p = fma(p, z, -0.14285714180976467);
    p = fma(p, z, 0.1999999999885511);
    p = fma(p, z, -0.3333333333332844);
    p = fma(p * z, t, t) + (red ? 0.78539816339744831 : 0.0);
    if (ay > ax) p = 1.5707963267948966 - p;
    if (x < 0.0) p = 3.1415926535897931 - p;
    return copysign(p, y);
#else
    return atan2_ool(y, x);
#endif
}
#ifndef PF_HELPER_INL
#define PF_HELPER_INL 1
#endif
#if PF_HELPER_INL
#define PF_HELPER PF_DEV
#else
#define PF_HELPER PF_NOINL
#endif
// IEEE division / square root inline (PF_MATH_INL=0: one out-of-line copy
// each; inline measured faster once the evaluation phases were inlined: C4
// evaluation 38.0 -> 36.7 ms)
#ifndef PF_MATH_INL
#define PF_MATH_INL 1
#endif
#if PF_MATH_INL
PF_DEV double ddiv(double a, double b) { return a / b; }
PF_DEV double dsqrt(double x) { return sqrt(x); }
#else
PF_NOINL double ddiv(double a, double b) { return a / b; }
PF_NOINL double dsqrt(double x) { return sqrt(x); }
#endif

// _kernels.py:59-80
PF_DEV void perp_basis_inl(double nx, double ny, double nz, double *e) {
    double ax = fabs(nx), ay = fabs(ny), az = fabs(nz);
    double ux, uy, uz;
    if (ax <= ay && ax <= az) { ux = 1.0; uy = 0.0; uz = 0.0; }
    else if (ay <= az) { ux = 0.0; uy = 1.0; uz = 0.0; }
    else { ux = 0.0; uy = 0.0; uz = 1.0; }
    double e1x = uy * nz - uz * ny;
    double e1y = uz * nx - ux * nz;
    double e1z = ux * ny - uy * nx;
    double inv = 1.0 / sqrt(e1x * e1x + e1y * e1y + e1z * e1z);
    e1x *= inv; e1y *= inv; e1z *= inv;
    e[0] = e1x; e[1] = e1y; e[2] = e1z;
    e[3] = ny * e1z - nz * e1y;
    e[4] = nz * e1x - nx * e1z;
    e[5] = nx * e1y - ny * e1x;
}
PF_HELPER void perp_basis(double nx, double ny, double nz, double *e) { perp_basis_inl(nx, ny, nz, e); }

template <class C>
PF_DEV void load_domain(Poly<C> &A, const CellIn &in) {
    const int L = pfw::lane();
    #pragma unroll 1
    for (int v = L; v < in.dnv; v += 32) {
        A.x[v] = in.dv[3 * v]; A.y[v] = in.dv[3 * v + 1]; A.z[v] = in.dv[3 * v + 2];
    }
    #pragma unroll 1
    for (int f = L; f < in.dnf; f += 32) {
        A.nx[f] = in.dp[4 * f]; A.ny[f] = in.dp[4 * f + 1]; A.nz[f] = in.dp[4 * f + 2];
        A.d[f] = in.dp[4 * f + 3];
        A.tag[f] = in.dt[f];
    }
    #pragma unroll 1
    for (int f = L; f <= in.dnf; f += 32) A.lp[f] = (uint16_t)in.dlp[f];
    #pragma unroll 1
    for (int k = L; k < in.dnl; k += 32) A.lv[k] = (uint16_t)in.dlv[k];
    if (L == 0) { A.nv = in.dnv; A.nf = in.dnf; A.nl = in.dnl; }
    pfw::sync();
}

// angle order of atan2(y, x) on (-pi, pi] without evaluating it: lower
// half-plane (including -pi = atan2(-0, x<0)) first, then orientation
PF_DEV int half_of(double x, double y) { return (y < 0.0 || (y == 0.0 && x < 0.0 && signbit(y))) ? 0 : 1; }
PF_DEV bool ang_lt(double xu, double yu, double xv, double yv) {
    const int hu = half_of(xu, yu), hv = half_of(xv, yv);
    if (hu != hv) return hu < hv;
    const double cr = xu * yv - yu * xv;
    if (cr != 0.0) return cr > 0.0;
    if (xu * xv + yu * yv >= 0.0) return false;  // same direction: equal angles
    return xu > 0.0;  // 0 before pi in the upper half
}

// max_v |v - p|^2 and max_v |v - p| (the running "rfar" of _kernels.py:1230-1237, 1341-1354)
template <class C>
PF_DEV double poly_rfar2(const Poly<C> &A, double px, double py, double pz) {
    double m = 0.0;
    #pragma unroll 1
    for (int v = pfw::lane(); v < A.nv; v += 32) {
        double d2 = sq(A.x[v] - px) + sq(A.y[v] - py) + sq(A.z[v] - pz);
        if (d2 > m) m = d2;
    }
    return pfw::max_d_inl(m);
}
template <class C>
PF_DEV double poly_rfar(const Poly<C> &A, double px, double py, double pz) {
    return sqrt(poly_rfar2(A, px, py, pz));
}

// the clip's rare paths (more than 32 vertices, dropped vertices) as helper
// functions; out of line (PF_COLD_OOL=1) measured slower (C4 build 47.5 ->
// 51.1 ms, the calls' register traffic), so they are inlined
#ifndef PF_COLD_OOL
#define PF_COLD_OOL 0
#endif
#if PF_COLD_OOL
#define PF_COLD PF_NOINL
#else
#define PF_COLD PF_DEV
#endif
// clip step 1-2 for polytopes of more than 32 vertices (rare: out of line, so
// the common single-chunk path keeps its registers).  Returns CLIP_UNTOUCHED /
// CLIP_EMPTY, or -1 with *K and this lane's *rmax share.
template <class W>
PF_COLD int clip_classify_wide(W *ws, const Poly<typename W::Cap> &A, Poly<typename W::Cap> &B, double nx,
                               double ny, double nz, double dd, double tol, double px, double py, double pz,
                               int *K_out, double *rmax_out) {
    using C = typename W::Cap;
    BuildScratch<C> &S = ws->u.b;
    const int L = pfw::lane();
    const unsigned lt = pfw::lanemask_lt();
    const int nv = A.nv;
    int K = 0;
    double rmax = 0.0;
    int n_out = 0;
    #pragma unroll 1
    for (int v0 = 0; v0 < nv; v0 += 32) {
        int v = v0 + L;
        bool out = false;
        if (v < nv) {
            double sv = nx * A.x[v] + ny * A.y[v] + nz * A.z[v] - dd;
            S.sd[v] = sv;
            out = sv > tol;
        }
        n_out += pfw::popc(pfw::ballot(out));
    }
    if (n_out == 0) return CLIP_UNTOUCHED;
    if (nv - n_out == 0) return CLIP_EMPTY;
    pfw::sync();
    #pragma unroll 1
    for (int v0 = 0; v0 < nv; v0 += 32) {
        int v = v0 + L;
        bool keep = v < nv && S.sd[v] <= tol;
        unsigned m = pfw::ballot(keep);
        if (keep) {
            int idx = K + pfw::popc(m & lt);
            S.vmap[v] = (uint16_t)idx;
            const double ax = A.x[v], ay = A.y[v], az = A.z[v];
            B.x[idx] = ax; B.y[idx] = ay; B.z[idx] = az;
            const double d2 = sq(ax - px) + sq(ay - py) + sq(az - pz);
            if (d2 > rmax) rmax = d2;
        } else if (v < nv) {
            S.vmap[v] = 0xffff;
        }
        K += pfw::popc(m);
    }
    *K_out = K;
    *rmax_out = rmax;
    return -1;
}

// clip step 5 (_kernels.py:297-315): drop the vertices no loop references
// any more (rare: only after a dropped facet emitted 1-2 entries); returns
// the vertex count
template <class W>
PF_COLD int clip_drop_unreferenced(W *ws, Poly<typename W::Cap> &B, int NVB, int NL2) {
    using C = typename W::Cap;
    BuildScratch<C> &S = ws->u.b;
    const int L = pfw::lane();
    const unsigned lt = pfw::lanemask_lt();
    #pragma unroll 1
    for (int v = L; v < NVB; v += 32) S.vmap[v] = 0;
    pfw::sync();
    #pragma unroll 1
    for (int k = L; k < NL2; k += 32) S.vmap[B.lv[k]] = 1;
    pfw::sync();
    int nref = 0;
    #pragma unroll 1
    for (int v0 = 0; v0 < NVB; v0 += 32) {
        int v = v0 + L;
        nref += pfw::popc(pfw::ballot(v < NVB && S.vmap[v] == 1));
    }
    if (nref != NVB) {
        int base = 0;
        #pragma unroll 1
        for (int v0 = 0; v0 < NVB; v0 += 32) {
            int v = v0 + L;
            bool r = v < NVB && S.vmap[v] == 1;
            unsigned m = pfw::ballot(r);
            double x = 0, y = 0, z = 0;
            int dst = base + pfw::popc(m & lt);
            if (r) { x = B.x[v]; y = B.y[v]; z = B.z[v]; }
            pfw::sync();
            if (r) { B.x[dst] = x; B.y[dst] = y; B.z[dst] = z; S.vmap[v] = (uint16_t)(dst + 2); }
            base += pfw::popc(m);
            pfw::sync();
        }
        #pragma unroll 1
        for (int k = L; k < NL2; k += 32) B.lv[k] = (uint16_t)(S.vmap[B.lv[k]] - 2);
        nref = base;
    }
    return nref;
}

// ---------------------------------------------------------------------------
// clip A by n.x <= dd into B (_kernels.py:109-319), warp-cooperative
// ---------------------------------------------------------------------------
template <class W>
PF_DEV int clip(W *ws, const Poly<typename W::Cap> &A, Poly<typename W::Cap> &B, int wa, double nx,
                  double ny, double nz, double dd, int tag, double tol, double px, double py, double pz,
                  double *rfar2) {
    // *rfar2 (on CLIP_CUT): max_v |v - p|^2 over B's vertices, from the kept and
    // the new vertices as they are produced (the reference's rfar pass,
    // _kernels.py:1341-1354, same terms and order per vertex; -1 when a dropped
    // vertex makes a full pass necessary)
    using C = typename W::Cap;
    BuildScratch<C> &S = ws->u.b;
    const uint8_t *lfa = S.lf[wa];
    uint8_t *lfb = S.lf[1 - wa];
    const int L = pfw::lane();
    const unsigned lt = pfw::lanemask_lt();
    const int nv = A.nv, nf = A.nf;
    if (cen_on(ws) && L == 0) { ws->cen[CEN_CLIPS]++; ws->cen[CEN_TESTS] += nv; }

    // 1. classify vertices (_kernels.py:121-134) and 2. keep the inside
    // ones in order (_kernels.py:137-147); one pass when nv <= 32 (the signed
    // distance stays in a register for the on-plane test of step 4)
    int K = 0;
    double s_reg = 0.0;
    int vmap_reg = 0xffff;
    double rmax = 0.0;  // this lane's share of max |v - p|^2 over B's vertices
    if (nv <= 32) {
        const int v = L;
        if (v < nv) {
            s_reg = nx * A.x[v] + ny * A.y[v] + nz * A.z[v] - dd;
            S.sd[v] = s_reg;
        }
        const unsigned m_out = pfw::ballot(v < nv && s_reg > tol);
        if (m_out == 0) return CLIP_UNTOUCHED;
        if (pfw::popc(m_out) == nv) return CLIP_EMPTY;
        const bool keep = v < nv && s_reg <= tol;
        const unsigned m = pfw::ballot(keep);
        if (keep) {
            vmap_reg = pfw::popc(m & lt);
            const double ax = A.x[v], ay = A.y[v], az = A.z[v];
            B.x[vmap_reg] = ax; B.y[vmap_reg] = ay; B.z[vmap_reg] = az;
            rmax = sq(ax - px) + sq(ay - py) + sq(az - pz);
        }
        if (v < nv) S.vmap[v] = (uint16_t)vmap_reg;
        K = pfw::popc(m);
    } else {
        const int r = clip_classify_wide(ws, A, B, nx, ny, nz, dd, tol, px, py, pz, &K, &rmax);
        if (r >= 0) return r;
    }
    pfw::sync();

    // 3a. lane per loop entry (edge a -> b of facet f): classification,
    // crossing entries in walk order (= entry order) and the facet's emitted
    // loop length (_kernels.py:160-228); both prefix counts from ballots
    const int nl = A.nl;
    int NE = 0, NEm = 0;
    #pragma unroll 1
    for (int k0 = 0; k0 < nl; k0 += 32) {
        const int k = k0 + L;
        bool ina = false, cr = false;
        int f = 0, a = 0, b = 0;
        if (k < nl) {
            f = lfa[k];
            const int kn = k + 1 == A.lp[f + 1] ? A.lp[f] : k + 1;
            a = A.lv[k];
            b = A.lv[kn];
            const double sa = S.sd[a], sb = S.sd[b];
            const bool inb = sb <= tol;
            ina = sa <= tol;
            cr = ina ? (!inb && sa < -tol) : (inb && sb < -tol);
            S.ecls[k] = (uint8_t)((ina ? 1 : 0) | (cr ? 2 : 0));
        }
        // both prefix counts from two ballots (an entry emits its inside tail
        // vertex and/or its crossing vertex)
        const unsigned mi = pfw::ballot(ina), mc = pfw::ballot(cr);
        if (k < nl) {
            const int pc = pfw::popc(mc & lt);
            const int pcr = NE + pc, pem = NEm + pfw::popc(mi & lt) + pc;
            if (cr && pcr < C::CE) { S.ea[pcr] = (uint16_t)a; S.eb[pcr] = (uint16_t)b; }
            S.epos[k] = (uint16_t)pem;
            S.cpos[k] = pcr;
            if (k == A.lp[f]) S.fscan0[f] = (uint16_t)pem;
            const int em = (ina ? 1 : 0) + (cr ? 1 : 0);
            // the facet's last entry records where its emission ends (3b
            // subtracts where it starts): no zeroing pass, no atomics
            if (k + 1 == A.lp[f + 1]) S.fk[f] = pem + em;
        }
        NE += pfw::popc(mc);
        NEm += pfw::popc(mi) + pfw::popc(mc);
    }
    pfw::sync();
    // 3b. prefix sums in facet order: kept-facet indices and loop bases
    int NFk = 0, NLk = 0;
    bool small_facet = false;  // a dropped facet that still emitted 1-2 entries
    #pragma unroll 1
    for (int f0 = 0; f0 < nf; f0 += 32) {
        int f = f0 + L;
        int kk = 0, keep = 0;
        if (f < nf) {
            kk = S.fk[f] - S.fscan0[f];
            S.fk[f] = kk;
            keep = kk >= 3;
        }
        small_facet |= pfw::any(kk >= 1 && kk <= 2);
        int tot;
        const int pk = pfw::excl_scan_inl((keep << 16) | (keep ? kk : 0), L, &tot);
        if (f < nf) {
            S.fout[f] = (uint16_t)(NFk + (pk >> 16));
            S.flb[f] = keep ? (uint16_t)(NLk + (pk & 0xffff)) : (uint16_t)0xffff;
        }
        NFk += tot >> 16;
        NLk += tot & 0xffff;
    }
    if (NE > C::CE) { if (L == 0) ws->oflow = 1; pfw::sync(); return CLIP_OVERFLOW; }
    pfw::sync();
    // 3d. first encounter of each edge creates the crossing vertex (_kernels.py:178-200)
    int NFirst = 0;
    #pragma unroll 1
    for (int q0 = 0; q0 < NE; q0 += 32) {
        int q = q0 + L;
        bool first = false;
        int mt = q;
        int a = 0, b = 0;
        if (q < NE) { a = S.ea[q]; b = S.eb[q]; }
        const int lo = a < b ? a : b, hi = a < b ? b : a;
        if (NE <= 32) {
            // one chunk: the entries of the same edge are the lanes with the same key
            const unsigned mm = pfw::match_any(q < NE ? (lo << 16) | hi : -1 - L);
            mt = __builtin_ctz_pf(mm);
        } else if (q < NE) {
            #pragma unroll 1
            for (int r = 0; r < q; r++) {
                int ra = S.ea[r], rb = S.eb[r];
                int rlo = ra < rb ? ra : rb, rhi = ra < rb ? rb : ra;
                if (rlo == lo && rhi == hi) { mt = r; break; }
            }
        }
        if (q < NE) {
            first = mt == q;
            S.emt[q] = (uint16_t)mt;
        }
        unsigned m = pfw::ballot(first);
        if (first) {
            int id = K + NFirst + pfw::popc(m & lt);
            S.eid[q] = (uint16_t)id;
            if (id < C::CV) {
                double sa = S.sd[a], sb = S.sd[b];
                double t = sa / (sa - sb);
                const double nxv = A.x[a] + t * (A.x[b] - A.x[a]);
                const double nyv = A.y[a] + t * (A.y[b] - A.y[a]);
                const double nzv = A.z[a] + t * (A.z[b] - A.z[a]);
                B.x[id] = nxv; B.y[id] = nyv; B.z[id] = nzv;
                const double d2 = sq(nxv - px) + sq(nyv - py) + sq(nzv - pz);
                if (d2 > rmax) rmax = d2;
            }
        }
        NFirst += pfw::popc(m);
    }
    const int NVB = K + NFirst;
    if (cen_on(ws) && L == 0) ws->cen[CEN_NEWV] += NFirst;
    if (NVB > C::CV || NFk > C::CF || NLk > C::CL) {
        if (!C::EXACT && L == 0) ws->oflow = 1;
        pfw::sync();
        return CLIP_OVERFLOW;
    }
    pfw::sync();
    #pragma unroll 1
    for (int q = L; q < NE; q += 32) {
        int mt = S.emt[q];
        if (mt != q) S.eid[q] = S.eid[mt];
    }
    pfw::sync();
    // 3e. emit kept facets (_kernels.py:229-241): lane per loop entry, then
    // lane per facet for the planes
    #pragma unroll 1
    for (int k = L; k < nl; k += 32) {
        const int f = lfa[k];
        const int lb = S.flb[f];
        if (lb == 0xffff) continue;
        const int o = S.fout[f];
        const int cl = S.ecls[k];
        int w = lb + S.epos[k] - S.fscan0[f];
        if (cl & 1) { B.lv[w] = S.vmap[A.lv[k]]; lfb[w] = (uint8_t)o; w++; }
        if (cl & 2) { B.lv[w] = S.eid[S.cpos[k]]; lfb[w] = (uint8_t)o; }
    }
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        int lb = S.flb[f];
        if (lb == 0xffff) continue;
        int o = S.fout[f];
        B.nx[o] = A.nx[f]; B.ny[o] = A.ny[f]; B.nz[o] = A.nz[f]; B.d[o] = A.d[f];
        B.tag[o] = A.tag[f];
        B.lp[o] = (uint16_t)lb;
        B.lp[o + 1] = (uint16_t)(lb + S.fk[f]);
    }
    // 4. new facet (_kernels.py:243-295).  on_new = kept on-plane vertices
    // (sa >= -tol when emitted, i.e. every kept vertex with sd >= -tol) and
    // all crossing vertices, in B index order.
    int ncp = 0;
    if (nv <= 32) {
        const bool on = L < nv && s_reg <= tol && s_reg >= -tol;
        const unsigned m = pfw::ballot(on);
        if (on) S.onl[pfw::popc(m & lt)] = (uint16_t)vmap_reg;
        ncp = pfw::popc(m);
    } else {
        #pragma unroll 1
        for (int v0 = 0; v0 < nv; v0 += 32) {
            int v = v0 + L;
            bool on = v < nv && S.sd[v] <= tol && S.sd[v] >= -tol;
            unsigned m = pfw::ballot(on);
            if (on) S.onl[ncp + pfw::popc(m & lt)] = S.vmap[v];
            ncp += pfw::popc(m);
        }
    }
    #pragma unroll 1
    for (int q = L; q < NFirst; q += 32) S.onl[ncp + q] = (uint16_t)(K + q);
    ncp += NFirst;
    if (ncp < 3) { pfw::sync(); return CLIP_DEGENERATE; }
    if (NFk + 1 > C::CF || NLk + ncp > C::CL) {
        if (!C::EXACT && L == 0) ws->oflow = 1;
        pfw::sync();
        return CLIP_OVERFLOW;
    }
    pfw::sync();
    // centroid: sequential sum in index order, computed redundantly by every lane
    // (lane a < 3 sums coordinate a: the same sequential sums and divisions)
    double cc = 0.0;
    if (L < 3) {
        const double *crd = L == 0 ? B.x : (L == 1 ? B.y : B.z);
        int q = 0;
        #pragma unroll 1
        for (; q + 4 <= ncp; q += 4) {  // loads first, then the sequential sum
            const double a0 = crd[S.onl[q]], a1 = crd[S.onl[q + 1]], a2 = crd[S.onl[q + 2]], a3 = crd[S.onl[q + 3]];
            cc += a0; cc += a1; cc += a2; cc += a3;
        }
        #pragma unroll 1
        for (; q < ncp; q++) cc += crd[S.onl[q]];
        cc /= (double)ncp;
    }
    const double ccx = pfw::shfl(cc, 0), ccy = pfw::shfl(cc, 1), ccz = pfw::shfl(cc, 2);
    double e[6];
    perp_basis_inl(nx, ny, nz, e);
    #pragma unroll 1
    for (int q = L; q < ncp; q += 32) {
        int v = S.onl[q];
        double rx = B.x[v] - ccx, ry = B.y[v] - ccy, rz = B.z[v] - ccz;
        const double yq = rx * e[3] + ry * e[4] + rz * e[5];
        const double xq = rx * e[0] + ry * e[1] + rz * e[2];
        S.sy[q] = yq;
        S.sd[q] = xq;
        S.half[q] = (uint8_t)half_of(xq, yq);
    }
    pfw::sync();
    // rank sort by (atan2 angle, index) -- the reference's insertion sort is
    // stable on that total order (_kernels.py:269-283); the angle order is
    // decided by half-plane and orientation instead of evaluating atan2.
    // Lanes take (u, q) pairs: q = lane mod W, W the smallest power of two
    // >= ncp (new facets are small: 32 / W comparisons per pass).
    {
        const int Wd = ncp <= 8 ? 8 : (ncp <= 16 ? 16 : 32);
        const int step = 32 / Wd;
        #pragma unroll 1
        for (int q0 = 0; q0 < ncp; q0 += Wd) {
            const int q = q0 + (L & (Wd - 1));
            int r = 0;
            int vq = 0;
            if (q < ncp) {
                const double xq = S.sd[q], yq = S.sy[q];
                const int hq = S.half[q];
                vq = S.onl[q];
                #pragma unroll 1
                for (int u = L / Wd; u < ncp; u += step) {
                    const double xu = S.sd[u], yu = S.sy[u];
                    const int hu = S.half[u];
                    bool lt, eq;
                    if (hu != hq) { lt = hu < hq; eq = false; }
                    else {
                        // ang_lt(u, q) and ang_lt(q, u) from one cross product
                        // (xq yu - yq xu == -(xu yq - yu xq) exactly)
                        const double cr = xu * yq - yu * xq;
                        if (cr != 0.0) { lt = cr > 0.0; eq = false; }
                        else if (xu * xq + yu * yq >= 0.0) { lt = false; eq = true; }
                        else { lt = xu > 0.0; eq = !(xu > 0.0) && !(xq > 0.0); }
                    }
                    r += (lt || (eq && S.onl[u] < vq)) ? 1 : 0;
                }
            }
            #pragma unroll 1
            for (int m = Wd; m < 32; m <<= 1) r += pfw::shfl_xor(r, m);
            if (L < Wd && q < ncp) { B.lv[NLk + r] = (uint16_t)vq; lfb[NLk + r] = (uint8_t)NFk; }
        }
    }
    if (L == 0) {
        B.nx[NFk] = nx; B.ny[NFk] = ny; B.nz[NFk] = nz; B.d[NFk] = dd;
        B.tag[NFk] = tag;
        B.lp[NFk] = (uint16_t)NLk;
        B.lp[NFk + 1] = (uint16_t)(NLk + ncp);
    }
    const int NF2 = NFk + 1, NL2 = NLk + ncp;
    pfw::sync();
    // 5. drop unreferenced vertices (_kernels.py:297-315).  A kept vertex can
    // only lose all its facets if some dropped facet emitted 1-2 entries.
    if (!small_facet) {
        *rfar2 = pfw::max_d_inl(rmax);
        if (L == 0) {
            B.nv = NVB; B.nf = NF2; B.nl = NL2;
            if (cen_on(ws)) { ws->cen[CEN_NFV] += ncp; ws->cen[CEN_CUTS]++; ws->cen[CEN_RFAR] += NVB; }
        }
        pfw::sync();
        return CLIP_CUT;
    }
    const int nref = clip_drop_unreferenced(ws, B, NVB, NL2);
    *rfar2 = -1.0;
    if (L == 0) {
        B.nv = nref; B.nf = NF2; B.nl = NL2;
        if (cen_on(ws)) { ws->cen[CEN_NFV] += ncp; ws->cen[CEN_CUTS]++; ws->cen[CEN_RFAR] += nref; }
    }
    pfw::sync();
    return CLIP_CUT;
}

// ---------------------------------------------------------------------------
// candidate gather over one distance shell [t_lo, t_hi) of d^2
// ---------------------------------------------------------------------------
PF_DEV int bucket_coord(double x, double lo, double ih, int gn) {
    double t = (x - lo) * ih;
    int b;
    if (!(t > -1.0)) b = 0;  // also catches NaN
    else if (t >= (double)gn) b = gn - 1;
    else b = (int)t;
    if (b < 0) b = 0;
    if (b >= gn) b = gn - 1;
    return b;
}

// returns the number of candidates (may exceed CC: overflow); *all_sites set
// when the bucket range spans the whole grid
template <bool SKIP_INNER, class W>
PF_DEV int gather_shell(W *ws, const CellIn &in, int self, double px, double py, double pz,
                        double t_lo, double t_hi, bool *all_sites) {
    using C = typename W::Cap;
    BuildScratch<C> &S = ws->u.b;
    const GridView &g = in.g;
    const int L = pfw::lane();
    double r = sqrt(t_hi) * (1.0 + 1e-9) + 1e-300;
    int i0 = bucket_coord(px - r, g.lo[0], g.ih[0], g.gn[0]);
    int i1 = bucket_coord(px + r, g.lo[0], g.ih[0], g.gn[0]);
    int j0 = bucket_coord(py - r, g.lo[1], g.ih[1], g.gn[1]);
    int j1 = bucket_coord(py + r, g.lo[1], g.ih[1], g.gn[1]);
    int k0 = bucket_coord(pz - r, g.lo[2], g.ih[2], g.gn[2]);
    int k1 = bucket_coord(pz + r, g.lo[2], g.ih[2], g.gn[2]);
    *all_sites = i0 == 0 && j0 == 0 && k0 == 0 && i1 == g.gn[0] - 1 && j1 == g.gn[1] - 1 &&
                 k1 == g.gn[2] - 1;
    const int ny = j1 - j0 + 1;
    const int nruns = (i1 - i0 + 1) * ny;
    // the grid arrays into registers: `in` lives in local memory and the
    // compiler must otherwise reload it after every (generic) shared store
    const double *__restrict__ gsx = g.sx, *__restrict__ gsy = g.sy, *__restrict__ gsz = g.sz;
    const int *__restrict__ gsid = g.sid, *__restrict__ gbst = g.bstart;
    const double *__restrict__ gpsi = in.psi;
    const int gn1 = g.gn[1], gn2 = g.gn[2];
    if (L == 0) S.ncand = 0;
    pfw::sync();
    bool beyond = false;
    #pragma unroll 1
    for (int r0 = 0; r0 < nruns; r0 += 32) {
        int rr = r0 + L;
        int st = 0, len = 0, la = 0, stb = 0;
        if (rr < nruns) {
            // the column's buckets [k0, k1] minus the middle ones lying wholly
            // inside the previous shells (d^2 < t_lo): two runs of sites.  Edge
            // buckets (which also hold clamped sites) are never skipped; the
            // 1e-6-bucket margins dwarf the rounding of the bucket assignment.
            const int ix = i0 + rr / ny, iy = j0 + rr % ny;
            const int base = (ix * gn1 + iy) * gn2;
            int ka1 = k1, kb0 = k1 + 1;
            if (SKIP_INNER && t_lo > 0.0 && ix > 0 && ix < g.gn[0] - 1 && iy > 0 && iy < g.gn[1] - 1) {
                const double hx = 1.0 / g.ih[0], hy = 1.0 / g.ih[1];
                const double xl = g.lo[0] + (ix - 1e-6) * hx, xh = g.lo[0] + (ix + 1 + 1e-6) * hx;
                const double yl = g.lo[1] + (iy - 1e-6) * hy, yh = g.lo[1] + (iy + 1 + 1e-6) * hy;
                const double dx = fmax(fabs(xl - px), fabs(xh - px));
                const double dy = fmax(fabs(yl - py), fabs(yh - py));
                const double rem = t_lo * (1.0 - 1e-9) - dx * dx - dy * dy;
                if (rem > 0.0) {
                    const double sz = sqrt(rem);
                    int kin0 = (int)ceil((pz - sz - g.lo[2]) * g.ih[2] + 1e-6);
                    int kin1 = (int)floor((pz + sz - g.lo[2]) * g.ih[2] - 1e-6) - 1;
                    if (kin0 < k0) kin0 = k0;
                    if (kin0 < 1) kin0 = 1;
                    if (kin1 > k1) kin1 = k1;
                    if (kin1 > g.gn[2] - 2) kin1 = g.gn[2] - 2;
                    if (kin0 <= kin1) { ka1 = kin0 - 1; kb0 = kin1 + 1; }
                }
            }
            st = gbst[base + k0];
            if (ka1 == k1) {
                len = la = gbst[base + k1 + 1] - st;
            } else {
                la = gbst[base + ka1 + 1] - st;
                stb = gbst[base + kb0];
                len = la + (gbst[base + k1 + 1] - stb);
            }
        }
        int tot;
        int off = pfw::excl_scan_inl(len, L, &tot);
        S.run_start[L] = st;
        S.run_off[L] = off;
        S.run_la[L] = la;
        S.run_stb[L] = stb;
        pfw::sync();
        int nr = nruns - r0 < 32 ? nruns - r0 : 32;
        #pragma unroll 1
        for (int q0 = 0; q0 < tot; q0 += 32) {
            int q = q0 + L;
            if (q < tot) {
                // last run whose offset <= q
                int lo = 0, hi = nr - 1;
                while (lo < hi) {
                    int mid = (lo + hi + 1) >> 1;
                    if (S.run_off[mid] <= q) lo = mid; else hi = mid - 1;
                }
                const int e = q - S.run_off[lo];
                int s = S.run_start[lo] + e;
                if (SKIP_INNER) {  // only later shells have two runs per column
                    const int la_ = S.run_la[lo];
                    if (e >= la_) s = S.run_stb[lo] + (e - la_);
                }
                int j = gsid[s];
                double d2 = sq(gsx[s] - px) + sq(gsy[s] - py) + sq(gsz[s] - pz);
                if (j != self && !(d2 < t_hi)) beyond = true;
                if (j != self && d2 >= t_lo && d2 < t_hi) {
                    int pos = pfw::atom_add(&S.ncand, 1);
                    if (pos < C::CC) {
                        S.cd2[pos] = d2; S.cj[pos] = j;
                        S.cx[pos] = gsx[s]; S.cy[pos] = gsy[s]; S.cz[pos] = gsz[s];
                        S.cw[pos] = gpsi ? gpsi[j] : 0.0;
                    }
                }
            }
        }
        pfw::sync();
    }
    if (pfw::any(beyond)) *all_sites = false;
    int nc = S.ncand;
    pfw::sync();
    return nc;
}

// sort the shell's candidates by (d2, j) in place (rank sort through registers)
template <class W>
PF_DEV void sort_candidates(W *ws, int nc) {
    using C = typename W::Cap;
    BuildScratch<C> &S = ws->u.b;
    const int L = pfw::lane();
    constexpr int PER = (C::CC + 31) / 32;
    double kd[PER];
    int kj[PER], kr[PER];
#pragma unroll
    for (int t = 0; t < PER; t++) {
        int q = t * 32 + L;
        kr[t] = -1;
        if (q < nc) {
            kd[t] = S.cd2[q];
            kj[t] = S.cj[q];
            int r = 0;
            #pragma unroll 1
            for (int u = 0; u < nc; u++) {
                double du = S.cd2[u];
                int ju = S.cj[u];
                r += (du < kd[t] || (du == kd[t] && ju < kj[t])) ? 1 : 0;
            }
            kr[t] = r;
        }
    }
    pfw::sync();
#pragma unroll
    for (int t = 0; t < PER; t++) {
        if (kr[t] >= 0) { S.cd2[kr[t]] = kd[t]; S.cj[kr[t]] = kj[t]; S.cord[kr[t]] = (uint16_t)(t * 32 + L); }
    }
    pfw::sync();
}

// Weight slack of site i's security radius rfar + sqrt(rfar^2 + slack).  The
// reference takes the global max - min weight (_kernels.py:1300-1306).  A site
// j can only cut the cell while |p_j - p_i| < rfar + sqrt(rfar^2 + psi_j -
// psi_i), so any bound of psi_j - psi_i over the sites the reference processes
// -- all within the ball-aware radius br of p_i -- is an exact slack: the sites
// between the two radii leave the polytope untouched (h_ij >= rfar), as the
// reference's own classification would find.  The bound is the max weight of
// the super-buckets covering the box p_i +- br.  br itself keeps the global
// slack (it is the reference's stop, not a property of the polytope).
// Thread-per-site (pf_runtime.cu k_cell_slack); host-callable for the emulator.
PF_DEV double cell_slack(const GridView &g, double px, double py, double pz, double psii, double dpsi) {
    if (!(psii > 0.0)) return dpsi;
    const double br = (sqrt(psii) + sqrt(psii + dpsi)) * (1.0 + 1e-12);
    const int f = g.sf;
    const int a0 = bucket_coord(px - br, g.lo[0], g.ih[0], g.gn[0]) / f;
    const int a1 = bucket_coord(px + br, g.lo[0], g.ih[0], g.gn[0]) / f;
    const int b0 = bucket_coord(py - br, g.lo[1], g.ih[1], g.gn[1]) / f;
    const int b1 = bucket_coord(py + br, g.lo[1], g.ih[1], g.gn[1]) / f;
    const int c0 = bucket_coord(pz - br, g.lo[2], g.ih[2], g.gn[2]) / f;
    const int c1 = bucket_coord(pz + br, g.lo[2], g.ih[2], g.gn[2]) / f;
    double m = -1e300;
    for (int a = a0; a <= a1; a++)
        for (int b = b0; b <= b1; b++)
            for (int c = c0; c <= c1; c++) {
                const double v = g.smax[(a * g.sgn[1] + b) * g.sgn[2] + c];
                m = v > m ? v : m;
            }
    const double dl = m - psii;
    return dl > 0.0 ? (dl < dpsi ? dl : dpsi) : 0.0;
}

// later shells (t_lo > 0) out of line: the first shell -- the only one of most
// cells at converged weights -- keeps the lean single-run gather
template <class W>
#ifndef PF_GATHER_INL
#define PF_GATHER_INL 0
#endif
#if PF_GATHER_INL
PF_DEV
#else
PF_NOINL
#endif
int gather_later(W *ws, const CellIn &in, int self, double px, double py, double pz, double t_lo,
                          double t_hi, bool *all_sites) {
    return gather_shell<true>(ws, in, self, px, py, pz, t_lo, t_hi, all_sites);
}

// ---------------------------------------------------------------------------
// build the Laguerre cell of site i (_kernels.py:1197-1355)
// returns 0 ok / 1 empty / 3 overflow; *which = buffer holding the cell
// ---------------------------------------------------------------------------
// HV: the general build (full mode with the heavy-site phase, packed
// outputs); HV = false is the ball-aware evaluation build, compiled without
// the other modes' paths (the heavy-site phase alone cost it ~25%)
template <class W, bool HV = true>
#ifndef PF_BUILD_CELL_INL
#define PF_BUILD_CELL_INL 1  // build_cell inlined into its kernels (out of line: C4 build 49.7 -> 57.8 ms)
#endif
#if PF_BUILD_CELL_INL
PF_DEV
#else
PF_NOINL
#endif
int build_cell(W *ws, const CellIn &in, int i, int *which_out, int *nclips) {
    using C = typename W::Cap;
    const double px = in.pts[3 * i], py = in.pts[3 * i + 1], pz = in.pts[3 * i + 2];
    const double psii = in.psi[i];
    const bool ball_aware = !HV || in.ball_aware != 0;  // hoisted: `in` is in local memory
    const double tol = in.tol, dpsi = in.dpsi_ptr ? *in.dpsi_ptr : in.dpsi;
    load_domain(ws->P[0], in);
    #pragma unroll 1
    for (int f = pfw::lane(); f < in.dnf; f += 32)
        #pragma unroll 1
        for (int k = in.dlp[f]; k < in.dlp[f + 1]; k++) ws->u.b.lf[0][k] = (uint8_t)f;
    pfw::sync();
    int which = 0;
    int ncl = 0;
    *nclips = 0;
    double rfar = poly_rfar(ws->P[0], px, py, pz);
    const double sq_ball = (ball_aware && psii > 0.0) ? sqrt(psii) : -1.0;
    const double sq_psi_slack = sqrt((psii > 0.0 ? psii : 0.0) + dpsi);
    if (ball_aware && psii <= 0.0) { *which_out = 0; return 0; }
    const double br = sq_ball + sq_psi_slack;

    // weight slack of the security radius: the per-cell bound of cell_slack()
    // when the runtime computed it, else the reference's global one
    double dpsi_s = (ball_aware && in.cslack) ? in.cslack[i] : dpsi;

    // Full mode with the heavy-site list (in.heavy_*): a site j can only cut
    // while |p_j - p_i| < rfar + sqrt(rfar^2 + psi_j - psi_i), so the slack
    // splits into the ordinary sites' (largest weight outside the list) and
    // that of the heavy sites not processed yet (lane k holds heavy site k).
    // The (d^2, j)-ordered stream of all sites stops at the ordinary radius;
    // the heavy sites beyond it follow in (d^2, j) order.  Everything skipped
    // is a site that leaves the polytope untouched at its turn (rfar only
    // shrinks), so the cuts and their order are the reference's -- without
    // the n - 1 candidates one huge weight makes every cell visit
    // (SURVEY.md §8(f) row 2).
    const bool heavy = HV && !ball_aware && in.heavy_idx != nullptr && in.nheavy > 0;
    const int Lh = pfw::lane();
    int hk = -1;
    double hw = 0.0;
    unsigned unseen = 0;
    double slack_rest = dpsi;
    if (heavy) {
        if (Lh < in.nheavy) { hk = in.heavy_idx[Lh]; hw = in.heavy_psi[Lh]; }
        unseen = pfw::ballot(Lh < in.nheavy && hk != i);  // the cell's own site is no candidate
        const double pr = in.heavy_psi[in.nheavy] - psii;
        slack_rest = pr > 0.0 ? (pr < dpsi ? pr : dpsi) : 0.0;
    }
    // the slack over the ordinary sites and the unprocessed heavy ones
    auto heavy_slack = [&]() {
        double sl = ((unseen >> Lh) & 1u) ? hw - psii : -1e300;
        sl = pfw::max_d_inl(sl);
        sl = sl > slack_rest ? sl : slack_rest;
        return sl > 0.0 ? (sl < dpsi ? sl : dpsi) : 0.0;
    };
    if (heavy) dpsi_s = heavy_slack();
    bool to_heavy = false;  // the ordinary stream is done: heavy-site phase

    double t_lo = -1.0;
    double t_hi = ball_aware ? br * br * (1.0 + 1e-14) : in.t_init;
    if (!(t_hi > 0.0)) t_hi = 1e-300;
    int ngot = 0;
    #pragma unroll 1
    for (;;) {
        bool all_sites = false;
        if (cen_on(ws) && pfw::lane() == 0) ws->cen[CEN_GATH]++;
        int nc = t_lo > 0.0 ? gather_later(ws, in, i, px, py, pz, t_lo, t_hi, &all_sites)
                            : gather_shell<false>(ws, in, i, px, py, pz, t_lo, t_hi, &all_sites);
        if (nc > C::CC) {
            // too many candidates in this shell: narrow it (ties at one d^2
            // cannot be split -> overflow)
            // (aim at 0.7 CC candidates, assuming a uniform density of sites in the shell)
            double base = t_lo > 0.0 ? t_lo : 0.0;
            const double rl3 = base * sqrt(base), rh3 = t_hi * sqrt(t_hi);
            const double r3 = rl3 + (rh3 - rl3) * (0.7 * C::CC / nc);
            double nt = cbrt(r3 * r3);
            const double half = base + (t_hi - base) * 0.5;
            if (!(nt < half)) nt = half;
            if (!(nt > base) || !(nt < t_hi)) {
                if (pfw::lane() == 0) ws->oflow = 1;
                pfw::sync();
                *which_out = which;
                *nclips = ncl;
                return 3;
            }
            t_hi = nt;
            continue;
        }
        sort_candidates(ws, nc);
        BuildScratch<C> &S = ws->u.b;
        // bisector planes of the shell's candidates, lane per candidate, with
        // the reference's operations (_kernels.py:1325-1330); a coincident
        // site keeps its weight for the tie rule (_kernels.py:1320-1324)
        #pragma unroll 1
        for (int c = pfw::lane(); c < nc; c += 32) {
            const double D2 = S.cd2[c];
            const double D = sqrt(D2);
            // the serial loop below needs only D (its stop test, _kernels.py:1309)
            // and whether the site is coincident: D replaces D^2, -1 marks it
            S.cd2[c] = D2 <= tol * tol ? -1.0 : D;
            if (D2 <= tol * tol) continue;
            const int sl = S.cord[c];
            const double psij = S.cw[sl];
            const double nxp = (S.cx[sl] - px) / D;
            const double nyp = (S.cy[sl] - py) / D;
            const double nzp = (S.cz[sl] - pz) / D;
            const double hij = 0.5 * (D2 + psii - psij) / D;
            S.cx[sl] = nxp; S.cy[sl] = nyp; S.cz[sl] = nzp;
            S.cw[sl] = (nxp * px + nyp * py + nzp * pz) + hij;
        }
        pfw::sync();
        double stop_r = rfar + sqrt(rfar * rfar + dpsi_s);
        if (ball_aware && br < stop_r) stop_r = br;
        double r_rest = heavy ? rfar + sqrt(rfar * rfar + slack_rest) : stop_r;
        #pragma unroll 1
        for (int c = 0; c < nc; c++) {
            // candidate c into registers; the warp syncs before any lane acts on
            // it (a lane that runs ahead must not overwrite the shared scratch
            // -- next shell's gather, evaluation workspace -- under a slower lane)
            const double Dc = S.cd2[c];  // sqrt(d^2), or -1 for a coincident site
            const int j = S.cj[c];
            const int sl = S.cord[c];
            const double nxc = S.cx[sl], nyc = S.cy[sl], nzc = S.cz[sl], ddc = S.cw[sl];
            pfw::sync();
            if (Dc >= stop_r) { *which_out = which; *nclips = ncl; return 0; }
            if (heavy) {
                const unsigned hm = pfw::ballot(hk == j) & unseen;
                if (hm) {  // a heavy site in the stream: processed here, at its turn
                    unseen &= ~hm;
                    dpsi_s = heavy_slack();
                    stop_r = rfar + sqrt(rfar * rfar + dpsi_s);
                } else if (Dc >= r_rest) {  // no ordinary site can cut any more
                    to_heavy = true;
                    break;
                }
            }
            if (Dc < 0.0) {
                const double psij = ddc;  // coincident site: the slot kept its weight
                if (psij > psii || (psij == psii && j < i)) { *which_out = which; *nclips = ncl; return 1; }
                continue;
            }
            ncl++;
            // Every vertex lies within rfar of the site, so a bisector plane
            // farther than rfar (h = dd - n.p) leaves the polytope untouched:
            // the reference's vertex classification would find no vertex with
            // s > tol.  Skip it (exact: the margin dwarfs the rounding of s, h
            // and rfar).  Same census as the classification.
            if (ddc - (nxc * px + nyc * py + nzc * pz) > rfar * (1.0 + 1e-12) + 1e-12) {
                if (cen_on(ws) && pfw::lane() == 0) { ws->cen[CEN_CLIPS]++; ws->cen[CEN_TESTS] += ws->P[which].nv; }
                continue;
            }
            double rfar2;
            int st = clip(ws, ws->P[which], ws->P[1 - which], which, nxc, nyc, nzc, ddc, j, tol, px, py, pz, &rfar2);
            if (st == CLIP_EMPTY) { *which_out = which; *nclips = ncl; return 1; }
            if (st == CLIP_OVERFLOW) { *which_out = which; *nclips = ncl; return 3; }
            if (st == CLIP_CUT) {
                which = 1 - which;
                // rfar and the stop radius from max |v - p|^2 as two independent
                // square roots (the reference squares the rounded rfar; the stop
                // radius only has to bound the cutting sites, which it does with a
                // margin of tol over the ulps: a site at the boundary leaves every
                // vertex within rounding of its plane)
                if (rfar2 < 0.0) rfar2 = poly_rfar2(ws->P[which], px, py, pz);
                rfar = sqrt(rfar2);
                stop_r = rfar + sqrt(rfar2 + dpsi_s);
                if (ball_aware && br < stop_r) stop_r = br;
                if (heavy) r_rest = rfar + sqrt(rfar2 + slack_rest);
            }
        }
        if (to_heavy || all_sites) break;
        if (heavy) stop_r = r_rest;  // the shells only carry the ordinary stream
        if (sqrt(t_hi) >= stop_r) break;
        // next shell: sized for ~0.7 CC candidates from the density seen so far
        // (volume x 8 at most), and never past the stop radius -- the shells
        // only batch the (d^2, j)-ordered candidate stream, any cut is exact
        ngot += nc;
        double f = ngot > 0 ? 1.0 + 0.7 * C::CC / ngot : 8.0;
        if (f > 8.0) f = 8.0;
        const double cf = cbrt(f);
        t_lo = t_hi;
        t_hi = t_hi * (cf * cf);
        const double tstop = stop_r * stop_r * (1.0 + 1e-12);
        if (t_hi > tstop) t_hi = tstop;
    }
    // heavy-site phase: the unprocessed heavy sites in (d^2, j) order, each
    // with the stream's tests and the bisector plane of _kernels.py:1325-1330
    if (heavy && unseen) {
        double hx = 0.0, hy = 0.0, hz = 0.0, hd2 = 0.0;
        if ((unseen >> Lh) & 1u) {
            hx = in.pts[3 * hk]; hy = in.pts[3 * hk + 1]; hz = in.pts[3 * hk + 2];
            hd2 = sq(hx - px) + sq(hy - py) + sq(hz - pz);
        }
        #pragma unroll 1
        while (unseen) {
            // the unprocessed heavy site first in (d^2, j) order
            int m = -1;
            #pragma unroll 1
            for (unsigned u = unseen; u; u &= u - 1) {
                const int k = __builtin_ctz_pf(u);
                const double dk = pfw::shfl(hd2, k);
                const int jk = pfw::shfl(hk, k);
                if (m < 0) { m = k; continue; }
                const double dm = pfw::shfl(hd2, m);
                const int jm = pfw::shfl(hk, m);
                if (dk < dm || (dk == dm && jk < jm)) m = k;
            }
            const double D2 = pfw::shfl(hd2, m);
            const int j = pfw::shfl(hk, m);
            const double psij = pfw::shfl(hw, m);
            const double cx = pfw::shfl(hx, m), cy = pfw::shfl(hy, m), cz = pfw::shfl(hz, m);
            const double D = sqrt(D2);
            // the remaining heavy sites are at least this far: none can cut
            if (D2 > tol * tol && D >= rfar + sqrt(rfar * rfar + dpsi_s)) break;
            unseen &= ~(1u << m);
            dpsi_s = heavy_slack();
            if (D2 <= tol * tol) {
                if (psij > psii || (psij == psii && j < i)) { *which_out = which; *nclips = ncl; return 1; }
                continue;
            }
            ncl++;
            const double nxc = (cx - px) / D, nyc = (cy - py) / D, nzc = (cz - pz) / D;
            const double hij = 0.5 * (D2 + psii - psij) / D;
            const double ddc = (nxc * px + nyc * py + nzc * pz) + hij;
            if (ddc - (nxc * px + nyc * py + nzc * pz) > rfar * (1.0 + 1e-12) + 1e-12) {
                if (cen_on(ws) && pfw::lane() == 0) { ws->cen[CEN_CLIPS]++; ws->cen[CEN_TESTS] += ws->P[which].nv; }
                continue;
            }
            double rfar2;
            int st = clip(ws, ws->P[which], ws->P[1 - which], which, nxc, nyc, nzc, ddc, j, tol, px, py, pz, &rfar2);
            if (st == CLIP_EMPTY) { *which_out = which; *nclips = ncl; return 1; }
            if (st == CLIP_OVERFLOW) { *which_out = which; *nclips = ncl; return 3; }
            if (st == CLIP_CUT) {
                which = 1 - which;
                if (rfar2 < 0.0) rfar2 = poly_rfar2(ws->P[which], px, py, pz);
                rfar = sqrt(rfar2);
            }
        }
    }
    *which_out = which;
    *nclips = ncl;
    return 0;
}

// ---------------------------------------------------------------------------
// evaluation (_kernels.py:411-1170)
//
// Lane-parallel over loop entries and boundary points instead of facets: the
// restriction emits every loop entry's points with one warp scan, so each
// facet's boundary ring is a contiguous run of the point pool, in the
// reference's walk order; the generalized-polygon integrals and the
// Gauss-Bonnet patch terms are then computed lane per boundary point and
// summed per facet with a segmented warp reduction (fixed shuffle tree:
// deterministic).  A facet walk done by one lane (the reference's loop)
// leaves 2/3 of the warp idle on the paper's scenes.
// ---------------------------------------------------------------------------
enum { PF_ONSPH = 1, PF_CONN = 2, PF_DEL = 4, PF_ENTRY = 8 };
enum { PF_DEAD = 0xff };  // pfac of a pool slot freed by the zero-length merge

// _edge_other_facet (_kernels.py:397-408): lowest facet != f holding the
// directed edge (bb -> a), through the per-cell vertex incidence table
template <class C>
PF_DEV int twin_facet(const EvalScratch<C> &E, const Poly<C> &P, int f, int a, int bb) {
    int g = -1;
    const int dg = E.vdeg[bb];
    if (dg <= 4) {
        #pragma unroll 1
        for (int t = 0; t < dg; t++) {
            const int k2 = E.vinc[bb * 4 + t];
            const int g2 = E.efac[k2];
            if (E.esv[k2] == a && g2 != f && (g < 0 || g2 < g)) g = g2;
        }
    } else {
        #pragma unroll 1
        for (int gg = 0; gg < P.nf && g < 0; gg++) {
            if (gg == f) continue;
            int s0 = P.lp[gg], mg = P.lp[gg + 1] - s0;
            #pragma unroll 1
            for (int ee = 0; ee < mg; ee++) {
                if (P.lv[s0 + ee] == bb && P.lv[s0 + (ee + 1 == mg ? 0 : ee + 1)] == a) { g = gg; break; }
            }
        }
    }
    return g;
}

// Restrict every facet to the ball (_kernels.py:411-675) into the point pool.
// Returns 0, 1 on a facet with more than MAX_P boundary points (the
// reference's kind -1), 2 on pool overflow.
template <class W>
PF_PHASE int restrict_all(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                          double psi, double R, double tol) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    const int nf = P.nf, nl = P.nl;
    const double ball_tol = tol * (2.0 * R + tol);
    // A. per facet: signed height, circle radius; OUTSIDE / UNTOUCHED / GENPOLY (_kernels.py:432-468)
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        const double s = P.d[f] - (P.nx[f] * px + P.ny[f] * py + P.nz[f] * pz);
        const double rc2 = psi - s * s;
        int kind = RF_OUTSIDE;
        double rc = 0.0;
        if (!(rc2 <= ball_tol)) {
            rc = dsqrt(rc2);
            const int s0 = P.lp[f], m = P.lp[f + 1] - s0;
            int n_in = 0;
            #pragma unroll 1
            for (int e = 0; e < m; e++) n_in += E.vin[P.lv[s0 + e]];
            kind = n_in == m ? RF_UNTOUCHED : RF_GENPOLY;
        }
        E.fh[f] = s; E.frc[f] = rc; E.fkind[f] = (uint8_t)kind; E.fmrg[f] = 0;
    }
    pfw::sync();
    // B. lane per loop entry (edge a -> bb of facet f): the points it adds to
    // the facet's ring (_kernels.py:470-587) -- a when inside the ball, then
    // the edge's sphere crossings in walk order, computed from the line of f
    // and its twin facet as the reference does.  The walk state before an
    // edge's crossings is always "inside" == (a inside), so every entry is
    // independent; the pool position comes from one warp scan.
    int base = 0;
    #pragma unroll 1
    for (int k0 = 0; k0 < nl; k0 += 32) {
        const int k = k0 + L;
        int cnt = 0, f = 0, fl0 = 0, fl1 = 0, fl2 = 0;
        double x0 = 0.0, y0 = 0.0, z0 = 0.0, x1 = 0.0, y1 = 0.0, z1 = 0.0;
        double x2 = 0.0, y2 = 0.0, z2 = 0.0;  // parity mode only: tail + spurious exit + entry
        if (k < nl) {
            f = E.efac[k];
            if (E.fkind[f] != RF_OUTSIDE) {
                const int a = P.lv[k], bb = E.esv[k];
                const bool ina = E.vin[a] != 0, inb = E.vin[bb] != 0;
                if (ina) { x0 = P.x[a]; y0 = P.y[a]; z0 = P.z[a]; cnt = 1; }
                if (!(ina && inb)) {
                    const double nx = P.nx[f], ny = P.ny[f], nz = P.nz[f], dd = P.d[f];
                    const int g = twin_facet(E, P, f, a, bb);
                    double gx, gy, gz, gd, c12, det, ux, uy, uz;
                    if (g >= 0) {
                        gx = P.nx[g]; gy = P.ny[g]; gz = P.nz[g]; gd = P.d[g];
                        c12 = nx * gx + ny * gy + nz * gz;
                        det = 1.0 - c12 * c12;
                        ux = ny * gz - nz * gy;
                        uy = nz * gx - nx * gz;
                        uz = nx * gy - ny * gx;
                    } else {
                        ux = P.x[bb] - P.x[a];
                        uy = P.y[bb] - P.y[a];
                        uz = P.z[bb] - P.z[a];
                        det = 1.0; c12 = 0.0; gd = 0.0; gx = 0.0; gy = 0.0; gz = 0.0;
                    }
                    const double un = dsqrt(ux * ux + uy * uy + uz * uz);
                    if (!(un < 1e-300 || det <= 1e-300)) {
                        ux = ddiv(ux, un); uy = ddiv(uy, un); uz = ddiv(uz, un);
                        if (ux < 0.0 || (ux == 0.0 && (uy < 0.0 || (uy == 0.0 && uz < 0.0)))) {
                            ux = -ux; uy = -uy; uz = -uz;
                        }
                        double ox, oy, oz;
                        if (g >= 0) {
                            const double r1 = dd - (nx * px + ny * py + nz * pz);
                            const double r2 = gd - (gx * px + gy * py + gz * pz);
                            const double al = ddiv(r1 - c12 * r2, det);
                            const double be = ddiv(r2 - c12 * r1, det);
                            ox = px + al * nx + be * gx;
                            oy = py + al * ny + be * gy;
                            oz = pz + al * nz + be * gz;
                        } else {
                            ox = P.x[a]; oy = P.y[a]; oz = P.z[a];
                        }
                        const double w0x = ox - px, w0y = oy - py, w0z = oz - pz;
                        const double bh = ux * w0x + uy * w0y + uz * w0z;
                        const double cc = w0x * w0x + w0y * w0y + w0z * w0z - psi;
                        const double disc = bh * bh - cc;
                        if (!(disc <= tol * tol)) {
                            const double sqd = dsqrt(disc);
                            const double t1 = -bh - sqd, t2 = -bh + sqd;
                            const double ta = ux * (P.x[a] - ox) + uy * (P.y[a] - oy) + uz * (P.z[a] - oz);
                            const double tb = ux * (P.x[bb] - ox) + uy * (P.y[bb] - oy) + uz * (P.z[bb] - oz);
                            const double tlo = ta < tb ? ta : tb;
                            const double thi = ta < tb ? tb : ta;
                            bool cur = ina;
                            #pragma unroll 1
                            for (int which = 0; which < 2; which++) {
                                const double t = (ta <= tb) == (which == 0) ? t1 : t2;
                                if (t <= tlo + tol || t >= thi - tol) continue;
                                // The first root in walk order is where the edge
                                // enters the ball.  After a vertex classified inside
                                // it can only pass the range test if that vertex lies
                                // outside the sphere by less than the tolerance; the
                                // reference then labels the entry an exit and closes
                                // the facet with a spurious arc (a whole circular
                                // segment too much).  It coincides with the vertex to
                                // ~tol: drop it.  Never fires on consistent geometry.
                                // (parity mode keeps it, as the reference does)
                                if (which == 0 && cur && !ws->strict) continue;
                                const double cxx = ox + t * ux, cxy = oy + t * uy, cxz = oz + t * uz;
                                const int fl = cur ? (PF_ONSPH | PF_CONN) : (PF_ONSPH | PF_ENTRY);
                                cur = !cur;
                                if (cnt == 0) { x0 = cxx; y0 = cxy; z0 = cxz; fl0 = fl; }
                                else if (cnt == 1) { x1 = cxx; y1 = cxy; z1 = cxz; fl1 = fl; }
                                else { x2 = cxx; y2 = cxy; z2 = cxz; fl2 = fl; }
                                cnt++;
                            }
                        }
                    }
                }
            }
        }
        int tot;
        const int pos = base + pfw::excl_scan_i(cnt, &tot);
        if (k < nl && k == P.lp[f]) E.fhead[f] = (int16_t)pos;  // ring of f starts here
        if (pos + cnt <= C::CP) {
            if (cnt > 0) { E.ppx[pos] = x0; E.ppy[pos] = y0; E.ppz[pos] = z0; E.pfl[pos] = (uint8_t)fl0; E.pfac[pos] = (uint8_t)f; }
            if (cnt > 1) { E.ppx[pos + 1] = x1; E.ppy[pos + 1] = y1; E.ppz[pos + 1] = z1; E.pfl[pos + 1] = (uint8_t)fl1; E.pfac[pos + 1] = (uint8_t)f; }
            if (cnt > 2) { E.ppx[pos + 2] = x2; E.ppy[pos + 2] = y2; E.ppz[pos + 2] = z2; E.pfl[pos + 2] = (uint8_t)fl2; E.pfac[pos + 2] = (uint8_t)f; }
        }
        base += tot;
    }
    if (base > C::CP) { pfw::sync(); return 2; }
    if (L == 0) { E.fhead[nf] = (int16_t)base; E.npool = base; }
    pfw::sync();
    // C. per facet: ring range; no point -> full circle or outside
    // (_kernels.py:590-607); fewer than 2 -> outside; the facet frame
    bool ovf = false;
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        int kind = E.fkind[f];
        const int np = E.fhead[f + 1] - E.fhead[f];
        E.fnp[f] = (int16_t)np;
        if (kind == RF_OUTSIDE) continue;
        const double nx = P.nx[f], ny = P.ny[f], nz = P.nz[f];
        double eb[6];
        perp_basis(nx, ny, nz, eb);
        if (kind == RF_GENPOLY) {
            if (np > REF_MAX_P) ovf = true;
            if (np == 0) {
                const double s = E.fh[f];
                const double qx = px + s * nx, qy = py + s * ny, qz = pz + s * nz;
                const int start = P.lp[f], m = P.lp[f + 1] - start;
                bool cin = true;
                #pragma unroll 1
                for (int e = 0; e < m; e++) {
                    int a = P.lv[start + e];
                    int bb = P.lv[start + (e + 1 == m ? 0 : e + 1)];
                    double p0u = (P.x[a] - qx) * eb[0] + (P.y[a] - qy) * eb[1] + (P.z[a] - qz) * eb[2];
                    double p0v = (P.x[a] - qx) * eb[3] + (P.y[a] - qy) * eb[4] + (P.z[a] - qz) * eb[5];
                    double p1u = (P.x[bb] - qx) * eb[0] + (P.y[bb] - qy) * eb[1] + (P.z[bb] - qz) * eb[2];
                    double p1v = (P.x[bb] - qx) * eb[3] + (P.y[bb] - qy) * eb[4] + (P.z[bb] - qz) * eb[5];
                    if ((p1u - p0u) * (-p0v) - (p1v - p0v) * (-p0u) < 0.0) { cin = false; break; }
                }
                kind = cin ? RF_FULLCIRCLE : RF_OUTSIDE;
            } else if (np < 2) {
                kind = RF_OUTSIDE;
            }
            E.fkind[f] = (uint8_t)kind;
        }
        #pragma unroll
        for (int t = 0; t < 6; t++) E.fe[t][f] = eb[t];
    }
    if (pfw::any(ovf)) return 1;
    pfw::sync();
    // D. a point is followed by an arc iff it exits the ball or the next point
    // enters it (_kernels.py:575-587, incl. the ring-closing first entry);
    // zero-length segment connectors are merge candidates (_kernels.py:612-636)
    const int npool = base;
    bool any_cand = false;
    #pragma unroll 1
    for (int q0 = 0; q0 < npool; q0 += 32) {
        const int q = q0 + L;
        int nfl = -1;
        if (q < npool) {
            const int f = E.pfac[q];
            if (E.fkind[f] == RF_GENPOLY) {
                const int head = E.fhead[f], np = E.fnp[f];
                const int j = q + 1 < head + np ? q + 1 : head;
                nfl = E.pfl[q];
                if (E.pfl[j] & PF_ENTRY) nfl |= PF_CONN;
                if (!(nfl & PF_CONN)) {
                    const double dxp = E.ppx[q] - E.ppx[j], dyp = E.ppy[q] - E.ppy[j], dzp = E.ppz[q] - E.ppz[j];
                    if (dxp * dxp + dyp * dyp + dzp * dzp <= tol * tol) { any_cand = true; E.fmrg[f] = 1; }
                }
            }
        }
        pfw::sync();
        if (nfl >= 0) E.pfl[q] = (uint8_t)nfl;
        pfw::sync();
    }
    if (pfw::any(any_cand)) {
        // sequential merge of the facets that have a candidate (rare)
        #pragma unroll 1
        for (int f = L; f < nf; f += 32) {
            if (!E.fmrg[f] || E.fkind[f] != RF_GENPOLY) continue;
            const int head = E.fhead[f], np = E.fnp[f];
            int kept = 0;
            #pragma unroll 1
            for (int t = 0; t < np; t++) {
                const int i = head + t, j = t + 1 < np ? i + 1 : head;
                const bool jdel = (E.pfl[j] & PF_DEL) != 0;  // only the wrap to a merged head
                const double dxp = E.ppx[i] - E.ppx[j], dyp = E.ppy[i] - E.ppy[j], dzp = E.ppz[i] - E.ppz[j];
                if (!(E.pfl[i] & PF_CONN) && !jdel && dxp * dxp + dyp * dyp + dzp * dzp <= tol * tol) {
                    if (E.pfl[i] & PF_ONSPH) E.pfl[j] |= PF_ONSPH;
                    E.pfl[i] |= PF_DEL;
                } else {
                    kept++;
                }
            }
            if (kept < np) {
                int w = head;
                #pragma unroll 1
                for (int t = 0; t < np; t++) {
                    const int i = head + t;
                    if (E.pfl[i] & PF_DEL) continue;
                    E.ppx[w] = E.ppx[i]; E.ppy[w] = E.ppy[i]; E.ppz[w] = E.ppz[i]; E.pfl[w] = E.pfl[i];
                    w++;
                }
                #pragma unroll 1
                for (; w < head + np; w++) E.pfac[w] = PF_DEAD;
                E.fnp[f] = (int16_t)kept;
                if (kept < 2) E.fkind[f] = RF_OUTSIDE;
            }
        }
        pfw::sync();
    }
    return 0;
}

// Degenerate arcs.  When a loop vertex sits within tolerance of the sphere,
// the reference can emit an arc connector whose two end points coincide to
// ~tol but come out in clockwise order; its sweep then wraps from ~-1e-9 to
// ~2 pi (_kernels.py:696-700 and 919-921), adding a whole disk / cap to the
// facet.  A long arc must pass through the antipode of its start point on the
// facet circle, so when that antipode lies outside the cell the arc can only
// be the short one.  This test only fires for end points closer than
// PF_ARC_CHORD * tol and only flips sweeps the geometry proves impossible
// (see tests/test_degenerate_arcs.py: Monte-Carlo volumes of such cells).
#define PF_ARC_CHORD 100.0
// below this sweep (rad) an arc's wrap is decided with the reference's formula
#define PF_SWEEP_AMBIG 1e-6
// (never called in parity mode: the reference keeps the wrapped sweep)
template <class C>
PF_HELPER bool long_arc_impossible(const Poly<C> &P, int f, double qx, double qy, double qz,
                                double dx, double dy, double dz, double rc, double tol) {
    double dn = dsqrt(dx * dx + dy * dy + dz * dz);
    if (!(dn > 0.0)) return false;
    double k = ddiv(rc, dn);
    double mx = qx - k * dx, my = qy - k * dy, mz = qz - k * dz;
    #pragma unroll 1
    for (int g = 0; g < P.nf; g++) {
        if (g == f) continue;
        if (P.nx[g] * mx + P.ny[g] * my + P.nz[g] * mz - P.d[g] > tol) return true;
    }
    return false;
}

// value-only normalisation (tangents): hardware rsqrt + one Newton step
PF_DEV double rsqrt_nr(double x) {
    double r = rsqrt(x);
    return r * fma(-0.5 * x * r, r, 1.5);
}

// boundary point q of a live ring: its facet, else -1
template <class C>
PF_DEV int ring_facet(const EvalScratch<C> &E, int q, bool need_area) {
    if (q >= E.npool) return -1;
    const int f = E.pfac[q];
    if (f == PF_DEAD) return -1;
    const int k = E.fkind[f];
    if (k != RF_GENPOLY && k != RF_UNTOUCHED) return -1;
    if (need_area && !(E.farea[f] > 0.0)) return -1;
    return f;
}

// first lane of this lane's run of equal keys / whether it is the run's last
// lane (runs of equal keys are contiguous in lane order)
PF_DEV int seg_first(int key) {
    const int prev = pfw::shfl(key, (pfw::lane() - 1) & 31);
    const unsigned heads = pfw::ballot(pfw::lane() == 0 || prev != key);
    return pfw::msb(heads & (0xffffffffu >> (31 - pfw::lane())));
}
PF_DEV bool seg_last(int key) {
    const int next = pfw::shfl(key, (pfw::lane() + 1) & 31);
    return pfw::lane() == 31 || next != key;
}

// _kernels.py:678-716 + 331-390: area, first moments and polar moment of the
// restricted facets, lane per boundary connector (point -> ring successor),
// summed per facet.  Same Green forms as the reference; an arc's
// trigonometric values come from its end-point coordinates (cos a = x/r,
// sin a = y/r, double-angle identities) and its sweep from one atan2 of
// (cross, dot), instead of 2 atan2 + 8 sin/cos per arc.  Agrees with the
// reference to rounding.
template <class W>
PF_PHASE void ring_integrals(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                             double tol) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    #pragma unroll 1
    for (int f = L; f < P.nf; f += 32) { E.farea[f] = 0.0; E.fcx[f] = 0.0; E.fcy[f] = 0.0; E.fip[f] = 0.0; }
    pfw::sync();
    const int npool = E.npool;
    #pragma unroll 1
    for (int q0 = 0; q0 < npool; q0 += 32) {
        const int q = q0 + L;
        const int f = ring_facet(E, q, false);
        double A = 0.0, Mx = 0.0, My = 0.0, Ip = 0.0;
        if (f >= 0) {
            const int head = E.fhead[f], np = E.fnp[f];
            const int j = q + 1 < head + np ? q + 1 : head;
            const double e0 = E.fe[0][f], e1 = E.fe[1][f], e2 = E.fe[2][f];
            const double e3 = E.fe[3][f], e4 = E.fe[4][f], e5 = E.fe[5][f];
            const double s = E.fh[f];
            const double qx = px + s * P.nx[f], qy = py + s * P.ny[f], qz = pz + s * P.nz[f];
            const double ax = E.ppx[q] - qx, ay = E.ppy[q] - qy, az = E.ppz[q] - qz;
            const double bx = E.ppx[j] - qx, by = E.ppy[j] - qy, bz = E.ppz[j] - qz;
            const double x0 = ax * e0 + ay * e1 + az * e2, y0 = ax * e3 + ay * e4 + az * e5;
            const double x1 = bx * e0 + by * e1 + bz * e2, y1 = bx * e3 + by * e4 + bz * e5;
            if (!(E.pfl[q] & PF_CONN)) {
                const double cr = fma(x0, y1, -x1 * y0);
                A = 0.5 * cr;
                const double dx = x1 - x0, dy = y1 - y0;
                const double xx = fma(x0, x0, fma(x0, x1, x1 * x1));
                const double yy = fma(y0, y0, fma(y0, y1, y1 * y1));
                Mx = dy * xx * (1.0 / 6.0);
                My = -dx * yy * (1.0 / 6.0);
                const double sx3 = (x0 + x1) * (x0 * x0 + x1 * x1);
                const double sy3 = (y0 + y1) * (y0 * y0 + y1 * y1);
                Ip = fma(dy, sx3, -dx * sy3) * (1.0 / 12.0);
            } else {
                const double r = E.frc[f];
                // cos / sin of the end-point angles (values only: rsqrt + one Newton step)
                const double q0 = x0 * x0 + y0 * y0, q1 = x1 * x1 + y1 * y1;
                const double ir0 = q0 > 0.0 ? rsqrt_nr(q0) : 0.0, ir1 = q1 > 0.0 ? rsqrt_nr(q1) : 0.0;
                const double c0 = q0 > 0.0 ? x0 * ir0 : 1.0, s0 = y0 * ir0;
                const double c1 = q1 > 0.0 ? x1 * ir1 : 1.0, s1 = y1 * ir1;
                double dth = atan2_val(fma(x0, y1, -y0 * x1), fma(x0, x1, y0 * y1));
                // end points (nearly) coincident: decide the wrap exactly as the
                // reference does, from the two end-point angles (_kernels.py:696-700)
                if (fabs(dth) < PF_SWEEP_AMBIG) dth = atan2_ool(y1, x1) - atan2_ool(y0, x0);
                if (dth <= 0.0) {
                    dth += 2.0 * PF_PI;
                    const double ch2 = (x1 - x0) * (x1 - x0) + (y1 - y0) * (y1 - y0);
                    if (!ws->strict && ch2 <= (PF_ARC_CHORD * tol) * (PF_ARC_CHORD * tol) &&
                        long_arc_impossible(P, f, qx, qy, qz, x0 * e0 + y0 * e3, x0 * e1 + y0 * e4,
                                            x0 * e2 + y0 * e5, r, tol))
                        dth -= 2.0 * PF_PI;
                }
                const double s20 = 2.0 * s0 * c0, c20 = fma(c0, c0, -s0 * s0);
                const double s21 = 2.0 * s1 * c1, c21 = fma(c1, c1, -s1 * s1);
                const double s40 = 2.0 * s20 * c20, s41 = 2.0 * s21 * c21;
                const double ic3 = (s1 - s1 * s1 * s1 * (1.0 / 3.0)) - (s0 - s0 * s0 * s0 * (1.0 / 3.0));
                const double is3 = (-c1 + c1 * c1 * c1 * (1.0 / 3.0)) - (-c0 + c0 * c0 * c0 * (1.0 / 3.0));
                const double ic4 = 0.375 * dth + 0.25 * (s21 - s20) + (s41 - s40) / 32.0;
                const double is4 = 0.375 * dth - 0.25 * (s21 - s20) + (s41 - s40) / 32.0;
                const double r2 = r * r;
                A = 0.5 * r2 * dth;
                Mx = 0.5 * r * r2 * ic3;
                My = 0.5 * r * r2 * is3;
                Ip = r * (1.0 / 3.0) * r2 * r * (ic4 + is4);
            }
        }
        const int rs = seg_first(f);
        const bool last = seg_last(f);
        A = pfw::seg_sum_d(A, rs);
        Mx = pfw::seg_sum_d(Mx, rs);
        My = pfw::seg_sum_d(My, rs);
        Ip = pfw::seg_sum_d(Ip, rs);
        if (f >= 0 && last) { E.farea[f] += A; E.fcx[f] += Mx; E.fcy[f] += My; E.fip[f] += Ip; }
        pfw::sync();
    }
}

// _kernels.py:819-835
PF_HELPER void project_from(double cx, double cy, double cz, double yx, double yy, double yz,
                         double px, double py, double pz, double psi, double *o) {
    double dx = yx - cx, dy = yy - cy, dz = yz - cz;
    double a = dx * dx + dy * dy + dz * dz;
    double wx = cx - px, wy = cy - py, wz = cz - pz;
    double b = dx * wx + dy * wy + dz * wz;
    double c0 = wx * wx + wy * wy + wz * wz - psi;
    double disc = b * b - a * c0;
    if (disc < 0.0) disc = 0.0;
    // values only: reciprocal instead of an IEEE division (<= 1 ulp apart)
    double t = (-b + dsqrt(disc)) * __drcp_rn(a);
    o[0] = cx + t * dx; o[1] = cy + t * dy; o[2] = cz + t * dz;
}

PF_DEV void cross3(const double *a, const double *b, double *o) {
    o[0] = fma(a[1], b[2], -a[2] * b[1]);
    o[1] = fma(a[2], b[0], -a[0] * b[2]);
    o[2] = fma(a[0], b[1], -a[1] * b[0]);
}
PF_DEV double dot3(const double *a, const double *b) { return fma(a[0], b[0], fma(a[1], b[1], a[2] * b[2])); }
// CCW angle from a to b around the unit axis m, in [0, 2 pi)
PF_DEV double ccw_angle(const double *a, const double *b, const double *m) {
    double c[3];
    cross3(a, b, c);
    double t = atan2_val(dot3(c, m), dot3(a, b));
    return t < 0.0 ? t + 2.0 * PF_PI : t;
}
PF_DEV void unit3(double *v) {
    double n2 = dot3(v, v);
    if (n2 > 0.0) {
        double inv = rsqrt_nr(n2);
        v[0] *= inv; v[1] *= inv; v[2] *= inv;
    }
}
// the CCW angle from a to b about m is <= the one from a to c (+1e-12 slack
// of the reference's phase comparison, _kernels.py:935-938), without atan2:
// compare half-turns, then the orientation of (b, c)
PF_DEV bool ccw_le(const double *a, const double *b, const double *c, const double *m) {
    double t[3];
    cross3(a, b, t);
    const double sb = dot3(t, m), cb = dot3(a, b);
    cross3(a, c, t);
    const double sc = dot3(t, m), cc = dot3(a, c);
    // half-plane index: 0 for angles in [0, pi), 1 for [pi, 2 pi)
    const int hb = (sb > 0.0 || (sb == 0.0 && cb > 0.0)) ? 0 : 1;
    const int hc = (sc > 0.0 || (sc == 0.0 && cc > 0.0)) ? 0 : 1;
    if (hb != hc) return hb < hc;
    cross3(b, c, t);
    return dot3(t, m) >= 0.0;
}

// Circle carrying connector i -> j of facet f on the sphere, seen from the
// interior point c (_kernels.py:870-946): an arc lies on the facet circle
// (axis n_f, offset s_f); a segment projects onto the circle of the plane
// through c, i and j, oriented so that the projection runs counter-clockwise.
// Returns whether the connector contributes; *uns is set when it is unstable.
// The reference decides the segment orientation with the projected midpoint;
// the rays from c (inside the circle) to the segment sweep less than a half
// turn counter-clockwise about m = (i - c) x (j - c), and central projection
// keeps that order, so the test can only fail when the sweep is within
// rounding of 0 or pi: it is evaluated when sin^2 of the sweep is < 1e-6.
template <class C>
PF_HELPER int conn_circle(const EvalScratch<C> &E, int i, int j, bool arc, double nfx, double nfy,
                         double nfz, double sf, double cx, double cy, double cz, double px,
                         double py, double pz, double psi, double *m, double *ee, bool *uns) {
    if (arc) {
        m[0] = nfx; m[1] = nfy; m[2] = nfz; *ee = sf;
        if (psi - sf * sf <= 0.0) { *uns = true; return 0; }
        return 1;
    }
    const double a3[3] = {E.ppx[i] - cx, E.ppy[i] - cy, E.ppz[i] - cz};
    const double b3[3] = {E.ppx[j] - cx, E.ppy[j] - cy, E.ppz[j] - cz};
    cross3(a3, b3, m);
    const double mn2 = dot3(m, m);
    if (!(mn2 > 0.0)) { *uns = true; return 0; }  // |m| < 1e-300 (reference) <=> |m|^2 underflows to 0
    const double im = rsqrt_nr(mn2);
    m[0] *= im; m[1] *= im; m[2] *= im;
    double e = m[0] * (cx - px) + m[1] * (cy - py) + m[2] * (cz - pz);
    *ee = e;
    if (psi - e * e <= 0.0) { *uns = true; return 0; }
    if (mn2 <= 1e-6 * dot3(a3, a3) * dot3(b3, b3)) {
        const double q[3] = {px + e * m[0], py + e * m[1], pz + e * m[2]};
        const double rp[3] = {E.prx[i] - q[0], E.pry[i] - q[1], E.prz[i] - q[2]};
        const double rq[3] = {E.prx[j] - q[0], E.pry[j] - q[1], E.prz[j] - q[2]};
        double h[3];
        project_from(cx, cy, cz, 0.5 * (E.ppx[i] + E.ppx[j]), 0.5 * (E.ppy[i] + E.ppy[j]),
                     0.5 * (E.ppz[i] + E.ppz[j]), px, py, pz, psi, h);
        const double rm[3] = {h[0] - q[0], h[1] - q[1], h[2] - q[2]};
        if (!ccw_le(rp, rm, rq, m)) {
            // traversal is clockwise around m: flip the circle normal, retry once
            m[0] = -m[0]; m[1] = -m[1]; m[2] = -m[2]; *ee = -e;
            if (!ccw_le(rp, rm, rq, m)) return 0;
        }
    }
    return 1;
}

// _kernels.py:838-1001, lane per boundary point.  Gauss-Bonnet:
// area = psi (2 pi - sum_arcs (e/R) sweep - sum_vertices theta).  Lane q owns
// the connector q -> succ(q) (its sweep, a CCW angle about the connector
// circle's axis from one atan2 of (cross, dot)) and the turning angle at q
// (from the end tangent of pred(q) -> q and the start tangent of its own
// connector).  Per facet: E.fpa = the clamped patch area, E.funs = unstable.
template <class W>
PF_PHASE void ring_patches(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                           double psi, double R, double tol, double cx, double cy, double cz) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    const double iR = ddiv(1.0, R);
    const int npool = E.npool;
    // central projections of the boundary points from c (_kernels.py:880-898)
    #pragma unroll 1
    for (int q = L; q < npool; q += 32) {
        if (ring_facet(E, q, true) < 0) continue;
        if (E.pfl[q] & PF_ONSPH) { E.prx[q] = E.ppx[q]; E.pry[q] = E.ppy[q]; E.prz[q] = E.ppz[q]; }
        else {
            double o[3];
            project_from(cx, cy, cz, E.ppx[q], E.ppy[q], E.ppz[q], px, py, pz, psi, o);
            E.prx[q] = o[0]; E.pry[q] = o[1]; E.prz[q] = o[2];
        }
    }
    #pragma unroll 1
    for (int f = L; f < P.nf; f += 32) { E.fpa[f] = 0.0; E.funs[f] = 0; }
    pfw::sync();
    #pragma unroll 1
    for (int q0 = 0; q0 < npool; q0 += 32) {
        const int q = q0 + L;
        const int f = ring_facet(E, q, true);
        double term = 0.0, unst = 0.0;
        if (f >= 0) {
            const int head = E.fhead[f], np = E.fnp[f];
            const int j = q + 1 < head + np ? q + 1 : head;
            const int pq = q > head ? q - 1 : head + np - 1;
            const double nfx = P.nx[f], nfy = P.ny[f], nfz = P.nz[f], sf = E.fh[f];
            const double prq[3] = {E.prx[q], E.pry[q], E.prz[q]};
            bool uns = false;
            double m[3], ee;
            double tout[3] = {0.0, 0.0, 0.0}, tin[3] = {0.0, 0.0, 0.0};
            const bool arc = (E.pfl[q] & PF_CONN) != 0;
            if (conn_circle(E, q, j, arc, nfx, nfy, nfz, sf, cx, cy, cz, px, py, pz, psi, m, &ee, &uns)) {
                const double qc[3] = {px + ee * m[0], py + ee * m[1], pz + ee * m[2]};
                const double rp[3] = {prq[0] - qc[0], prq[1] - qc[1], prq[2] - qc[2]};
                const double rq[3] = {E.prx[j] - qc[0], E.pry[j] - qc[1], E.prz[j] - qc[2]};
                double dPQ = ccw_angle(rp, rq, m);
                if (arc && (dPQ < PF_SWEEP_AMBIG || dPQ > 2.0 * PF_PI - PF_SWEEP_AMBIG)) {
                    // (nearly) coincident end points: the reference's frame angles
                    // phQ - phP decide whether the arc wraps (_kernels.py:908-923)
                    double u[6];
                    perp_basis(m[0], m[1], m[2], u);
                    const double phP = atan2_ool(rp[0] * u[3] + rp[1] * u[4] + rp[2] * u[5],
                                                 rp[0] * u[0] + rp[1] * u[1] + rp[2] * u[2]);
                    const double phQ = atan2_ool(rq[0] * u[3] + rq[1] * u[4] + rq[2] * u[5],
                                                 rq[0] * u[0] + rq[1] * u[1] + rq[2] * u[2]);
                    dPQ = phQ - phP;
                    if (dPQ < 0.0) dPQ += 2.0 * PF_PI;
                }
                if (arc && dPQ > PF_PI) {
                    const double d0 = rp[0] - rq[0], d1 = rp[1] - rq[1], d2 = rp[2] - rq[2];
                    if (!ws->strict && d0 * d0 + d1 * d1 + d2 * d2 <= (PF_ARC_CHORD * tol) * (PF_ARC_CHORD * tol) &&
                        long_arc_impossible(P, f, qc[0], qc[1], qc[2], rp[0], rp[1], rp[2],
                                            dsqrt(psi - ee * ee), tol))
                        dPQ -= 2.0 * PF_PI;
                }
                term = ee * iR * dPQ;
                cross3(m, rp, tout);
                unit3(tout);
            }
            const bool parc = (E.pfl[pq] & PF_CONN) != 0;
            if (conn_circle(E, pq, q, parc, nfx, nfy, nfz, sf, cx, cy, cz, px, py, pz, psi, m, &ee, &uns)) {
                const double rq[3] = {prq[0] - (px + ee * m[0]), prq[1] - (py + ee * m[1]),
                                      prq[2] - (pz + ee * m[2])};
                cross3(m, rq, tin);
                unit3(tin);
            }
            // turning angle at q
            double cr[3];
            cross3(tin, tout, cr);
            const double nv[3] = {(prq[0] - px) * iR, (prq[1] - py) * iR, (prq[2] - pz) * iR};
            const double th = atan2_val(dot3(cr, nv), dot3(tin, tout));
            if (fabs(th) > PF_PI - 1e-7) uns = true;
            term += th;
            unst = uns ? 1.0 : 0.0;
        }
        const int rs = seg_first(f);
        const bool last = seg_last(f);
        term = pfw::seg_sum_d(term, rs);
        unst = pfw::seg_sum_d(unst, rs);
        if (f >= 0 && last) { E.fpa[f] += term; if (unst > 0.0) E.funs[f] = 1; }
        pfw::sync();
    }
    #pragma unroll 1
    for (int f = L; f < P.nf; f += 32) {
        const int k = E.fkind[f];
        if (!((k == RF_GENPOLY || k == RF_UNTOUCHED) && E.farea[f] > 0.0)) continue;
        double area = psi * (2.0 * PF_PI - E.fpa[f]);
        if (area < -1e-9 * PF_FOUR_PI * psi || area > PF_FOUR_PI * psi * (1.0 + 1e-9)) E.funs[f] = 1;
        if (area < 0.0) area = 0.0;
        if (area > PF_FOUR_PI * psi) area = PF_FOUR_PI * psi;
        E.fpa[f] = area;
    }
    pfw::sync();
}

// result of one cell evaluation (uniform across the warp)
struct CellRes {
    int status;
    double vol, K, cx, cy, cz, ix, iy, iz, m2;
    int flags;
};

// Evaluation state of one cell between the phases below (uniform across the
// warp).  The phases are separate functions so that a kernel can run them
// block-synchronously: all warps of a block then execute the same phase and
// share its instructions (the whole evaluation does not fit the instruction
// cache; warps in different phases thrash it).
struct EvalState {
    double R, kbar;
    double ix, iy, iz, bx, by, bz;
    int done;     // res is final
    int attempt;  // next projection attempt (4: finished)
};

// _kernels.py:1008-1026: defaults, vertex-in-ball flags, twin-facet table
template <class W>
PF_PHASE void eval_setup(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                         double psi, double tol, CellRes *res, EvalState *st) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    const int nf = P.nf;
    res->flags = 0;
    res->status = CELL_EMPTY; res->vol = 0.0; res->K = 0.0;
    res->cx = px; res->cy = py; res->cz = pz; res->ix = px; res->iy = py; res->iz = pz; res->m2 = 0.0;
    st->done = 0; st->attempt = 0; st->kbar = 0.0;
    if (psi <= 0.0) { st->done = 1; return; }
    const double R = dsqrt(psi);
    st->R = R;
    const double ball_tol = tol * (2.0 * R + tol);
    #pragma unroll 1
    for (int v = L; v < P.nv; v += 32) {
        double wx = P.x[v] - px, wy = P.y[v] - py, wz = P.z[v] - pz;
        double q = wx * wx + wy * wy + wz * wz - psi;
        E.vin[v] = q <= ball_tol ? 1 : 0;
        E.vdeg[v] = 0;
    }
    // loop-entry facet and successor vertex, for the twin-facet table
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        const int s0 = P.lp[f], m = P.lp[f + 1] - s0;
        #pragma unroll 1
        for (int e = 0; e < m; e++) {
            E.efac[s0 + e] = (uint8_t)f;
            E.esv[s0 + e] = P.lv[s0 + (e + 1 == m ? 0 : e + 1)];
        }
    }
    pfw::sync();
    #pragma unroll 1
    for (int k = L; k < P.nl; k += 32) {
        const int a = P.lv[k];
        const int slot = pfw::atom_add_u8(&E.vdeg[a]);
        if (slot < 4) E.vinc[a * 4 + slot] = (uint16_t)k;
    }
    pfw::sync();
}

// restriction of every facet (_kernels.py:1027-1040)
template <class W>
PF_PHASE void eval_restrict(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                            double psi, double tol, CellRes *res, EvalState *st) {
    const int rst = restrict_all(ws, P, px, py, pz, psi, st->R, tol);
    if (rst == 2) {
        if (pfw::lane() == 0) ws->oflow = 1;
        pfw::sync();
        res->flags = FLAG_RETRY;
        st->done = 1;
    } else if (rst == 1) {  // reference: first facet with kind < 0 aborts the cell
        res->flags = FLAG_OVERFLOW;
        st->done = 1;
    }
}

// facet integrals, full-ball / empty decision (_kernels.py:1041-1092)
template <class W>
PF_PHASE void eval_integrals(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                             double psi, double tol, int want_m2, CellRes *res, EvalState *st) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    const int nf = P.nf;
    ring_integrals(ws, P, px, py, pz, tol);
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        const int kind = E.fkind[f];
        const double s = E.fh[f];
        const double qx = px + s * P.nx[f], qy = py + s * P.ny[f], qz = pz + s * P.nz[f];
        if (kind == RF_FULLCIRCLE) {
            const double rc = E.frc[f], rc2 = rc * rc;
            E.farea[f] = PF_PI * rc2;
            E.fcx[f] = qx; E.fcy[f] = qy; E.fcz[f] = qz;
            E.fip[f] = 0.5 * PF_PI * (rc2 * rc2);
        } else if (kind != RF_OUTSIDE && E.farea[f] > 0.0) {
            const double ia = ddiv(1.0, E.farea[f]);
            const double u = E.fcx[f] * ia, v = E.fcy[f] * ia;
            E.fcx[f] = qx + u * E.fe[0][f] + v * E.fe[3][f];
            E.fcy[f] = qy + u * E.fe[1][f] + v * E.fe[4][f];
            E.fcz[f] = qz + u * E.fe[2][f] + v * E.fe[5][f];
        } else {
            E.fkind[f] = RF_OUTSIDE;
            E.farea[f] = 0.0; E.fcx[f] = px; E.fcy[f] = py; E.fcz[f] = pz; E.fip[f] = 0.0;
        }
    }
    pfw::sync();
    if (cen_on(ws)) {
        int cross = 0, seg = 0, arc = 0, bp = 0, proj = 0, fc = 0;
        #pragma unroll 1
        for (int f = L; f < nf; f += 32) fc += E.fkind[f] == RF_FULLCIRCLE;
        #pragma unroll 1
        for (int q = L; q < E.npool; q += 32) {
            if (ring_facet(E, q, false) < 0) continue;
            bp++;
            if (E.pfl[q] & PF_ONSPH) cross++; else proj++;
            if (E.pfl[q] & PF_CONN) arc++; else seg++;
        }
        cross = pfw::sum_i(cross); seg = pfw::sum_i(seg); arc = pfw::sum_i(arc);
        bp = pfw::sum_i(bp); proj = pfw::sum_i(proj); fc = pfw::sum_i(fc);
        if (L == 0) {
            ws->cen[CEN_LOOP] += P.nl; ws->cen[CEN_CROSS] += cross; ws->cen[CEN_SEG] += seg;
            ws->cen[CEN_ARC] += arc; ws->cen[CEN_BPTS] += bp; ws->cen[CEN_PROJ] += proj;
            ws->cen[CEN_FULLC] += fc;
        }
        pfw::sync();
    }
    bool any_area = false;
    #pragma unroll 1
    for (int f0 = 0; f0 < nf; f0 += 32) {
        int f = f0 + L;
        any_area |= pfw::any(f < nf && E.fkind[f] != RF_OUTSIDE && E.farea[f] > 0.0);
    }
    // NB: reference sets any_present before the A <= 0 demotion; a demoted
    // GENPOLY still counts as "present" there.  Demotion always comes with
    // area 0, so (any_present && any_area) == any_area except for that case,
    // which the full-ball/empty branch below treats identically.
    if (!any_area) {
        bool inside = true;
        #pragma unroll 1
        for (int f0 = 0; f0 < nf; f0 += 32) {
            int f = f0 + L;
            inside &= !pfw::any(f < nf && E.fh[f] < -tol);
        }
        if ((inside && nf > 0) || nf == 0) {
            const double R = st->R;
            res->status = CELL_FULLBALL;
            res->vol = PF_FOUR_PI / 3.0 * psi * R;
            res->K = PF_FOUR_PI * psi;
            res->m2 = want_m2 ? PF_FOUR_PI * psi * R * R * R / 5.0 : 0.0;
        }
        st->done = 1;
    }
}

// interior point (_kernels.py:723-816): ray per restricted facet, lane per
// facet; the ray midpoints and margins reuse the facet-frame slots
template <class W>
PF_PHASE void eval_interior(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                            double psi, double tol, CellRes *res, EvalState *st) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    const int nf = P.nf;
    double *smx = E.fe[0], *smy = E.fe[1], *smz = E.fe[2], *smg = E.fe[3];
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        E.fseg[f] = 0;
        if (E.fkind[f] == RF_OUTSIDE || E.farea[f] <= 0.0) continue;
        double ox = E.fcx[f], oy = E.fcy[f], oz = E.fcz[f];
        double dx = -P.nx[f], dy = -P.ny[f], dz = -P.nz[f];
        double wx = ox - px, wy = oy - py, wz = oz - pz;
        double bh = dx * wx + dy * wy + dz * wz;
        double cc = wx * wx + wy * wy + wz * wz - psi;
        double disc = bh * bh - cc;
        if (disc <= 0.0) continue;
        // ray [t_lo, t_hi] inside every other facet plane; the extreme ratios
        // num/den are tracked as fractions (positive denominators), one
        // division each at the end instead of one per plane
        double hn = -bh + dsqrt(disc), hd = 1.0;  // t_hi = hn / hd
        double ln = 0.0, ld = 1.0;                // t_lo = ln / ld
        bool ok = true;
        #pragma unroll 1
        for (int g = 0; g < nf; g++) {
            if (g == f) continue;
            double den = P.nx[g] * dx + P.ny[g] * dy + P.nz[g] * dz;
            double num = P.d[g] - (P.nx[g] * ox + P.ny[g] * oy + P.nz[g] * oz);
            if (den > tol) {
                if (num * hd < hn * den) { hn = num; hd = den; }
            } else if (den < -tol) {
                if (-num * ld > ln * -den) { ln = -num; ld = -den; }
            } else if (num < -tol) {
                ok = false;
                break;
            }
        }
        if (!ok) continue;
        const double t_hi = hd == 1.0 ? hn : ddiv(hn, hd);
        const double t_lo = ld == 1.0 ? ln : ddiv(ln, ld);
        if (t_hi - t_lo <= tol) continue;
        double tm = 0.5 * (t_lo + t_hi);
        double mx = ox + tm * dx, my = oy + tm * dy, mz = oz + tm * dz;
        double mg = st->R - dsqrt(sq(mx - px) + sq(my - py) + sq(mz - pz));  // st->R == dsqrt(psi)
        #pragma unroll 1
        for (int g = 0; g < nf; g++) {
            double d2 = P.d[g] - (P.nx[g] * mx + P.ny[g] * my + P.nz[g] * mz);
            if (d2 < mg) mg = d2;
        }
        E.fseg[f] = 1;
        smx[f] = mx; smy[f] = my; smz[f] = mz; smg[f] = mg;
    }
    pfw::sync();
    // average of the ray midpoints and the deepest one (first on ties)
    double sx = 0.0, sy = 0.0, sz = 0.0, bm = -1.0;
    int nseg = 0, bf = -1;
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        if (!E.fseg[f]) continue;
        sx += smx[f]; sy += smy[f]; sz += smz[f];
        nseg++;
        if (smg[f] > bm) { bm = smg[f]; bf = f; }
    }
    sx = pfw::sum_d(sx); sy = pfw::sum_d(sy); sz = pfw::sum_d(sz);
    nseg = pfw::sum_i(nseg);
    // argmax margin, lowest facet index among equal margins
    #pragma unroll 1
    for (int m = 16; m > 0; m >>= 1) {
        double om = pfw::shfl_xor(bm, m);
        int of = pfw::shfl_xor(bf, m);
        if (om > bm || (om == bm && of >= 0 && (bf < 0 || of < bf))) { bm = om; bf = of; }
    }
    const double best_margin = bm;
    st->bx = px; st->by = py; st->bz = pz;
    if (bf >= 0 && best_margin > -1.0) { st->bx = smx[bf]; st->by = smy[bf]; st->bz = smz[bf]; }
    bool ok = nseg > 0;
    if (ok) {
        double inv = ddiv(1.0, (double)nseg);
        double cx = sx * inv, cy = sy * inv, cz = sz * inv;
        double mg = st->R - dsqrt(sq(cx - px) + sq(cy - py) + sq(cz - pz));
        #pragma unroll 1
        for (int g = L; g < nf; g += 32) {
            double d2 = P.d[g] - (P.nx[g] * cx + P.ny[g] * cy + P.nz[g] * cz);
            if (d2 < mg) mg = d2;
        }
        mg = -pfw::max_d(-mg);
        if (mg <= 0.0) {
            if (best_margin > 0.0) { cx = st->bx; cy = st->by; cz = st->bz; }
            else ok = false;
        }
        st->ix = cx; st->iy = cy; st->iz = cz;
    }
    if (!ok) {
        res->flags = FLAG_DEGENERATE_INTERIOR;
        st->done = 1;
    }
}

// one attempt of the occluded areas with perturb-and-retry (_kernels.py:1100-1128)
template <class W>
PF_PHASE void eval_patch_attempt(W *ws, const Poly<typename W::Cap> &P, double px, double py,
                                 double pz, double psi, double tol, CellRes *res, EvalState *st) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    const int nf = P.nf;
    const double R = st->R;
    ring_patches(ws, P, px, py, pz, psi, R, tol, st->ix, st->iy, st->iz);
    // first unstable facet in facet order (the reference stops there)
    int first_bad = nf;
    #pragma unroll 1
    for (int f0 = 0; f0 < nf; f0 += 32) {
        int f = f0 + L;
        unsigned mb = pfw::ballot(f < nf && E.funs[f] &&
                                  !(E.fkind[f] == RF_OUTSIDE || E.fkind[f] == RF_FULLCIRCLE ||
                                    E.farea[f] <= 0.0));
        if (mb && first_bad == nf) first_bad = f0 + __builtin_ctz_pf(mb);
    }
    const bool bad = first_bad < nf;
    double kb = 0.0;
    #pragma unroll 1
    for (int f = L; f < first_bad; f += 32) {
        if (E.fkind[f] == RF_OUTSIDE || E.farea[f] <= 0.0) continue;
        if (E.fkind[f] == RF_FULLCIRCLE) kb += 2.0 * PF_PI * R * (R - E.fh[f]);
        else kb += E.fpa[f];
    }
    st->kbar = pfw::sum_d(kb);
    pfw::sync();
    const int attempt = st->attempt;
    if (!bad) { st->attempt = 4; return; }
    if (attempt == 3) { res->flags |= FLAG_UNSTABLE_PROJECTION; st->attempt = 4; return; }
    double w = 0.35 * (double)(attempt + 1);
    st->ix = st->ix + w * (st->bx - st->ix);
    st->iy = st->iy + w * (st->by - st->iy);
    st->iz = st->iz + w * (st->bz - st->iz);
    st->attempt = attempt + 1;
}

// K, volume, centroid, second moment (_kernels.py:1130-1170)
template <class W>
PF_PHASE void eval_final(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                         double psi, int want_m2, CellRes *res, EvalState *st) {
    using C = typename W::Cap;
    EvalScratch<C> &E = ws->u.e;
    const int L = pfw::lane();
    const int nf = P.nf;
    const double R = st->R;
    double K = PF_FOUR_PI * psi - st->kbar;
    if (K < 0.0) K = 0.0;
    if (K > PF_FOUR_PI * psi) K = PF_FOUR_PI * psi;
    double vol = 0.0;
    double mx = 0.0, my = 0.0, mz = 0.0, nsx = 0.0, nsy = 0.0, nsz = 0.0, m2 = 0.0;
    #pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        if (E.fkind[f] == RF_OUTSIDE || E.farea[f] <= 0.0) continue;
        double fa = E.farea[f], fh = E.fh[f];
        double pv = fh * fa * (1.0 / 3.0);
        vol += pv;
        mx += pv * 0.75 * (E.fcx[f] - px);
        my += pv * 0.75 * (E.fcy[f] - py);
        mz += pv * 0.75 * (E.fcz[f] - pz);
        nsx += P.nx[f] * fa;
        nsy += P.ny[f] * fa;
        nsz += P.nz[f] * fa;
        if (want_m2) m2 += (fh * 0.2) * (E.fip[f] + fh * fh * fa);
    }
    vol = R * K * (1.0 / 3.0) + pfw::sum_d(vol);
    mx = pfw::sum_d(mx); my = pfw::sum_d(my); mz = pfw::sum_d(mz);
    nsx = pfw::sum_d(nsx); nsy = pfw::sum_d(nsy); nsz = pfw::sum_d(nsz);
    m2 = want_m2 ? R * R * R * K * 0.2 + pfw::sum_d(m2) : 0.0;
    mx += 0.25 * psi * (-nsx);
    my += 0.25 * psi * (-nsy);
    mz += 0.25 * psi * (-nsz);
    double ccx, ccy, ccz;
    if (vol > 0.0) { double iv = ddiv(1.0, vol); ccx = px + mx * iv; ccy = py + my * iv; ccz = pz + mz * iv; }
    else { vol = 0.0; ccx = px; ccy = py; ccz = pz; }
    res->status = CELL_CLIPPED;
    res->vol = vol; res->K = K; res->cx = ccx; res->cy = ccy; res->cz = ccz;
    res->ix = st->ix; res->iy = st->iy; res->iz = st->iz; res->m2 = m2;
    st->done = 1;
}

// _kernels.py:1008-1170, all phases in sequence.  Returns with res filled in
// every lane.  On pool overflow sets ws->oflow (fast instantiation).
template <class W>
PF_DEV void evaluate_cell(W *ws, const Poly<typename W::Cap> &P, double px, double py, double pz,
                          double psi, double tol, int want_m2, CellRes *res) {
    EvalState st;
    eval_setup(ws, P, px, py, pz, psi, tol, res, &st);
    if (!st.done) eval_restrict(ws, P, px, py, pz, psi, tol, res, &st);
    if (!st.done) eval_integrals(ws, P, px, py, pz, psi, tol, want_m2, res, &st);
    if (!st.done) eval_interior(ws, P, px, py, pz, psi, tol, res, &st);
    #pragma unroll 1
    while (!st.done && st.attempt < 4) eval_patch_attempt(ws, P, px, py, pz, psi, tol, res, &st);
    if (!st.done) eval_final(ws, P, px, py, pz, psi, want_m2, res, &st);
}

// ---------------------------------------------------------------------------
// one cell end to end (_kernels.py:1374-1474).  Returns the cell's flags;
// FLAG_RETRY means nothing was written and the cell must be re-run on the
// reference-capacity instantiation.
// ---------------------------------------------------------------------------
// Phase A of one cell: build.  Returns -1 when the cell needs evaluation
// (polytope in ws->P[*which]), else the cell's final flag word with its
// outputs already written (empty / overflow), or FLAG_RETRY.
// _batch_build's per-cell output (_kernels.py:1508-1555): status 1 empty
// (counts 0), 3 overflow (build overflow or beyond the caller's strides), 0 ok
template <class W>
PF_NOINL int write_packed(W *ws, const CellOut &out, int i, int st, int which) {
    const int L = pfw::lane();
    const Poly<typename W::Cap> &A = ws->P[which];
    if (st == 1) {
        if (L == 0) { out.pk_status[i] = 1; out.pk_nv[i] = 0; out.pk_nf[i] = 0; out.pk_nl[i] = 0; }
        return 0;
    }
    if (st == 3 || A.nv > out.smv || A.nf > out.smfb || A.nl > out.sml) {
        if (L == 0) out.pk_status[i] = 3;
        return FLAG_OVERFLOW;
    }
    const size_t iv = (size_t)i * out.smv, jf = (size_t)i * out.smfb, kl = (size_t)i * out.sml;
    #pragma unroll 1
    for (int v = L; v < A.nv; v += 32) {
        out.pk_verts[3 * (iv + v)] = A.x[v]; out.pk_verts[3 * (iv + v) + 1] = A.y[v];
        out.pk_verts[3 * (iv + v) + 2] = A.z[v];
    }
    #pragma unroll 1
    for (int f = L; f < A.nf; f += 32) {
        out.pk_planes[4 * (jf + f)] = A.nx[f]; out.pk_planes[4 * (jf + f) + 1] = A.ny[f];
        out.pk_planes[4 * (jf + f) + 2] = A.nz[f]; out.pk_planes[4 * (jf + f) + 3] = A.d[f];
        out.pk_tags[jf + f] = A.tag[f];
    }
    #pragma unroll 1
    for (int f = L; f <= A.nf; f += 32) out.pk_lp[(size_t)i * (out.smfb + 1) + f] = A.lp[f];
    #pragma unroll 1
    for (int k = L; k < A.nl; k += 32) out.pk_lv[kl + k] = A.lv[k];
    if (L == 0) { out.pk_status[i] = 0; out.pk_nv[i] = A.nv; out.pk_nf[i] = A.nf; out.pk_nl[i] = A.nl; }
    return 0;
}

template <class W, bool HV = true>
PF_DEV int cell_phase_build(W *ws, const CellIn &in, const CellOut &out, int i, int *which) {
    const int L = pfw::lane();
    if (L == 0) {
        ws->oflow = 0;
        ws->strict = in.strict;
        ws->cen_on = out.census16 != nullptr;
        if (W::CEN)
#pragma unroll 1
            for (int k = 0; k < 16; k++) ws->cen[k] = 0;
    }
    pfw::sync();
    int nclips;
    int st = build_cell<W, HV>(ws, in, i, which, &nclips);
    if (ws->oflow) {
        pfw::sync();
        if (!W::Cap::EXACT) return FLAG_RETRY;
        st = 3;
    }
    if (out.census && L == 0) out.census[i] = nclips;
    if (HV && out.pk_status) return write_packed(ws, out, i, st, *which);
    const double px = in.pts[3 * i], py = in.pts[3 * i + 1], pz = in.pts[3 * i + 2];
    if (st == 3) {
        if (L == 0) {
            if (out.status) out.status[i] = CELL_EMPTY;
            if (out.vol) out.vol[i] = 0.0;
            if (out.ksur) out.ksur[i] = 0.0;
            if (out.fcount) out.fcount[i] = 0;
            if (out.fcount32) out.fcount32[i] = 0;
        }
        return FLAG_OVERFLOW | FLAG_BUILD_OVERFLOW;
    }
    if (st == 1) {
        if (L == 0) {
            if (out.status) out.status[i] = CELL_EMPTY;
            if (out.vol) out.vol[i] = 0.0;
            if (out.ksur) out.ksur[i] = 0.0;
            if (out.cent) { out.cent[3 * i] = px; out.cent[3 * i + 1] = py; out.cent[3 * i + 2] = pz; }
            if (out.ipt) { out.ipt[3 * i] = px; out.ipt[3 * i + 1] = py; out.ipt[3 * i + 2] = pz; }
            if (out.m2) out.m2[i] = 0.0;
            if (out.fcount) out.fcount[i] = 0;
            if (out.fcount32) out.fcount32[i] = 0;
        }
        return 0;
    }
    return -1;
}

// Phase B: evaluate the polytope in ws->P[which] and write the outputs.
template <class W>
PF_PHASE int eval_write(W *ws, const CellIn &in, const CellOut &out, int i, int which, CellRes r);
template <class W>
PF_DEV int cell_phase_eval(W *ws, const CellIn &in, const CellOut &out, int i, int which) {
    const double px = in.pts[3 * i], py = in.pts[3 * i + 1], pz = in.pts[3 * i + 2];
    CellRes r;
    evaluate_cell(ws, ws->P[which], px, py, pz, in.psi[i], in.tol, in.want_m2, &r);
    return eval_write(ws, in, out, i, which, r);
}
// write one evaluated cell's outputs (_kernels.py:1441-1474); returns its flags
template <class W>
PF_PHASE int eval_write(W *ws, const CellIn &in, const CellOut &out, int i, int which, CellRes r) {
    const int L = pfw::lane();
    const double px = in.pts[3 * i], py = in.pts[3 * i + 1], pz = in.pts[3 * i + 2];
    const Poly<typename W::Cap> &P = ws->P[which];
    if (ws->oflow) {
        pfw::sync();
        if (!W::Cap::EXACT) return FLAG_RETRY;
        // beyond even the reference-capacity pool: report as overflow
        r.flags = FLAG_OVERFLOW;
        r.status = CELL_EMPTY; r.vol = 0.0; r.K = 0.0;
        r.cx = px; r.cy = py; r.cz = pz; r.ix = px; r.iy = py; r.iz = pz; r.m2 = 0.0;
    }
    int flags = r.flags;
    if (L == 0) {
        if (out.status) out.status[i] = r.status;
        if (out.vol) out.vol[i] = r.vol;
        if (out.ksur) out.ksur[i] = r.K;
        if (out.cent) { out.cent[3 * i] = r.cx; out.cent[3 * i + 1] = r.cy; out.cent[3 * i + 2] = r.cz; }
        if (out.ipt) { out.ipt[3 * i] = r.ix; out.ipt[3 * i + 1] = r.iy; out.ipt[3 * i + 2] = r.iz; }
        if (out.m2) out.m2[i] = r.m2;
    }
    // restricted facet summaries in facet order, zero-area facets dropped (_kernels.py:1456-1474)
    int nk = 0;
    if (r.status == CELL_CLIPPED) {
        const EvalScratch<typename W::Cap> &E = ws->u.e;
        const unsigned lt = pfw::lanemask_lt();
        const int smf = out.smf;
        #pragma unroll 1
        for (int f0 = 0; f0 < P.nf; f0 += 32) {
            int f = f0 + L;
            bool keep = f < P.nf && !(E.fkind[f] == RF_OUTSIDE || E.farea[f] <= 0.0);
            unsigned m = pfw::ballot(keep);
            int slot = nk + pfw::popc(m & lt);
            if (keep && slot < smf) {
                size_t o = (size_t)i * smf + slot;
                if (out.ftag) out.ftag[o] = P.tag[f];
                if (out.ftag32) out.ftag32[o] = P.tag[f];
                if (out.farea) out.farea[o] = E.farea[f];
                if (out.fh) out.fh[o] = E.fh[f];
                if (out.fnrm) { out.fnrm[3 * o] = P.nx[f]; out.fnrm[3 * o + 1] = P.ny[f]; out.fnrm[3 * o + 2] = P.nz[f]; }
                if (out.fcent) { out.fcent[3 * o] = E.fcx[f]; out.fcent[3 * o + 1] = E.fcy[f]; out.fcent[3 * o + 2] = E.fcz[f]; }
            }
            nk += pfw::popc(m);
        }
        if (cen_on(ws) && L == 0) { ws->cen[CEN_RFAC] += nk; ws->cen[CEN_RFAC_NF] += nk * P.nf; }
        if (nk > smf) { nk = smf; flags |= FLAG_OVERFLOW; }
    }

    if (L == 0) {
        if (out.fcount) out.fcount[i] = nk;
        if (out.fcount32) out.fcount32[i] = nk;
        if (out.flags) out.flags[i] = flags;
    }
    pfw::sync();
    return flags;
}

template <class W>
PF_DEV int run_cell_impl(W *ws, const CellIn &in, const CellOut &out, int i) {
    int which = 0;
    int r = cell_phase_build(ws, in, out, i, &which);
    if (r >= 0) return r;
    return cell_phase_eval(ws, in, out, i, which);
}

// polytope hand-off between the split build / evaluate kernels (global memory)
template <class C>
PF_DEV void poly_store(const Poly<C> &A, Poly<C> *g) {
    const int L = pfw::lane();
#pragma unroll 1
    for (int v = L; v < A.nv; v += 32) { g->x[v] = A.x[v]; g->y[v] = A.y[v]; g->z[v] = A.z[v]; }
#pragma unroll 1
    for (int f = L; f < A.nf; f += 32) {
        g->nx[f] = A.nx[f]; g->ny[f] = A.ny[f]; g->nz[f] = A.nz[f]; g->d[f] = A.d[f]; g->tag[f] = A.tag[f];
    }
#pragma unroll 1
    for (int f = L; f <= A.nf; f += 32) g->lp[f] = A.lp[f];
#pragma unroll 1
    for (int k = L; k < A.nl; k += 32) g->lv[k] = A.lv[k];
    if (L == 0) { g->nv = A.nv; g->nf = A.nf; g->nl = A.nl; }
}
#ifdef __CUDACC__
// One-lane bulk (TMA) copy of a whole polytope record HBM -> shared memory,
// completion tracked by a per-warp mbarrier (transaction bytes); the record and
// the shared layout are the same Poly<C> (16-byte multiple, 16-byte aligned).
PF_DEV void mbar_init(unsigned long long *mb) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// the same in two halves: issue (every lane done with A), and wait
template <class C>
PF_DEV void poly_load_tma_issue(const Poly<C> *g, Poly<C> &A, unsigned long long *mb) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
    pfw::sync();
    if (pfw::lane() == 0) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&A);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a),
                     "r"((unsigned)sizeof(Poly<C>)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(g), "r"((unsigned)sizeof(Poly<C>)), "r"(a) : "memory");
    }
}
PF_DEV void poly_load_tma_wait(unsigned long long *mb, unsigned &phase) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(phase) : "memory");
    phase ^= 1u;
}
template <class C>
PF_DEV void poly_load_tma(const Poly<C> *g, Poly<C> &A, unsigned long long *mb, unsigned &phase) {
    static_assert(sizeof(Poly<C>) % 16 == 0, "bulk copy size");
    const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
    pfw::sync();  // every lane is done with the previous cell's polytope
    if (pfw::lane() == 0) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&A);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a),
                     "r"((unsigned)sizeof(Poly<C>)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(g), "r"((unsigned)sizeof(Poly<C>)), "r"(a) : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(phase) : "memory");
    phase ^= 1u;
}
// bulk (TMA) store of a whole polytope record shared -> HBM (async; the
// shared buffer may be reused after poly_store_tma_wait)
template <class C>
PF_DEV void poly_store_tma(const Poly<C> &A, Poly<C> *g) {
    pfw::sync();
    if (pfw::lane() == 0) {
        const unsigned src = (unsigned)__cvta_generic_to_shared(&A);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(src),
                     "r"((unsigned)sizeof(Poly<C>)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
}
PF_DEV void poly_store_tma_wait() {
    if (pfw::lane() == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    pfw::sync();
}
#endif

template <class C>
PF_DEV void poly_load(const Poly<C> *g, Poly<C> &A) {
    const int L = pfw::lane();
    const int nv = g->nv, nf = g->nf, nl = g->nl;
#pragma unroll 1
    for (int v = L; v < nv; v += 32) { A.x[v] = g->x[v]; A.y[v] = g->y[v]; A.z[v] = g->z[v]; }
#pragma unroll 1
    for (int f = L; f < nf; f += 32) {
        A.nx[f] = g->nx[f]; A.ny[f] = g->ny[f]; A.nz[f] = g->nz[f]; A.d[f] = g->d[f]; A.tag[f] = g->tag[f];
    }
#pragma unroll 1
    for (int f = L; f <= nf; f += 32) A.lp[f] = g->lp[f];
#pragma unroll 1
    for (int k = L; k < nl; k += 32) A.lv[k] = g->lv[k];
    if (L == 0) { A.nv = nv; A.nf = nf; A.nl = nl; }
    pfw::sync();
}

// per-cell epilogue shared by the fused and the split kernels
template <class W>
PF_DEV void cell_finish(W *ws, const CellOut &out, int i, int r) {
    if (!(r & FLAG_RETRY) && pfw::lane() == 0) {
        if (W::CEN && out.census16)
#pragma unroll 1
            for (int k = 0; k < 16; k++) out.census16[(size_t)i * 16 + k] = k < CEN_N ? ws->cen[k] : 0;
        if (out.flags) out.flags[i] = r;
    }
    pfw::sync();
}

template <class W>
PF_DEV int run_cell(W *ws, const CellIn &in, const CellOut &out, int i) {
    int r = run_cell_impl(ws, in, out, i);
    cell_finish(ws, out, i, r);
    return r;
}

}  // namespace pf
