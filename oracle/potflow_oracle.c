/*
 * potflow_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's numba kernels
 * (/root/reference/pkg/src/potflow/_kernels.py) used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg.  Nothing in paper_2601_05765_b200/ links or loads this file.
 *
 * Floating-point contract: every expression keeps the reference's evaluation
 * order, the file is compiled with -ffp-contract=off (numba emits no FMA,
 * SURVEY.md §0.6) and transcendentals are glibc's atan2/sin/cos, exactly what
 * numba calls.  With that, this restatement is bit-identical to the numba
 * reference on every output (pinned by tests/test_oracle_golden.py against
 * fixtures produced by the reference itself, tests/golden/make_golden.py).
 *
 * Function-by-function correspondence (reference file:line):
 *   perp_basis          _kernels.py:59-80
 *   clip_into           _kernels.py:109-319
 *   piece_integrals     _kernels.py:331-390
 *   edge_other_facet    _kernels.py:397-408
 *   restrict_facet_seq  _kernels.py:411-675
 *   seq_integrals       _kernels.py:678-716
 *   interior_point      _kernels.py:723-816
 *   project_from        _kernels.py:819-835
 *   patch_area_seq      _kernels.py:838-1001
 *   evaluate_cell       _kernels.py:1008-1170
 *   bucket_of           _kernels.py:1177-1194
 *   build_cell          _kernels.py:1197-1355
 *   batch_evaluate      _kernels.py:1362-1478
 *   batch_build         _kernels.py:1481-1559
 *   knn                 _kernels.py:1562-1620
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

/* capacities, _kernels.py:24-27 */
#define MAX_V 512
#define MAX_F 160
#define MAX_L 2048
#define MAX_P 256

enum { CLIP_CUT = 0, CLIP_UNTOUCHED = 1, CLIP_EMPTY = 2, CLIP_OVERFLOW = 3, CLIP_DEGENERATE = 4 };
enum { RF_OUTSIDE = 0, RF_UNTOUCHED = 1, RF_FULLCIRCLE = 2, RF_GENPOLY = 3 };
enum { CELL_EMPTY = 0, CELL_FULLBALL = 1, CELL_CLIPPED = 2 };
enum { FLAG_OVERFLOW = 1, FLAG_DEGENERATE_INTERIOR = 2, FLAG_UNSTABLE_PROJECTION = 4 };

static const double PI = 3.141592653589793;
#define FOUR_PI (4.0 * PI)

/* packed cell (_kernels.py:10-18) */
typedef struct {
    double *v;   /* [MAX_V*3] */
    i64 *c;      /* [3] */
    double *pl;  /* [MAX_F*4] */
    i64 *tg;     /* [MAX_F] */
    i64 *lp;     /* [MAX_F+1] */
    i64 *lv;     /* [MAX_L] */
} PCell;

#define V(cell, i, k) ((cell).v[(i) * 3 + (k)])
#define PL(cell, f, k) ((cell).pl[(f) * 4 + (k)])

/* _kernels.py:59-80 */
static void perp_basis(double nx, double ny, double nz, double *e) {
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

/* _kernels.py:83-102 */
static void cell_copy(const double *vs, const i64 *cs, const double *ps, const i64 *ts,
                      const i64 *lps, const i64 *lvs, PCell d) {
    i64 nv = cs[0], nf = cs[1], nl = cs[2];
    memcpy(d.v, vs, sizeof(double) * 3 * nv);
    memcpy(d.pl, ps, sizeof(double) * 4 * nf);
    memcpy(d.tg, ts, sizeof(i64) * nf);
    memcpy(d.lp, lps, sizeof(i64) * (nf + 1));
    memcpy(d.lv, lvs, sizeof(i64) * nl);
    d.c[0] = nv; d.c[1] = nf; d.c[2] = nl;
}

/* per-thread scratch for clip_into */
typedef struct {
    double sd[MAX_V];
    i64 vmap[MAX_V];
    i64 cut_ea[MAX_V], cut_eb[MAX_V], cut_vi[MAX_V];
    unsigned char on_new[MAX_V];
    i64 tmp[MAX_L];
    double ang[MAX_V];
    i64 aidx[MAX_V];
    i64 ref[MAX_V];
} ClipScratch;

/* _kernels.py:109-319 */
static int clip_into(PCell A, PCell B, double nx, double ny, double nz, double dd,
                     i64 tag, double tol, ClipScratch *S) {
    i64 nv = A.c[0], nf = A.c[1];
    double *sd = S->sd;
    i64 n_out = 0, n_in = 0;
    for (i64 v = 0; v < nv; v++) {
        double s = nx * V(A, v, 0) + ny * V(A, v, 1) + nz * V(A, v, 2) - dd;
        sd[v] = s;
        if (s > tol) n_out++; else n_in++;
    }
    if (n_out == 0) return CLIP_UNTOUCHED;
    if (n_in == 0) return CLIP_EMPTY;

    i64 *vmap = S->vmap;
    i64 nvb = 0;
    for (i64 v = 0; v < nv; v++) {
        vmap[v] = -1;
        if (sd[v] <= tol) {
            if (nvb >= MAX_V) return CLIP_OVERFLOW;
            V(B, nvb, 0) = V(A, v, 0); V(B, nvb, 1) = V(A, v, 1); V(B, nvb, 2) = V(A, v, 2);
            vmap[v] = nvb;
            nvb++;
        }
    }
    i64 n_cut = 0;
    memset(S->on_new, 0, MAX_V);
    unsigned char *on_new = S->on_new;
    i64 *tmp = S->tmp;
    i64 nfb = 0, nlb = 0;
    B.lp[0] = 0;
    for (i64 f = 0; f < nf; f++) {
        i64 start = A.lp[f];
        i64 m = A.lp[f + 1] - start;
        i64 k = 0;
        for (i64 e = 0; e < m; e++) {
            i64 a = A.lv[start + e];
            i64 b = A.lv[start + (e + 1) % m];
            double sa = sd[a], sb = sd[b];
            int ina = sa <= tol, inb = sb <= tol;
            int cross = 0;
            if (ina) {
                tmp[k++] = vmap[a];
                if (sa >= -tol) on_new[vmap[a]] = 1;
                if ((!inb) && sa < -tol) cross = 1;
            } else {
                if (inb && sb < -tol) cross = 1;
            }
            if (cross) {
                i64 idx = -1;
                i64 lo = a < b ? a : b;
                i64 hi = a < b ? b : a;
                for (i64 q = 0; q < n_cut; q++) {
                    if (S->cut_ea[q] == lo && S->cut_eb[q] == hi) { idx = S->cut_vi[q]; break; }
                }
                if (idx < 0) {
                    if (nvb >= MAX_V || n_cut >= MAX_V) return CLIP_OVERFLOW;
                    double t = sa / (sa - sb);
                    V(B, nvb, 0) = V(A, a, 0) + t * (V(A, b, 0) - V(A, a, 0));
                    V(B, nvb, 1) = V(A, a, 1) + t * (V(A, b, 1) - V(A, a, 1));
                    V(B, nvb, 2) = V(A, a, 2) + t * (V(A, b, 2) - V(A, a, 2));
                    idx = nvb;
                    S->cut_ea[n_cut] = lo; S->cut_eb[n_cut] = hi; S->cut_vi[n_cut] = idx;
                    n_cut++;
                    nvb++;
                }
                tmp[k++] = idx;
                on_new[idx] = 1;
            }
        }
        if (k >= 3) {
            if (nfb >= MAX_F || nlb + k > MAX_L) return CLIP_OVERFLOW;
            for (int q = 0; q < 4; q++) PL(B, nfb, q) = PL(A, f, q);
            B.tg[nfb] = A.tg[f];
            for (i64 q = 0; q < k; q++) B.lv[nlb + q] = tmp[q];
            nlb += k;
            nfb++;
            B.lp[nfb] = nlb;
        }
    }
    /* new facet */
    i64 ncp = 0;
    double ccx = 0.0, ccy = 0.0, ccz = 0.0;
    for (i64 v = 0; v < nvb; v++) {
        if (on_new[v] == 1) {
            ncp++;
            ccx += V(B, v, 0); ccy += V(B, v, 1); ccz += V(B, v, 2);
        }
    }
    if (ncp < 3) return CLIP_DEGENERATE;
    ccx /= (double)ncp; ccy /= (double)ncp; ccz /= (double)ncp;
    double e[6];
    perp_basis(nx, ny, nz, e);
    double *ang = S->ang;
    i64 *aidx = S->aidx;
    i64 q = 0;
    for (i64 v = 0; v < nvb; v++) {
        if (on_new[v] == 1) {
            double rx = V(B, v, 0) - ccx, ry = V(B, v, 1) - ccy, rz = V(B, v, 2) - ccz;
            ang[q] = atan2(rx * e[3] + ry * e[4] + rz * e[5], rx * e[0] + ry * e[1] + rz * e[2]);
            aidx[q] = v;
            q++;
        }
    }
    for (i64 i = 1; i < ncp; i++) {
        double av = ang[i];
        i64 iv = aidx[i];
        i64 j = i - 1;
        while (j >= 0 && (ang[j] > av || (ang[j] == av && aidx[j] > iv))) {
            ang[j + 1] = ang[j]; aidx[j + 1] = aidx[j]; j--;
        }
        ang[j + 1] = av; aidx[j + 1] = iv;
    }
    if (nfb >= MAX_F || nlb + ncp > MAX_L) return CLIP_OVERFLOW;
    PL(B, nfb, 0) = nx; PL(B, nfb, 1) = ny; PL(B, nfb, 2) = nz; PL(B, nfb, 3) = dd;
    B.tg[nfb] = tag;
    for (i64 i = 0; i < ncp; i++) B.lv[nlb + i] = aidx[i];
    nlb += ncp;
    nfb++;
    B.lp[nfb] = nlb;

    /* drop unreferenced vertices */
    i64 *ref = S->ref;
    for (i64 v = 0; v < nvb; v++) ref[v] = -1;
    i64 nv2 = 0;
    for (i64 k2 = 0; k2 < nlb; k2++) {
        i64 v = B.lv[k2];
        if (ref[v] < 0) ref[v] = 0;
    }
    for (i64 v = 0; v < nvb; v++) {
        if (ref[v] == 0) { ref[v] = nv2; nv2++; }
    }
    if (nv2 != nvb) {
        for (i64 v = 0; v < nvb; v++) {
            if (ref[v] >= 0 && ref[v] != v) {
                V(B, ref[v], 0) = V(B, v, 0); V(B, ref[v], 1) = V(B, v, 1); V(B, ref[v], 2) = V(B, v, 2);
            }
        }
        for (i64 k2 = 0; k2 < nlb; k2++) B.lv[k2] = ref[B.lv[k2]];
    }
    B.c[0] = nv2; B.c[1] = nfb; B.c[2] = nlb;
    return CLIP_CUT;
}

/* piece rows: [kind, x0, y0, x1, y1, cx, cy, r, a0, a1]; _kernels.py:331-390 */
static void piece_integrals(const double *pieces, i64 npc, double *out) {
    double A = 0.0, Mx = 0.0, My = 0.0, Ip = 0.0;
    for (i64 i = 0; i < npc; i++) {
        const double *p = pieces + 10 * i;
        int kind = (int)p[0];
        if (kind == 0) {
            double x0 = p[1], y0 = p[2], x1 = p[3], y1 = p[4];
            double cr = x0 * y1 - x1 * y0;
            A += 0.5 * cr;
            double dx = x1 - x0, dy = y1 - y0;
            Mx += dy * (x0 * x0 + x0 * x1 + x1 * x1) / 6.0;
            My += -dx * (y0 * y0 + y0 * y1 + y1 * y1) / 6.0;
            double sx3 = x0 * x0 * x0 + x0 * x0 * x1 + x0 * x1 * x1 + x1 * x1 * x1;
            double sy3 = y0 * y0 * y0 + y0 * y0 * y1 + y0 * y1 * y1 + y1 * y1 * y1;
            Ip += (dy * sx3 - dx * sy3) / 12.0;
        } else {
            double cx = p[5], cy = p[6], r = p[7], a0, a1;
            if (kind == 2) { a0 = 0.0; a1 = 2.0 * PI; }
            else { a0 = p[8]; a1 = p[9]; }
            double dth = a1 - a0;
            double s0 = sin(a0), s1 = sin(a1), c0 = cos(a0), c1 = cos(a1);
            double s20 = sin(2.0 * a0), s21 = sin(2.0 * a1);
            double s40 = sin(4.0 * a0), s41 = sin(4.0 * a1);
            double ic = s1 - s0;
            double isn = c0 - c1;
            double ic2 = 0.5 * dth + 0.25 * (s21 - s20);
            double is2 = 0.5 * dth - 0.25 * (s21 - s20);
            double ic3 = (s1 - s1 * s1 * s1 / 3.0) - (s0 - s0 * s0 * s0 / 3.0);
            double is3 = (-c1 + c1 * c1 * c1 / 3.0) - (-c0 + c0 * c0 * c0 / 3.0);
            double ic4 = 0.375 * dth + 0.25 * (s21 - s20) + (s41 - s40) / 32.0;
            double is4 = 0.375 * dth - 0.25 * (s21 - s20) + (s41 - s40) / 32.0;
            A += 0.5 * (r * r * dth + cx * r * ic + cy * r * isn);
            Mx += 0.5 * r * (cx * cx * ic + 2.0 * cx * r * ic2 + r * r * ic3);
            My += 0.5 * r * (cy * cy * isn + 2.0 * cy * r * is2 + r * r * is3);
            Ip += (r / 3.0) * (cx * cx * cx * ic + 3.0 * cx * cx * r * ic2
                               + 3.0 * cx * r * r * ic3 + r * r * r * ic4
                               + cy * cy * cy * isn + 3.0 * cy * cy * r * is2
                               + 3.0 * cy * r * r * is3 + r * r * r * is4);
        }
    }
    out[0] = A; out[1] = Mx; out[2] = My; out[3] = Ip;
}

/* _kernels.py:397-408 */
static i64 edge_other_facet(const i64 *lp, const i64 *lv, i64 nf, i64 f, i64 a, i64 b) {
    for (i64 g = 0; g < nf; g++) {
        if (g == f) continue;
        i64 s = lp[g], m = lp[g + 1] - s;
        for (i64 e = 0; e < m; e++)
            if (lv[s + e] == b && lv[s + (e + 1) % m] == a) return g;
    }
    return -1;
}

/* _kernels.py:411-675.  Returns kind (-1 on MAX_P overflow); writes npts, s, rc. */
static int restrict_facet_seq(PCell C, i64 f, double px, double py, double pz, double psi,
                              double tol, double *pts, unsigned char *on_sph,
                              unsigned char *conn, i64 *npts_out, double *s_out, double *rc_out) {
    i64 nf = C.c[1];
    double nx = PL(C, f, 0), ny = PL(C, f, 1), nz = PL(C, f, 2), dd = PL(C, f, 3);
    double s = dd - (nx * px + ny * py + nz * pz);
    double rc2 = psi - s * s;
    double R = sqrt(psi);
    *s_out = s; *npts_out = 0; *rc_out = 0.0;
    if (rc2 <= tol * (2.0 * R + tol)) return RF_OUTSIDE;
    double rc = sqrt(rc2);
    *rc_out = rc;
    double qx = px + s * nx, qy = py + s * ny, qz = pz + s * nz;
    i64 start = C.lp[f];
    i64 m = C.lp[f + 1] - start;
    double ball_tol = tol * (2.0 * R + tol);
    unsigned char inside[MAX_L];
    i64 n_in = 0;
    for (i64 e = 0; e < m; e++) {
        i64 v = C.lv[start + e];
        double wx = V(C, v, 0) - px, wy = V(C, v, 1) - py, wz = V(C, v, 2) - pz;
        double q = wx * wx + wy * wy + wz * wz - psi;
        if (q <= ball_tol) { inside[e] = 1; n_in++; } else inside[e] = 0;
    }
    if (n_in == m) {
        for (i64 e = 0; e < m; e++) {
            i64 v = C.lv[start + e];
            pts[3 * e] = V(C, v, 0); pts[3 * e + 1] = V(C, v, 1); pts[3 * e + 2] = V(C, v, 2);
            on_sph[e] = 0; conn[e] = 0;
        }
        *npts_out = m;
        return RF_UNTOUCHED;
    }
    i64 npts = 0;
    int first_entry = 0;
    int cur_inside = inside[0] == 1;
    for (i64 e = 0; e < m; e++) {
        i64 a = C.lv[start + e];
        i64 bb = C.lv[start + (e + 1) % m];
        int ina = inside[e] == 1;
        int inb = inside[(e + 1) % m] == 1;
        if (ina) {
            if (npts >= MAX_P) return -1;
            pts[3 * npts] = V(C, a, 0); pts[3 * npts + 1] = V(C, a, 1); pts[3 * npts + 2] = V(C, a, 2);
            on_sph[npts] = 0; conn[npts] = 0;
            npts++;
            cur_inside = 1;
        }
        if (ina && inb) continue;
        i64 g = edge_other_facet(C.lp, C.lv, nf, f, a, bb);
        double gx, gy, gz, gd, c12, det, ux, uy, uz;
        if (g >= 0) {
            gx = PL(C, g, 0); gy = PL(C, g, 1); gz = PL(C, g, 2); gd = PL(C, g, 3);
            c12 = nx * gx + ny * gy + nz * gz;
            det = 1.0 - c12 * c12;
            ux = ny * gz - nz * gy;
            uy = nz * gx - nx * gz;
            uz = nx * gy - ny * gx;
        } else {
            ux = V(C, bb, 0) - V(C, a, 0);
            uy = V(C, bb, 1) - V(C, a, 1);
            uz = V(C, bb, 2) - V(C, a, 2);
            det = 1.0; c12 = 0.0; gd = 0.0; gx = 0.0; gy = 0.0; gz = 0.0;
        }
        double un = sqrt(ux * ux + uy * uy + uz * uz);
        if (un < 1e-300 || det <= 1e-300) { cur_inside = inb; continue; }
        ux /= un; uy /= un; uz /= un;
        if (ux < 0.0 || (ux == 0.0 && (uy < 0.0 || (uy == 0.0 && uz < 0.0)))) {
            ux = -ux; uy = -uy; uz = -uz;
        }
        double x0x, x0y, x0z;
        if (g >= 0) {
            double r1 = dd - (nx * px + ny * py + nz * pz);
            double r2 = gd - (gx * px + gy * py + gz * pz);
            double al = (r1 - c12 * r2) / det;
            double be = (r2 - c12 * r1) / det;
            x0x = px + al * nx + be * gx;
            x0y = py + al * ny + be * gy;
            x0z = pz + al * nz + be * gz;
        } else {
            x0x = V(C, a, 0); x0y = V(C, a, 1); x0z = V(C, a, 2);
        }
        double w0x = x0x - px, w0y = x0y - py, w0z = x0z - pz;
        double bh = ux * w0x + uy * w0y + uz * w0z;
        double cc = w0x * w0x + w0y * w0y + w0z * w0z - psi;
        double disc = bh * bh - cc;
        if (disc <= tol * tol) { cur_inside = inb; continue; }
        double sq = sqrt(disc);
        double t1 = -bh - sq, t2 = -bh + sq;
        double ta = ux * (V(C, a, 0) - x0x) + uy * (V(C, a, 1) - x0y) + uz * (V(C, a, 2) - x0z);
        double tb = ux * (V(C, bb, 0) - x0x) + uy * (V(C, bb, 1) - x0y) + uz * (V(C, bb, 2) - x0z);
        double tlo = ta < tb ? ta : tb;
        double thi = ta < tb ? tb : ta;
        for (int which = 0; which < 2; which++) {
            double t;
            if (ta <= tb) t = which == 0 ? t1 : t2;
            else t = which == 0 ? t2 : t1;
            if (t <= tlo + tol || t >= thi - tol) continue;
            if (npts >= MAX_P) return -1;
            double cxx = x0x + t * ux, cxy = x0y + t * uy, cxz = x0z + t * uz;
            if (cur_inside) {
                pts[3 * npts] = cxx; pts[3 * npts + 1] = cxy; pts[3 * npts + 2] = cxz;
                on_sph[npts] = 1; conn[npts] = 1;
                npts++;
                cur_inside = 0;
            } else {
                if (npts > 0) conn[npts - 1] = 1;
                else first_entry = 1;
                pts[3 * npts] = cxx; pts[3 * npts + 1] = cxy; pts[3 * npts + 2] = cxz;
                on_sph[npts] = 1; conn[npts] = 0;
                npts++;
                cur_inside = 1;
            }
        }
        cur_inside = inb;
    }
    if (npts == 0) {
        double e[6];
        perp_basis(nx, ny, nz, e);
        int cin = 1;
        for (i64 ee = 0; ee < m; ee++) {
            i64 a = C.lv[start + ee];
            i64 bb = C.lv[start + (ee + 1) % m];
            double p0u = (V(C, a, 0) - qx) * e[0] + (V(C, a, 1) - qy) * e[1] + (V(C, a, 2) - qz) * e[2];
            double p0v = (V(C, a, 0) - qx) * e[3] + (V(C, a, 1) - qy) * e[4] + (V(C, a, 2) - qz) * e[5];
            double p1u = (V(C, bb, 0) - qx) * e[0] + (V(C, bb, 1) - qy) * e[1] + (V(C, bb, 2) - qz) * e[2];
            double p1v = (V(C, bb, 0) - qx) * e[3] + (V(C, bb, 1) - qy) * e[4] + (V(C, bb, 2) - qz) * e[5];
            if ((p1u - p0u) * (-p0v) - (p1v - p0v) * (-p0u) < 0.0) { cin = 0; break; }
        }
        if (cin) return RF_FULLCIRCLE;
        return RF_OUTSIDE;
    }
    if (first_entry) conn[npts - 1] = 1;
    /* drop zero-length connectors */
    i64 k = 0;
    for (i64 i = 0; i < npts; i++) {
        i64 j = (i + 1) % npts;
        double dxp = pts[3 * i] - pts[3 * j];
        double dyp = pts[3 * i + 1] - pts[3 * j + 1];
        double dzp = pts[3 * i + 2] - pts[3 * j + 2];
        if (conn[i] == 0 && dxp * dxp + dyp * dyp + dzp * dzp <= tol * tol) {
            if (on_sph[i] == 1) on_sph[j] = 1;
            pts[3 * i] = NAN;
        } else {
            k++;
        }
    }
    if (k < npts) {
        i64 w = 0;
        for (i64 i = 0; i < npts; i++) {
            if (!isnan(pts[3 * i])) {
                pts[3 * w] = pts[3 * i]; pts[3 * w + 1] = pts[3 * i + 1]; pts[3 * w + 2] = pts[3 * i + 2];
                on_sph[w] = on_sph[i]; conn[w] = conn[i];
                w++;
            }
        }
        npts = w;
    }
    if (npts < 2) { *npts_out = 0; return RF_OUTSIDE; }
    int has_arc = 0;
    double e[6];
    perp_basis(nx, ny, nz, e);
    double best = 1e300;
    i64 bi = 0;
    for (i64 i = 0; i < npts; i++) {
        if (conn[i] == 1) {
            has_arc = 1;
            double rx = pts[3 * i] - qx, ry = pts[3 * i + 1] - qy, rz = pts[3 * i + 2] - qz;
            double aang = atan2(rx * e[3] + ry * e[4] + rz * e[5], rx * e[0] + ry * e[1] + rz * e[2]);
            if (aang < best) { best = aang; bi = i; }
        }
    }
    if (has_arc && bi != 0) {
        double tmp[3 * MAX_P];
        unsigned char tos[MAX_P], tco[MAX_P];
        for (i64 i = 0; i < npts; i++) {
            i64 j = (bi + i) % npts;
            tmp[3 * i] = pts[3 * j]; tmp[3 * i + 1] = pts[3 * j + 1]; tmp[3 * i + 2] = pts[3 * j + 2];
            tos[i] = on_sph[j]; tco[i] = conn[j];
        }
        for (i64 i = 0; i < npts; i++) {
            pts[3 * i] = tmp[3 * i]; pts[3 * i + 1] = tmp[3 * i + 1]; pts[3 * i + 2] = tmp[3 * i + 2];
            on_sph[i] = tos[i]; conn[i] = tco[i];
        }
    }
    *npts_out = npts;
    return RF_GENPOLY;
}

/* _kernels.py:678-716; out = A, cx, cy, cz, Ip */
static void seq_integrals(const double *pts, const unsigned char *conn, i64 npts,
                          double nx, double ny, double nz, double qx, double qy, double qz,
                          double rc, double *out) {
    double e[6];
    perp_basis(nx, ny, nz, e);
    double pieces[10 * MAX_P];
    for (i64 i = 0; i < npts; i++) {
        i64 j = (i + 1) % npts;
        double *p = pieces + 10 * i;
        double x0 = (pts[3 * i] - qx) * e[0] + (pts[3 * i + 1] - qy) * e[1] + (pts[3 * i + 2] - qz) * e[2];
        double y0 = (pts[3 * i] - qx) * e[3] + (pts[3 * i + 1] - qy) * e[4] + (pts[3 * i + 2] - qz) * e[5];
        double x1 = (pts[3 * j] - qx) * e[0] + (pts[3 * j + 1] - qy) * e[1] + (pts[3 * j + 2] - qz) * e[2];
        double y1 = (pts[3 * j] - qx) * e[3] + (pts[3 * j + 1] - qy) * e[4] + (pts[3 * j + 2] - qz) * e[5];
        if (conn[i] == 0) {
            p[0] = 0.0; p[1] = x0; p[2] = y0; p[3] = x1; p[4] = y1;
        } else {
            double a0 = atan2(y0, x0);
            double a1 = atan2(y1, x1);
            double sweep = a1 - a0;
            if (sweep <= 0.0) sweep += 2.0 * PI;
            p[0] = 1.0; p[5] = 0.0; p[6] = 0.0; p[7] = rc; p[8] = a0; p[9] = a0 + sweep;
        }
    }
    double r[4];
    piece_integrals(pieces, npts, r);
    double A = r[0], Mx = r[1], My = r[2], Ip = r[3];
    double cx, cy, cz;
    if (A > 0.0) {
        cx = qx + (Mx / A) * e[0] + (My / A) * e[3];
        cy = qy + (Mx / A) * e[1] + (My / A) * e[4];
        cz = qz + (Mx / A) * e[2] + (My / A) * e[5];
    } else {
        cx = qx; cy = qy; cz = qz;
    }
    out[0] = A; out[1] = cx; out[2] = cy; out[3] = cz; out[4] = Ip;
}

static inline double sq(double x) { return x * x; }

/* _kernels.py:723-816; out = cx, cy, cz, bx, by, bz; returns ok */
static int interior_point(PCell C, i64 nf, const i64 *fkind, const double *farea,
                          const double *fcx, const double *fcy, const double *fcz,
                          double px, double py, double pz, double psi, double tol, double *out) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    i64 nseg = 0;
    double best_margin = -1.0;
    double bx = px, by = py, bz = pz;
    for (i64 f = 0; f < nf; f++) {
        if (fkind[f] == RF_OUTSIDE || farea[f] <= 0.0) continue;
        double ox = fcx[f], oy = fcy[f], oz = fcz[f];
        double dx = -PL(C, f, 0), dy = -PL(C, f, 1), dz = -PL(C, f, 2);
        double wx = ox - px, wy = oy - py, wz = oz - pz;
        double bh = dx * wx + dy * wy + dz * wz;
        double cc = wx * wx + wy * wy + wz * wz - psi;
        double disc = bh * bh - cc;
        if (disc <= 0.0) continue;
        double t_hi = -bh + sqrt(disc);
        double t_lo = 0.0;
        int ok = 1;
        for (i64 g = 0; g < nf; g++) {
            if (g == f) continue;
            double den = PL(C, g, 0) * dx + PL(C, g, 1) * dy + PL(C, g, 2) * dz;
            double num = PL(C, g, 3) - (PL(C, g, 0) * ox + PL(C, g, 1) * oy + PL(C, g, 2) * oz);
            if (den > tol) {
                double tc = num / den;
                if (tc < t_hi) t_hi = tc;
            } else if (den < -tol) {
                double tc = num / den;
                if (tc > t_lo) t_lo = tc;
            } else {
                if (num < -tol) { ok = 0; break; }
            }
        }
        if (!ok || t_hi - t_lo <= tol) continue;
        double tm = 0.5 * (t_lo + t_hi);
        double mx = ox + tm * dx, my = oy + tm * dy, mz = oz + tm * dz;
        sx += mx; sy += my; sz += mz;
        nseg++;
        double mg = sqrt(psi) - sqrt(sq(mx - px) + sq(my - py) + sq(mz - pz));
        for (i64 g = 0; g < nf; g++) {
            double d2 = PL(C, g, 3) - (PL(C, g, 0) * mx + PL(C, g, 1) * my + PL(C, g, 2) * mz);
            if (d2 < mg) mg = d2;
        }
        if (mg > best_margin) { best_margin = mg; bx = mx; by = my; bz = mz; }
    }
    out[3] = bx; out[4] = by; out[5] = bz;
    if (nseg == 0) { out[0] = px; out[1] = py; out[2] = pz; return 0; }
    double cx = sx / (double)nseg, cy = sy / (double)nseg, cz = sz / (double)nseg;
    double mg = sqrt(psi) - sqrt(sq(cx - px) + sq(cy - py) + sq(cz - pz));
    for (i64 g = 0; g < nf; g++) {
        double d2 = PL(C, g, 3) - (PL(C, g, 0) * cx + PL(C, g, 1) * cy + PL(C, g, 2) * cz);
        if (d2 < mg) mg = d2;
    }
    if (mg <= 0.0) {
        if (best_margin > 0.0) { out[0] = bx; out[1] = by; out[2] = bz; return 1; }
        out[0] = px; out[1] = py; out[2] = pz; return 0;
    }
    out[0] = cx; out[1] = cy; out[2] = cz;
    return 1;
}

/* _kernels.py:819-835 */
static void project_from(double cx, double cy, double cz, double yx, double yy, double yz,
                         double px, double py, double pz, double psi, double *o) {
    double dx = yx - cx, dy = yy - cy, dz = yz - cz;
    double a = dx * dx + dy * dy + dz * dz;
    double wx = cx - px, wy = cy - py, wz = cz - pz;
    double b = dx * wx + dy * wy + dz * wz;
    double c0 = wx * wx + wy * wy + wz * wz - psi;
    double disc = b * b - a * c0;
    if (disc < 0.0) disc = 0.0;
    double t = (-b + sqrt(disc)) / a;
    o[0] = cx + t * dx; o[1] = cy + t * dy; o[2] = cz + t * dz;
}

/* _kernels.py:838-1001 */
static double patch_area_seq(const double *pts, const unsigned char *on_sph,
                             const unsigned char *conn, i64 npts,
                             double nx, double ny, double nz, double s,
                             double px, double py, double pz, double psi,
                             double cx, double cy, double cz, double tol, int *unstable_out) {
    (void)tol;
    double R = sqrt(psi);
    double proj[3 * MAX_P], tin[3 * MAX_P], tout[3 * MAX_P];
    for (i64 i = 0; i < npts; i++) {
        if (on_sph[i] == 1) {
            proj[3 * i] = pts[3 * i]; proj[3 * i + 1] = pts[3 * i + 1]; proj[3 * i + 2] = pts[3 * i + 2];
        } else {
            project_from(cx, cy, cz, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], px, py, pz, psi, proj + 3 * i);
        }
    }
    /* tin/tout hold np.empty garbage in the reference when a connector is
     * skipped; those cells are always flagged unstable and re-run, so any
     * deterministic fill is equivalent. */
    for (i64 i = 0; i < 3 * npts; i++) { tin[i] = 0.0; tout[i] = 0.0; }
    double kg_sum = 0.0;
    int unstable = 0;
    for (i64 i = 0; i < npts; i++) {
        i64 j = (i + 1) % npts;
        double mx, my, mz, ee;
        if (conn[i] == 1) {
            mx = nx; my = ny; mz = nz; ee = s;
        } else {
            double ax = pts[3 * i] - cx, ay = pts[3 * i + 1] - cy, az = pts[3 * i + 2] - cz;
            double bx2 = pts[3 * j] - cx, by2 = pts[3 * j + 1] - cy, bz2 = pts[3 * j + 2] - cz;
            mx = ay * bz2 - az * by2;
            my = az * bx2 - ax * bz2;
            mz = ax * by2 - ay * bx2;
            double mn = sqrt(mx * mx + my * my + mz * mz);
            if (mn < 1e-300) { unstable = 1; continue; }
            mx /= mn; my /= mn; mz /= mn;
            ee = mx * (cx - px) + my * (cy - py) + mz * (cz - pz);
        }
        for (int attempt = 0; attempt < 2; attempt++) {
            double qx = px + ee * mx, qy = py + ee * my, qz = pz + ee * mz;
            double rr2 = psi - ee * ee;
            if (rr2 <= 0.0) { unstable = 1; break; }
            double u[6];
            perp_basis(mx, my, mz, u);
            double rpx = proj[3 * i] - qx, rpy = proj[3 * i + 1] - qy, rpz = proj[3 * i + 2] - qz;
            double phP = atan2(rpx * u[3] + rpy * u[4] + rpz * u[5], rpx * u[0] + rpy * u[1] + rpz * u[2]);
            double rqx = proj[3 * j] - qx, rqy = proj[3 * j + 1] - qy, rqz = proj[3 * j + 2] - qz;
            double phQ = atan2(rqx * u[3] + rqy * u[4] + rqz * u[5], rqx * u[0] + rqy * u[1] + rqz * u[2]);
            double dPQ = phQ - phP;
            if (dPQ < 0.0) dPQ += 2.0 * PI;
            double sweep;
            if (conn[i] == 1) {
                sweep = dPQ;
            } else {
                double mxp = 0.5 * (pts[3 * i] + pts[3 * j]);
                double myp = 0.5 * (pts[3 * i + 1] + pts[3 * j + 1]);
                double mzp = 0.5 * (pts[3 * i + 2] + pts[3 * j + 2]);
                double h[3];
                project_from(cx, cy, cz, mxp, myp, mzp, px, py, pz, psi, h);
                double rmx = h[0] - qx, rmy = h[1] - qy, rmz = h[2] - qz;
                double phM = atan2(rmx * u[3] + rmy * u[4] + rmz * u[5], rmx * u[0] + rmy * u[1] + rmz * u[2]);
                double dPM = phM - phP;
                if (dPM < 0.0) dPM += 2.0 * PI;
                if (dPM <= dPQ + 1e-12) {
                    sweep = dPQ;
                } else {
                    mx = -mx; my = -my; mz = -mz; ee = -ee;
                    continue;
                }
            }
            kg_sum += (ee / R) * sweep;
            double t0x = my * rpz - mz * rpy, t0y = mz * rpx - mx * rpz, t0z = mx * rpy - my * rpx;
            double tn = sqrt(t0x * t0x + t0y * t0y + t0z * t0z);
            if (tn > 0.0) { t0x /= tn; t0y /= tn; t0z /= tn; }
            tout[3 * i] = t0x; tout[3 * i + 1] = t0y; tout[3 * i + 2] = t0z;
            double t1x = my * rqz - mz * rqy, t1y = mz * rqx - mx * rqz, t1z = mx * rqy - my * rqx;
            tn = sqrt(t1x * t1x + t1y * t1y + t1z * t1z);
            if (tn > 0.0) { t1x /= tn; t1y /= tn; t1z /= tn; }
            tin[3 * j] = t1x; tin[3 * j + 1] = t1y; tin[3 * j + 2] = t1z;
            break;
        }
    }
    double th_sum = 0.0;
    for (i64 i = 0; i < npts; i++) {
        double ax = tin[3 * i], ay = tin[3 * i + 1], az = tin[3 * i + 2];
        double bx2 = tout[3 * i], by2 = tout[3 * i + 1], bz2 = tout[3 * i + 2];
        double nxv = (proj[3 * i] - px) / R, nyv = (proj[3 * i + 1] - py) / R, nzv = (proj[3 * i + 2] - pz) / R;
        double crx = ay * bz2 - az * by2, cry = az * bx2 - ax * bz2, crz = ax * by2 - ay * bx2;
        double sv = crx * nxv + cry * nyv + crz * nzv;
        double cv = ax * bx2 + ay * by2 + az * bz2;
        double th = atan2(sv, cv);
        if (fabs(th) > PI - 1e-7) unstable = 1;
        th_sum += th;
    }
    double area = psi * (2.0 * PI - kg_sum - th_sum);
    if (area < -1e-9 * FOUR_PI * psi || area > FOUR_PI * psi * (1.0 + 1e-9)) unstable = 1;
    if (area < 0.0) area = 0.0;
    if (area > FOUR_PI * psi) area = FOUR_PI * psi;
    *unstable_out = unstable;
    return area;
}

/* per-thread scratch for evaluate_cell */
typedef struct {
    i64 fkind[MAX_F], fnp[MAX_F];
    double farea[MAX_F], fh[MAX_F], fcx[MAX_F], fcy[MAX_F], fcz[MAX_F], fip[MAX_F], frc[MAX_F];
    double seq_pts[MAX_F][3 * MAX_P];
    unsigned char seq_os[MAX_F][MAX_P], seq_cn[MAX_F][MAX_P];
} EvalScratch;

/* _kernels.py:1008-1170.  r = status, vol, K, cx, cy, cz, ix, iy, iz, m2 ; returns flags */
static i64 evaluate_cell(PCell C, double px, double py, double pz, double psi, double tol,
                         int want_m2, EvalScratch *E, double *r) {
    i64 nf = C.c[1];
    i64 flags = 0;
#define RET_EMPTY() do { r[0] = CELL_EMPTY; r[1] = 0.0; r[2] = 0.0; r[3] = px; r[4] = py; r[5] = pz; \
        r[6] = px; r[7] = py; r[8] = pz; r[9] = 0.0; return flags; } while (0)
    if (psi <= 0.0) RET_EMPTY();
    double R = sqrt(psi);
    int any_present = 0;
    for (i64 f = 0; f < nf; f++) {
        i64 npts; double s, rc;
        int kind = restrict_facet_seq(C, f, px, py, pz, psi, tol, E->seq_pts[f], E->seq_os[f],
                                      E->seq_cn[f], &npts, &s, &rc);
        if (kind < 0) { flags |= FLAG_OVERFLOW; RET_EMPTY(); }
        E->fkind[f] = kind; E->fh[f] = s; E->frc[f] = rc; E->fnp[f] = npts;
        if (kind == RF_OUTSIDE) {
            E->farea[f] = 0.0; E->fcx[f] = px; E->fcy[f] = py; E->fcz[f] = pz; E->fip[f] = 0.0;
            continue;
        }
        any_present = 1;
        double qx = px + s * PL(C, f, 0), qy = py + s * PL(C, f, 1), qz = pz + s * PL(C, f, 2);
        if (kind == RF_FULLCIRCLE) {
            E->farea[f] = PI * rc * rc;
            E->fcx[f] = qx; E->fcy[f] = qy; E->fcz[f] = qz;
            double rc2 = rc * rc;
            E->fip[f] = 0.5 * PI * (rc2 * rc2);
        } else {
            double o[5];
            seq_integrals(E->seq_pts[f], E->seq_cn[f], npts, PL(C, f, 0), PL(C, f, 1), PL(C, f, 2),
                          qx, qy, qz, rc, o);
            if (o[0] <= 0.0) {
                E->fkind[f] = RF_OUTSIDE;
                E->farea[f] = 0.0; E->fcx[f] = px; E->fcy[f] = py; E->fcz[f] = pz; E->fip[f] = 0.0;
                continue;
            }
            E->farea[f] = o[0]; E->fcx[f] = o[1]; E->fcy[f] = o[2]; E->fcz[f] = o[3]; E->fip[f] = o[4];
        }
    }
    int any_area = 0;
    for (i64 f = 0; f < nf; f++)
        if (E->fkind[f] != RF_OUTSIDE && E->farea[f] > 0.0) { any_area = 1; break; }
    if (!any_present || !any_area) {
        int inside = 1;
        for (i64 f = 0; f < nf; f++)
            if (E->fh[f] < -tol) { inside = 0; break; }
        if ((inside && nf > 0) || nf == 0) {
            r[0] = CELL_FULLBALL; r[1] = FOUR_PI / 3.0 * psi * R; r[2] = FOUR_PI * psi;
            r[3] = px; r[4] = py; r[5] = pz; r[6] = px; r[7] = py; r[8] = pz;
            r[9] = want_m2 ? FOUR_PI * psi * R * R * R / 5.0 : 0.0;
            return flags;
        }
        RET_EMPTY();
    }
    double ip[6];
    int ok = interior_point(C, nf, E->fkind, E->farea, E->fcx, E->fcy, E->fcz, px, py, pz, psi, tol, ip);
    if (!ok) { flags |= FLAG_DEGENERATE_INTERIOR; RET_EMPTY(); }
    double ix = ip[0], iy = ip[1], iz = ip[2], bx = ip[3], by = ip[4], bz = ip[5];
    double kbar = 0.0;
    for (int attempt = 0; attempt < 4; attempt++) {
        kbar = 0.0;
        int bad = 0;
        for (i64 f = 0; f < nf; f++) {
            if (E->fkind[f] == RF_OUTSIDE || E->farea[f] <= 0.0) continue;
            if (E->fkind[f] == RF_FULLCIRCLE) { kbar += 2.0 * PI * R * (R - E->fh[f]); continue; }
            int uns;
            double a = patch_area_seq(E->seq_pts[f], E->seq_os[f], E->seq_cn[f], E->fnp[f],
                                      PL(C, f, 0), PL(C, f, 1), PL(C, f, 2), E->fh[f],
                                      px, py, pz, psi, ix, iy, iz, tol, &uns);
            if (uns) { bad = 1; break; }
            kbar += a;
        }
        if (!bad) break;
        if (attempt == 3) { flags |= FLAG_UNSTABLE_PROJECTION; break; }
        double w = 0.35 * (double)(attempt + 1);
        ix = ix + w * (bx - ix);
        iy = iy + w * (by - iy);
        iz = iz + w * (bz - iz);
    }
    double K = FOUR_PI * psi - kbar;
    if (K < 0.0) K = 0.0;
    if (K > FOUR_PI * psi) K = FOUR_PI * psi;
    double vol = R * K / 3.0;
    double mx = 0.0, my = 0.0, mz = 0.0, nsx = 0.0, nsy = 0.0, nsz = 0.0;
    double m2 = want_m2 ? R * R * R * K / 5.0 : 0.0;
    for (i64 f = 0; f < nf; f++) {
        if (E->fkind[f] == RF_OUTSIDE || E->farea[f] <= 0.0) continue;
        double pv = E->fh[f] * E->farea[f] / 3.0;
        vol += pv;
        mx += pv * 0.75 * (E->fcx[f] - px);
        my += pv * 0.75 * (E->fcy[f] - py);
        mz += pv * 0.75 * (E->fcz[f] - pz);
        nsx += PL(C, f, 0) * E->farea[f];
        nsy += PL(C, f, 1) * E->farea[f];
        nsz += PL(C, f, 2) * E->farea[f];
        if (want_m2) m2 += (E->fh[f] / 5.0) * (E->fip[f] + E->fh[f] * E->fh[f] * E->farea[f]);
    }
    mx += 0.25 * psi * (-nsx);
    my += 0.25 * psi * (-nsy);
    mz += 0.25 * psi * (-nsz);
    double ccx, ccy, ccz;
    if (vol > 0.0) { ccx = px + mx / vol; ccy = py + my / vol; ccz = pz + mz / vol; }
    else { vol = 0.0; ccx = px; ccy = py; ccz = pz; }
    r[0] = CELL_CLIPPED; r[1] = vol; r[2] = K; r[3] = ccx; r[4] = ccy; r[5] = ccz;
    r[6] = ix; r[7] = iy; r[8] = iz; r[9] = m2;
    return flags;
#undef RET_EMPTY
}

typedef struct {
    const i64 *start, *sites;
    double lox, loy, loz, ihx, ihy, ihz;
    i64 gnx, gny, gnz;
    double h_min;
} Grid;

/* _kernels.py:1177-1194 */
static void bucket_of(const Grid *G, double x, double y, double z, i64 *b) {
    i64 ix = (i64)((x - G->lox) * G->ihx);
    i64 iy = (i64)((y - G->loy) * G->ihy);
    i64 iz = (i64)((z - G->loz) * G->ihz);
    if (ix < 0) ix = 0;
    if (iy < 0) iy = 0;
    if (iz < 0) iz = 0;
    if (ix >= G->gnx) ix = G->gnx - 1;
    if (iy >= G->gny) iy = G->gny - 1;
    if (iz >= G->gnz) iz = G->gnz - 1;
    b[0] = ix; b[1] = iy; b[2] = iz;
}

typedef struct {
    double dom_v[MAX_V * 3];
    i64 dom_c[3];
    double dom_p[MAX_F * 4];
    i64 dom_t[MAX_F], dom_lp[MAX_F + 1], dom_lv[MAX_L];
} Domain;

typedef struct {
    double vA[MAX_V * 3], vB[MAX_V * 3];
    i64 cA[3], cB[3];
    double pA[MAX_F * 4], pB[MAX_F * 4];
    i64 tA[MAX_F], tB[MAX_F], lpA[MAX_F + 1], lpB[MAX_F + 1], lvA[MAX_L], lvB[MAX_L];
    ClipScratch clip;
    EvalScratch ev;
    double *cand_d2;
    i64 *cand_j;
    i64 n_clips;  /* census: processed candidates */
} CellWork;

static PCell cw_A(CellWork *w) { PCell c = {w->vA, w->cA, w->pA, w->tA, w->lpA, w->lvA}; return c; }
static PCell cw_B(CellWork *w) { PCell c = {w->vB, w->cB, w->pB, w->tB, w->lpB, w->lvB}; return c; }

/* _kernels.py:1197-1355 ; returns status (0 ok / 1 empty / 3 overflow), *which */
static int build_cell(i64 i, i64 n, const double *pts, const double *psi, double dpsi_max,
                      int ball_aware, const Domain *D, const Grid *G, double tol,
                      CellWork *w, int *which_out) {
    double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
    double psii = psi[i];
    PCell A = cw_A(w), B = cw_B(w);
    cell_copy(D->dom_v, D->dom_c, D->dom_p, D->dom_t, D->dom_lp, D->dom_lv, A);
    int which = 0;
    double *cand_d2 = w->cand_d2;
    i64 *cand_j = w->cand_j;
    i64 ncand = 0, ptr = 0;
    i64 bb[3];
    bucket_of(G, px, py, pz, bb);
    i64 ring = 0;
    double covered = 0.0;
    int rings_done = 0;
    double rfar = 0.0;
    w->n_clips = 0;
    for (i64 v = 0; v < A.c[0]; v++) {
        double d2 = sq(V(A, v, 0) - px) + sq(V(A, v, 1) - py) + sq(V(A, v, 2) - pz);
        if (d2 > rfar) rfar = d2;
    }
    rfar = sqrt(rfar);
    double sq_ball = (ball_aware && psii > 0.0) ? sqrt(psii) : -1.0;
    double sq_psi_slack = sqrt((psii > 0.0 ? psii : 0.0) + dpsi_max);
    (void)n;
    for (;;) {
        double stop_r = rfar + sqrt(rfar * rfar + dpsi_max);
        if (ball_aware) {
            if (psii <= 0.0) break;
            double br = sq_ball + sq_psi_slack;
            if (br < stop_r) stop_r = br;
        }
        for (;;) {
            int need_more = 0;
            if (!rings_done)
                if (ptr >= ncand || cand_d2[ptr] > covered * covered) need_more = 1;
            if (!need_more) break;
            int added = 0, any_cell = 0;
            for (i64 dx = -ring; dx <= ring; dx++) {
                i64 ix = bb[0] + dx;
                if (ix < 0 || ix >= G->gnx) continue;
                for (i64 dy = -ring; dy <= ring; dy++) {
                    i64 iy = bb[1] + dy;
                    if (iy < 0 || iy >= G->gny) continue;
                    for (i64 dz = -ring; dz <= ring; dz++) {
                        i64 adx = dx < 0 ? -dx : dx, ady = dy < 0 ? -dy : dy, adz = dz < 0 ? -dz : dz;
                        i64 mxa = adx > ady ? adx : ady;
                        if (adz > mxa) mxa = adz;
                        if (mxa != ring) continue;
                        i64 iz = bb[2] + dz;
                        if (iz < 0 || iz >= G->gnz) continue;
                        any_cell = 1;
                        i64 lin = (ix * G->gny + iy) * G->gnz + iz;
                        for (i64 q = G->start[lin]; q < G->start[lin + 1]; q++) {
                            i64 j = G->sites[q];
                            if (j == i) continue;
                            double d2 = sq(pts[3 * j] - px) + sq(pts[3 * j + 1] - py) + sq(pts[3 * j + 2] - pz);
                            cand_d2[ncand] = d2;
                            cand_j[ncand] = j;
                            ncand++;
                            added = 1;
                        }
                    }
                }
            }
            covered = (double)ring * G->h_min;
            ring++;
            if (ring > G->gnx + G->gny + G->gnz && !any_cell) { rings_done = 1; covered = 1e300; }
            if (added) {
                for (i64 a = ptr + 1; a < ncand; a++) {
                    double dv2 = cand_d2[a];
                    i64 jv = cand_j[a];
                    i64 b = a - 1;
                    while (b >= ptr && (cand_d2[b] > dv2 || (cand_d2[b] == dv2 && cand_j[b] > jv))) {
                        cand_d2[b + 1] = cand_d2[b]; cand_j[b + 1] = cand_j[b]; b--;
                    }
                    cand_d2[b + 1] = dv2; cand_j[b + 1] = jv;
                }
            }
        }
        if (ptr >= ncand && rings_done) break;
        if (ptr >= ncand) continue;
        double dnext = sqrt(cand_d2[ptr]);
        double lb = dnext;
        if (!rings_done && covered < lb) lb = covered;
        if (lb >= stop_r) break;
        if (!rings_done && dnext * dnext > covered * covered) continue;
        i64 j = cand_j[ptr];
        ptr++;
        double D2 = cand_d2[ptr - 1];
        if (D2 <= tol * tol) {
            if (psi[j] > psii || (psi[j] == psii && j < i)) { *which_out = which; return 1; }
            continue;
        }
        w->n_clips++;
        double Dd = sqrt(D2);
        double nxp = (pts[3 * j] - px) / Dd;
        double nyp = (pts[3 * j + 1] - py) / Dd;
        double nzp = (pts[3 * j + 2] - pz) / Dd;
        double hij = 0.5 * (D2 + psii - psi[j]) / Dd;
        double dd = (nxp * px + nyp * py + nzp * pz) + hij;
        int st = which == 0 ? clip_into(A, B, nxp, nyp, nzp, dd, j, tol, &w->clip)
                            : clip_into(B, A, nxp, nyp, nzp, dd, j, tol, &w->clip);
        if (st == CLIP_EMPTY) { *which_out = which; return 1; }
        if (st == CLIP_OVERFLOW) { *which_out = which; return 3; }
        if (st == CLIP_CUT) {
            which = 1 - which;
            PCell cc = which == 0 ? A : B;
            rfar = 0.0;
            for (i64 v = 0; v < cc.c[0]; v++) {
                double d2 = sq(V(cc, v, 0) - px) + sq(V(cc, v, 1) - py) + sq(V(cc, v, 2) - pz);
                if (d2 > rfar) rfar = d2;
            }
            rfar = sqrt(rfar);
        }
    }
    *which_out = which;
    return 0;
}

static void domain_load(Domain *D, const double *dv, const i64 *dc, const double *dp, const i64 *dt,
                        const i64 *dlp, const i64 *dlv) {
    memcpy(D->dom_v, dv, sizeof(double) * 3 * MAX_V);
    memcpy(D->dom_c, dc, sizeof(i64) * 3);
    memcpy(D->dom_p, dp, sizeof(double) * 4 * MAX_F);
    memcpy(D->dom_t, dt, sizeof(i64) * MAX_F);
    memcpy(D->dom_lp, dlp, sizeof(i64) * (MAX_F + 1));
    memcpy(D->dom_lv, dlv, sizeof(i64) * MAX_L);
}

/* ---------------------------------------------------------------------------
 * exported entry points (ctypes; argument lists mirror the reference)
 * ------------------------------------------------------------------------- */

int pfo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void pfo_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* _kernels.py:1362-1478.  Processes cells [i0, i1) (whole batch when i1 <= i0).
 * clip_count (optional, may be NULL) receives the processed-candidate census. */
i64 pfo_batch_evaluate(i64 n, const double *pts, const double *psi,
                       const double *dv, const i64 *dc, const double *dp, const i64 *dt,
                       const i64 *dlp, const i64 *dlv,
                       const i64 *grid_start, const i64 *grid_sites,
                       double lox, double loy, double loz, double ihx, double ihy, double ihz,
                       i64 gnx, i64 gny, i64 gnz, double h_min, double tol, double dpsi_max,
                       int ball_aware, int want_m2, i64 smf,
                       i64 *status, double *vol, double *ksur, double *cent, double *ipt, double *m2,
                       i64 *fcount, i64 *ftag, double *farea_o, double *fh_o, double *fnrm,
                       double *fcent_o, i64 i0, i64 i1, i64 *clip_count, const i64 *cells) {
    /* cells != NULL: evaluate only cells[i0..i1) (a bounded sample) */
    if (i1 <= i0) { i0 = 0; i1 = cells ? 0 : n; }
    Domain *D = (Domain *)malloc(sizeof(Domain));
    domain_load(D, dv, dc, dp, dt, dlp, dlv);
    Grid G = {grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz, gnx, gny, gnz, h_min};
    i64 *flags_all = (i64 *)calloc((size_t)(i1 - i0 > 0 ? i1 - i0 : 1), sizeof(i64));
#pragma omp parallel
    {
        CellWork *w = (CellWork *)malloc(sizeof(CellWork));
        w->cand_d2 = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        w->cand_j = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(dynamic, 64)
        for (i64 ii = i0; ii < i1; ii++) {
            const i64 i = cells ? cells[ii] : ii;
            int which;
            int st = build_cell(i, n, pts, psi, dpsi_max, ball_aware, D, &G, tol, w, &which);
            if (clip_count) clip_count[i] = w->n_clips;
            i64 li = ii - i0;
            if (st == 3) {
                flags_all[li] = FLAG_OVERFLOW;
                status[i] = CELL_EMPTY; vol[i] = 0.0; ksur[i] = 0.0; fcount[i] = 0;
                continue;
            }
            if (st == 1) {
                status[i] = CELL_EMPTY; vol[i] = 0.0; ksur[i] = 0.0;
                for (int k = 0; k < 3; k++) { cent[3 * i + k] = pts[3 * i + k]; ipt[3 * i + k] = pts[3 * i + k]; }
                m2[i] = 0.0; fcount[i] = 0;
                continue;
            }
            PCell C = which == 0 ? cw_A(w) : cw_B(w);
            i64 nf = C.c[1];
            double r[10];
            i64 fl = evaluate_cell(C, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], psi[i], tol, want_m2, &w->ev, r);
            flags_all[li] = fl;
            status[i] = (i64)r[0]; vol[i] = r[1]; ksur[i] = r[2];
            cent[3 * i] = r[3]; cent[3 * i + 1] = r[4]; cent[3 * i + 2] = r[5];
            ipt[3 * i] = r[6]; ipt[3 * i + 1] = r[7]; ipt[3 * i + 2] = r[8];
            m2[i] = r[9];
            i64 nk = 0;
            if ((i64)r[0] == CELL_CLIPPED) {
                for (i64 f = 0; f < nf; f++) {
                    if (w->ev.fkind[f] == RF_OUTSIDE || w->ev.farea[f] <= 0.0) continue;
                    if (nk >= smf) { flags_all[li] |= FLAG_OVERFLOW; break; }
                    i64 o = i * smf + nk;
                    ftag[o] = C.tg[f];
                    farea_o[o] = w->ev.farea[f];
                    fh_o[o] = w->ev.fh[f];
                    fnrm[3 * o] = PL(C, f, 0); fnrm[3 * o + 1] = PL(C, f, 1); fnrm[3 * o + 2] = PL(C, f, 2);
                    fcent_o[3 * o] = w->ev.fcx[f]; fcent_o[3 * o + 1] = w->ev.fcy[f]; fcent_o[3 * o + 2] = w->ev.fcz[f];
                    nk++;
                }
            }
            fcount[i] = nk;
        }
        free(w->cand_d2); free(w->cand_j); free(w);
    }
    i64 err = 0;
    for (i64 i = 0; i < i1 - i0; i++) err |= flags_all[i];
    free(flags_all); free(D);
    return err;
}

/* _kernels.py:1481-1559 */
i64 pfo_batch_build(i64 n, const double *pts, const double *psi,
                    const double *dv, const i64 *dc, const double *dp, const i64 *dt,
                    const i64 *dlp, const i64 *dlv,
                    const i64 *grid_start, const i64 *grid_sites,
                    double lox, double loy, double loz, double ihx, double ihy, double ihz,
                    i64 gnx, i64 gny, i64 gnz, double h_min, double tol, double dpsi_max,
                    int ball_aware, i64 smv, i64 smf, i64 sml,
                    i64 *out_status, i64 *out_nv, i64 *out_nf, i64 *out_nl,
                    double *out_verts, double *out_planes, i64 *out_tags, i64 *out_lp, i64 *out_lv) {
    Domain *D = (Domain *)malloc(sizeof(Domain));
    domain_load(D, dv, dc, dp, dt, dlp, dlv);
    Grid G = {grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz, gnx, gny, gnz, h_min};
    i64 *flags_all = (i64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(i64));
#pragma omp parallel
    {
        CellWork *w = (CellWork *)malloc(sizeof(CellWork));
        w->cand_d2 = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        w->cand_j = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(dynamic, 64)
        for (i64 i = 0; i < n; i++) {
            int which;
            int st = build_cell(i, n, pts, psi, dpsi_max, ball_aware, D, &G, tol, w, &which);
            if (st == 1) { out_status[i] = 1; out_nv[i] = 0; out_nf[i] = 0; out_nl[i] = 0; continue; }
            if (st == 3) { out_status[i] = 3; flags_all[i] = FLAG_OVERFLOW; continue; }
            PCell C = which == 0 ? cw_A(w) : cw_B(w);
            if (C.c[0] > smv || C.c[1] > smf || C.c[2] > sml) {
                out_status[i] = 3; flags_all[i] = FLAG_OVERFLOW; continue;
            }
            out_status[i] = 0; out_nv[i] = C.c[0]; out_nf[i] = C.c[1]; out_nl[i] = C.c[2];
            for (i64 v = 0; v < C.c[0]; v++)
                for (int k = 0; k < 3; k++) out_verts[(i * smv + v) * 3 + k] = V(C, v, k);
            for (i64 f = 0; f < C.c[1]; f++) {
                for (int k = 0; k < 4; k++) out_planes[(i * smf + f) * 4 + k] = PL(C, f, k);
                out_tags[i * smf + f] = C.tg[f];
                out_lp[i * (smf + 1) + f] = C.lp[f];
            }
            out_lp[i * (smf + 1) + C.c[1]] = C.lp[C.c[1]];
            for (i64 k = 0; k < C.c[2]; k++) out_lv[i * sml + k] = C.lv[k];
        }
        free(w->cand_d2); free(w->cand_j); free(w);
    }
    i64 err = 0;
    for (i64 i = 0; i < n; i++) err |= flags_all[i];
    free(flags_all); free(D);
    return err;
}

/* _kernels.py:1562-1620 */
i64 pfo_knn(i64 n, const double *pts, const i64 *grid_start, const i64 *grid_sites,
            double lox, double loy, double loz, double ihx, double ihy, double ihz,
            i64 gnx, i64 gny, i64 gnz, double h_min, double qx, double qy, double qz,
            i64 k, i64 *out_idx) {
    if (k > n) k = n;
    if (k <= 0) return 0;
    Grid G = {grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz, gnx, gny, gnz, h_min};
    double *cand_d2 = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    i64 *cand_j = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    i64 ncand = 0;
    i64 bb[3];
    bucket_of(&G, qx, qy, qz, bb);
    i64 ring = 0;
    double covered = 0.0;
    i64 got = 0;
    for (;;) {
        int any_cell = 0;
        for (i64 dx = -ring; dx <= ring; dx++) {
            i64 ix = bb[0] + dx;
            if (ix < 0 || ix >= gnx) continue;
            for (i64 dy = -ring; dy <= ring; dy++) {
                i64 iy = bb[1] + dy;
                if (iy < 0 || iy >= gny) continue;
                for (i64 dz = -ring; dz <= ring; dz++) {
                    i64 adx = dx < 0 ? -dx : dx, ady = dy < 0 ? -dy : dy, adz = dz < 0 ? -dz : dz;
                    i64 mxa = adx > ady ? adx : ady;
                    if (adz > mxa) mxa = adz;
                    if (mxa != ring) continue;
                    i64 iz = bb[2] + dz;
                    if (iz < 0 || iz >= gnz) continue;
                    any_cell = 1;
                    i64 lin = (ix * gny + iy) * gnz + iz;
                    for (i64 q = grid_start[lin]; q < grid_start[lin + 1]; q++) {
                        i64 j = grid_sites[q];
                        cand_d2[ncand] = sq(pts[3 * j] - qx) + sq(pts[3 * j + 1] - qy) + sq(pts[3 * j + 2] - qz);
                        cand_j[ncand] = j;
                        ncand++;
                    }
                }
            }
        }
        covered = (double)ring * h_min;
        ring++;
        int done_grid = ring > gnx + gny + gnz && !any_cell;
        if (ncand >= k || done_grid) {
            for (i64 a = 1; a < ncand; a++) {
                double dv2 = cand_d2[a];
                i64 jv = cand_j[a];
                i64 b = a - 1;
                while (b >= 0 && (cand_d2[b] > dv2 || (cand_d2[b] == dv2 && cand_j[b] > jv))) {
                    cand_d2[b + 1] = cand_d2[b]; cand_j[b + 1] = cand_j[b]; b--;
                }
                cand_d2[b + 1] = dv2; cand_j[b + 1] = jv;
            }
            if (done_grid || (ncand >= k && cand_d2[k - 1] <= covered * covered)) {
                for (i64 q = 0; q < k; q++) out_idx[q] = cand_j[q];
                got = k;
                break;
            }
        }
    }
    free(cand_d2); free(cand_j);
    return got;
}

/* single-clip utility (geom.clip_cell, geom.py:478-503) */
int pfo_clip(const double *va, const i64 *ca, const double *pa, const i64 *ta, const i64 *lpa,
             const i64 *lva, double *vb, i64 *cb, double *pb, i64 *tb, i64 *lpb, i64 *lvb,
             double nx, double ny, double nz, double dd, i64 tag, double tol) {
    ClipScratch *S = (ClipScratch *)malloc(sizeof(ClipScratch));
    PCell A = {(double *)va, (i64 *)ca, (double *)pa, (i64 *)ta, (i64 *)lpa, (i64 *)lva};
    PCell B = {vb, cb, pb, tb, lpb, lvb};
    int st = clip_into(A, B, nx, ny, nz, dd, tag, tol, S);
    free(S);
    return st;
}

/* generalized polygon integrals (geom.polygon_area & co., geom.py:316-346) */
void pfo_piece_integrals(const double *pieces, i64 npc, double *out) {
    piece_integrals(pieces, npc, out);
}
