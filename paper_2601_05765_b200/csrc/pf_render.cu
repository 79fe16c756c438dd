// pf_render.cu -- offline rendering of the fluid surface straight from the
// restricted diagram (SPEC.md:406-463 module `renderer`, PAPER.md:392-436;
// SURVEY §8(f) row 4), thread per pixel / per sample.
//
// The fluid is the union of the restricted cells, i.e. the set of points whose
// power-nearest site's ball contains them -- the union of the balls
// B(p_i, sqrt(psi_i)).  Hence:
//  * first_hit (SPEC "nearest ray-sphere hit inside the owning cell") is the
//    smallest entry parameter over the balls: the first point of the union
//    lies on the entered ball's sphere, in that ball's Laguerre cell;
//  * Depth (SPEC "normalized in-fluid path length") is the length of the ray
//    inside the union of the balls: the union of the per-ball chords;
//  * sample_surface draws points uniformly on the free-surface patches K_i:
//    a point of sphere i belongs to K_i iff no other ball strictly contains it
//    and it lies in the domain;
//  * Smooth sphere-traces the cubic smooth union of the sphere distances.
// Every ray walks the bucket grid of pf_grid_build with a 3D DDA; at each
// bucket it tests the sites of the buckets within the largest ball radius.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/potflow_b200.h"

extern unsigned long long pf_internal_launches_add(unsigned long long k);
extern int pf_internal_set_err(const char *msg);

namespace {

#define RCK(x)                                                                       \
    do {                                                                             \
        cudaError_t _e = (x);                                                        \
        if (_e != cudaSuccess) {                                                     \
            char _b[256];                                                            \
            snprintf(_b, sizeof _b, "%s:%d %s: %s", __FILE__, __LINE__, #x,         \
                     cudaGetErrorString(_e));                                        \
            return pf_internal_set_err(_b);                                          \
        }                                                                            \
    } while (0)

struct Grid {
    const double *pts;  // [n, 3] original order
    const double *sx, *sy, *sz;
    const int *sid, *bstart;
    int gn[3];
    double lo[3], h[3];
    int reach;  // buckets within the largest ball radius
};

__device__ __forceinline__ bool bucket_ok(const Grid &g, int bx, int by, int bz) {
    return bx >= 0 && by >= 0 && bz >= 0 && bx < g.gn[0] && by < g.gn[1] && bz < g.gn[2];
}

// smallest t >= tmin with the ray entering a ball of the sites in bucket b
__device__ void test_bucket(const Grid &g, int bx, int by, int bz, const double *o, const double *d,
                            const double *__restrict__ psi, double tmin, double &best, int &who) {
    if (!bucket_ok(g, bx, by, bz)) return;
    const int lin = (bx * g.gn[1] + by) * g.gn[2] + bz;
    for (int s = g.bstart[lin]; s < g.bstart[lin + 1]; s++) {
        const int i = g.sid[s];
        const double ps = psi[i];
        if (!(ps > 0.0)) continue;
        const double wx = o[0] - g.sx[s], wy = o[1] - g.sy[s], wz = o[2] - g.sz[s];
        const double b = d[0] * wx + d[1] * wy + d[2] * wz;
        const double c = wx * wx + wy * wy + wz * wz - ps;
        const double disc = b * b - c;
        if (disc < 0.0) continue;
        const double t = -b - sqrt(disc);
        const double te = t >= tmin ? t : (c <= 0.0 ? tmin : -1.0);  // origin inside the ball: hit at tmin
        if (te >= tmin && (te < best || (te == best && i < who))) { best = te; who = i; }
    }
}

// pixel ray (cam: eye[3], forward[3], right[3], up[3], tan(fov/2), aspect),
// clipped to the grid box: false when it misses the box
struct Ray {
    double o[3], d[3], t0, t1;
};
__device__ bool pixel_ray(const Grid &g, const double *cam, int px, int py, int w, int h, Ray &r) {
    const double sx = (2.0 * (px + 0.5) / w - 1.0) * cam[12] * cam[13];
    const double sy = (1.0 - 2.0 * (py + 0.5) / h) * cam[12];
    for (int a = 0; a < 3; a++) r.d[a] = cam[3 + a] + sx * cam[6 + a] + sy * cam[9 + a];
    const double dn = sqrt(r.d[0] * r.d[0] + r.d[1] * r.d[1] + r.d[2] * r.d[2]);
    for (int a = 0; a < 3; a++) { r.d[a] /= dn; r.o[a] = cam[a]; }
    r.t0 = 0.0;
    r.t1 = 1e300;
    for (int a = 0; a < 3; a++) {
        const double lo = g.lo[a], hi = g.lo[a] + g.gn[a] * g.h[a];
        if (fabs(r.d[a]) < 1e-300) {
            if (r.o[a] < lo || r.o[a] > hi) return false;
            continue;
        }
        double ta = (lo - r.o[a]) / r.d[a], tb = (hi - r.o[a]) / r.d[a];
        if (ta > tb) { const double tt = ta; ta = tb; tb = tt; }
        r.t0 = fmax(r.t0, ta);
        r.t1 = fmin(r.t1, tb);
    }
    return r.t0 <= r.t1;
}

// 3D DDA over the buckets the ray crosses
struct DDA {
    int b[3], step[3];
    double tnext[3], tdel[3];
    __device__ void init(const Grid &g, const Ray &r) {
        for (int a = 0; a < 3; a++) {
            const double p = r.o[a] + r.t0 * r.d[a];
            const int c = (int)floor((p - g.lo[a]) / g.h[a]);
            b[a] = c < 0 ? 0 : (c >= g.gn[a] ? g.gn[a] - 1 : c);
            if (r.d[a] > 0.0) {
                step[a] = 1;
                tnext[a] = (g.lo[a] + (b[a] + 1) * g.h[a] - r.o[a]) / r.d[a];
                tdel[a] = g.h[a] / r.d[a];
            } else if (r.d[a] < 0.0) {
                step[a] = -1;
                tnext[a] = (g.lo[a] + b[a] * g.h[a] - r.o[a]) / r.d[a];
                tdel[a] = -g.h[a] / r.d[a];
            } else {
                step[a] = 0;
                tnext[a] = 1e300;
                tdel[a] = 1e300;
            }
        }
    }
    __device__ double exit_t() const { return fmin(tnext[0], fmin(tnext[1], tnext[2])); }
    // next bucket; false when the ray leaves the grid
    __device__ bool advance(const Grid &g) {
        const int a = tnext[0] <= tnext[1] ? (tnext[0] <= tnext[2] ? 0 : 2) : (tnext[1] <= tnext[2] ? 1 : 2);
        b[a] += step[a];
        if (b[a] < 0 || b[a] >= g.gn[a]) return false;
        tnext[a] += tdel[a];
        return true;
    }
};

__global__ void k_first_hit(Grid g, const double *__restrict__ psi, int w, int h, const double *cam,
                            int *__restrict__ hit_id, double *__restrict__ hit_t) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y * blockDim.y + threadIdx.y;
    if (px >= w || py >= h) return;
    double best = 1e300;
    int who = -1;
    Ray r;
    if (pixel_ray(g, cam, px, py, w, h, r)) {
        DDA q;
        q.init(g, r);
        const int R = g.reach;
        for (int guard = 0; guard < 4 * (g.gn[0] + g.gn[1] + g.gn[2]) + 8; guard++) {
            for (int i = -R; i <= R; i++)
                for (int j = -R; j <= R; j++)
                    for (int k = -R; k <= R; k++)
                        test_bucket(g, q.b[0] + i, q.b[1] + j, q.b[2] + k, r.o, r.d, psi, r.t0, best, who);
            const double texit = q.exit_t();
            if (best <= texit || texit > r.t1) break;
            if (!q.advance(g)) break;
        }
    }
    hit_id[py * w + px] = who;
    hit_t[py * w + px] = who >= 0 ? best : -1.0;
}

// Depth: length of the ray inside the union of the balls (clipped to the grid
// box, which holds the domain).  Every ball chord [a, b] is assigned to the
// DDA segment holding its entry a (half-open segments partition [t0, t1]); the
// ball is found there, since ray(a) lies on its sphere within rmax <= reach of
// the segment's bucket.  Processing the chords by increasing a -- segment by
// segment, insertion-sorted inside one -- the union length is the classic
// sweep: len += max(0, b - max(a, c)), c = max(c, b).
enum { DEPTH_MAXI = 48 };
__global__ void k_depth(Grid g, const double *__restrict__ psi, int w, int h, const double *cam,
                        double *__restrict__ depth) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y * blockDim.y + threadIdx.y;
    if (px >= w || py >= h) return;
    double len = 0.0;
    Ray r;
    if (pixel_ray(g, cam, px, py, w, h, r)) {
        DDA q;
        q.init(g, r);
        const int R = g.reach;
        double ia[DEPTH_MAXI], ib[DEPTH_MAXI];
        double cov = r.t0, s0 = r.t0;
        for (int guard = 0; guard < 4 * (g.gn[0] + g.gn[1] + g.gn[2]) + 8; guard++) {
            const double texit = q.exit_t();
            const double s1 = fmin(texit, r.t1);
            int ni = 0;
            for (int i = -R; i <= R; i++)
                for (int j = -R; j <= R; j++)
                    for (int k = -R; k <= R; k++) {
                        const int bx = q.b[0] + i, by = q.b[1] + j, bz = q.b[2] + k;
                        if (!bucket_ok(g, bx, by, bz)) continue;
                        const int lin = (bx * g.gn[1] + by) * g.gn[2] + bz;
                        for (int s = g.bstart[lin]; s < g.bstart[lin + 1]; s++) {
                            const double ps = psi[g.sid[s]];
                            if (!(ps > 0.0)) continue;
                            const double wx = r.o[0] - g.sx[s], wy = r.o[1] - g.sy[s], wz = r.o[2] - g.sz[s];
                            const double b = r.d[0] * wx + r.d[1] * wy + r.d[2] * wz;
                            const double disc = b * b - (wx * wx + wy * wy + wz * wz - ps);
                            if (disc < 0.0) continue;
                            const double sq = sqrt(disc);
                            const double a = fmax(-b - sq, r.t0), e = fmin(-b + sq, r.t1);
                            if (!(e > a) || a < s0 || a >= s1) continue;
                            if (ni == DEPTH_MAXI) { len = -1.0; goto done; }
                            int u = ni++;
                            while (u > 0 && ia[u - 1] > a) { ia[u] = ia[u - 1]; ib[u] = ib[u - 1]; u--; }
                            ia[u] = a;
                            ib[u] = e;
                        }
                    }
            for (int u = 0; u < ni; u++) {
                const double lo = fmax(ia[u], cov);
                if (ib[u] > lo) len += ib[u] - lo;
                cov = fmax(cov, ib[u]);
            }
            if (texit >= r.t1) break;
            if (!q.advance(g)) break;
            s0 = s1;
        }
    }
done:
    depth[py * w + px] = len;
}

// Cubic smooth union of the sphere distances d_j = |x - p_j| - sqrt(psi_j):
//   f = d_min - (k/6) sum_{j != argmin} h_j^3,  h_j = max(k - (d_j - d_min), 0) / k
// (for two spheres the cubic polynomial smooth-min; k -> 0 gives the plain
// min; f <= d_min everywhere).  Spheres within reach of x's bucket; when none
// is nearer than the neighbourhood's coverage, the coverage bound is returned
// (a lower bound of the distance, enough for the tracing step).  *lip: a local
// Lipschitz bound 1 + sum h_j^2 for the tracing step.
__device__ double smooth_sdf(const Grid &g, const double *__restrict__ psi, const double *x, double k, double rmax,
                             int R, double *lip) {
    int c[3];
    double out = 0.0;  // distance from x to the grid box
    for (int a = 0; a < 3; a++) {
        const double t = (x[a] - g.lo[a]) / g.h[a];
        const int b = (int)floor(t);
        c[a] = b < 0 ? 0 : (b >= g.gn[a] ? g.gn[a] - 1 : b);
        const double lo = g.lo[a], hi = g.lo[a] + g.gn[a] * g.h[a];
        const double o = x[a] < lo ? lo - x[a] : (x[a] > hi ? x[a] - hi : 0.0);
        out = fmax(out, o);
    }
    const double hmin = fmin(g.h[0], fmin(g.h[1], g.h[2]));
    const double cover = R * hmin + out - rmax;  // every sphere outside the neighbourhood is farther
    double dmin = 1e300;
    for (int i = -R; i <= R; i++)
        for (int j = -R; j <= R; j++)
            for (int l = -R; l <= R; l++) {
                const int bx = c[0] + i, by = c[1] + j, bz = c[2] + l;
                if (!bucket_ok(g, bx, by, bz)) continue;
                const int lin = (bx * g.gn[1] + by) * g.gn[2] + bz;
                for (int s = g.bstart[lin]; s < g.bstart[lin + 1]; s++) {
                    const double ps = psi[g.sid[s]];
                    if (!(ps > 0.0)) continue;
                    const double dx = x[0] - g.sx[s], dy = x[1] - g.sy[s], dz = x[2] - g.sz[s];
                    dmin = fmin(dmin, sqrt(dx * dx + dy * dy + dz * dz) - sqrt(ps));
                }
            }
    *lip = 1.0;
    if (!(dmin < cover)) return cover;
    double sum = 0.0, l2 = 0.0;
    bool self = false;  // the argmin itself (first sphere at d_min) is not a term
    for (int i = -R; i <= R; i++)
        for (int j = -R; j <= R; j++)
            for (int l = -R; l <= R; l++) {
                const int bx = c[0] + i, by = c[1] + j, bz = c[2] + l;
                if (!bucket_ok(g, bx, by, bz)) continue;
                const int lin = (bx * g.gn[1] + by) * g.gn[2] + bz;
                for (int s = g.bstart[lin]; s < g.bstart[lin + 1]; s++) {
                    const double ps = psi[g.sid[s]];
                    if (!(ps > 0.0)) continue;
                    const double dx = x[0] - g.sx[s], dy = x[1] - g.sy[s], dz = x[2] - g.sz[s];
                    const double dj = sqrt(dx * dx + dy * dy + dz * dz) - sqrt(ps);
                    if (dj == dmin && !self) { self = true; continue; }
                    const double hj = fmax(k - (dj - dmin), 0.0) / k;
                    sum += hj * hj * hj;
                    l2 += hj * hj;
                }
            }
    *lip = 1.0 + l2;
    return dmin - (k / 6.0) * sum;
}

// Smooth: sphere tracing of smooth_sdf (<= 64 steps, surface eps), from just
// before the Raw hit (the smooth surface encloses the union of the balls); rays
// without a Raw hit start at the grid entry.  Normal: central differences.
__global__ void k_smooth(Grid g, const double *__restrict__ psi, int w, int h, const double *cam, double k,
                         double rmax, int R, double eps, const double *__restrict__ raw_t,
                         double *__restrict__ out_t, double *__restrict__ out_n) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y * blockDim.y + threadIdx.y;
    if (px >= w || py >= h) return;
    const int pix = py * w + px;
    double th = -1.0, nrm[3] = {0.0, 0.0, 0.0};
    Ray r;
    if (pixel_ray(g, cam, px, py, w, h, r)) {
        const double tr = raw_t[pix];
        double t = tr >= 0.0 ? fmax(r.t0, tr - 2.0 * k - 4.0 * eps) : r.t0;
        for (int it = 0; it < 64 && t <= r.t1; it++) {
            double x[3], lip;
            for (int a = 0; a < 3; a++) x[a] = r.o[a] + t * r.d[a];
            const double f = smooth_sdf(g, psi, x, k, rmax, R, &lip);
            if (f < eps) { th = t; break; }
            t += f / lip;
        }
        if (th < 0.0 && tr >= 0.0) th = tr;  // step budget spent: keep the Raw hit
        if (th >= 0.0) {
            const double e = fmax(eps, 1e-9);
            double x[3], lip;
            for (int a = 0; a < 3; a++) x[a] = r.o[a] + th * r.d[a];
            for (int a = 0; a < 3; a++) {
                const double xa = x[a];
                x[a] = xa + e;
                const double fp = smooth_sdf(g, psi, x, k, rmax, R, &lip);
                x[a] = xa - e;
                const double fm = smooth_sdf(g, psi, x, k, rmax, R, &lip);
                x[a] = xa;
                nrm[a] = fp - fm;
            }
            const double nn = sqrt(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
            for (int a = 0; a < 3; a++) nrm[a] = nn > 0.0 ? nrm[a] / nn : 0.0;
        }
    }
    out_t[pix] = th;
    for (int a = 0; a < 3; a++) out_n[3 * pix + a] = nrm[a];
}

__global__ void k_sdf_points(Grid g, const double *__restrict__ psi, int64_t m, const double *__restrict__ xq,
                             double k, double rmax, int R, double *__restrict__ out) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        double lip;
        out[q] = smooth_sdf(g, psi, xq + 3 * q, k, rmax, R, &lip);
    }
}

// counter-based uniform in [0, 1): splitmix64 of (seed, sample, draw)
__device__ __forceinline__ double urand(uint64_t seed, uint64_t s, uint64_t k) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (s * 0x100000001B3ull + k + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

// sample_surface: sample q draws uniform points on sphere cell[q] until one
// lies on the free-surface patch K_i (in the domain, strictly inside no other
// ball); at most max_tries[q] draws (status[q] = 1 when exhausted)
__global__ void k_sample(Grid g, const double *__restrict__ pts, const double *__restrict__ psi, int64_t m,
                         const int64_t *__restrict__ cell, const int64_t *__restrict__ max_tries,
                         const double *__restrict__ dp, int dnf, uint64_t seed, double *__restrict__ xo,
                         double *__restrict__ no, int32_t *__restrict__ status) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = cell[q];
        const double r = sqrt(psi[i]);
        const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        int st = 1;
        double x[3] = {p[0], p[1], p[2]}, u[3] = {0.0, 0.0, 1.0};
        for (int64_t tr = 0; tr < max_tries[q]; tr++) {
            const double z = 1.0 - 2.0 * urand(seed, (uint64_t)q, 2 * (uint64_t)tr);
            const double ph = 6.283185307179586 * urand(seed, (uint64_t)q, 2 * (uint64_t)tr + 1);
            const double s = sqrt(fmax(0.0, 1.0 - z * z));
            u[0] = s * cos(ph); u[1] = s * sin(ph); u[2] = z;
            for (int a = 0; a < 3; a++) x[a] = p[a] + r * u[a];
            bool ok = true;
            for (int f = 0; f < dnf && ok; f++)
                if (dp[4 * f] * x[0] + dp[4 * f + 1] * x[1] + dp[4 * f + 2] * x[2] > dp[4 * f + 3]) ok = false;
            int c[3];
            for (int a = 0; a < 3; a++) {
                const int b = (int)floor((x[a] - g.lo[a]) / g.h[a]);
                c[a] = b < 0 ? 0 : (b >= g.gn[a] ? g.gn[a] - 1 : b);
            }
            const int R = g.reach;
            for (int di = -R; di <= R && ok; di++)
                for (int dj = -R; dj <= R && ok; dj++)
                    for (int dk = -R; dk <= R && ok; dk++) {
                        const int bx = c[0] + di, by = c[1] + dj, bz = c[2] + dk;
                        if (!bucket_ok(g, bx, by, bz)) continue;
                        const int lin = (bx * g.gn[1] + by) * g.gn[2] + bz;
                        for (int sl = g.bstart[lin]; sl < g.bstart[lin + 1]; sl++) {
                            const int j = g.sid[sl];
                            if (j == i) continue;
                            const double dx = x[0] - g.sx[sl], dy = x[1] - g.sy[sl], dz = x[2] - g.sz[sl];
                            if (dx * dx + dy * dy + dz * dz < psi[j]) { ok = false; break; }
                        }
                    }
            if (ok) { st = 0; break; }
        }
        for (int a = 0; a < 3; a++) { xo[3 * q + a] = x[a]; no[3 * q + a] = u[a]; }
        status[q] = st;
    }
}


// ---------------------------------------------------------------------------
// traverse (SPEC renderer `traverse`, PAPER §6 "load the current cell's
// neighbors and iteratively intersect facets facing the ray ... until the
// closest facet is the domain boundary"): thread per ray, walking the
// unrestricted power diagram (packed cells of pf_batch_build in full mode).
// The fluid is the union of V_i ∩ B_i, so within the power cell i the fluid
// part of the ray is its chord of the ball B_i: every cell span is split into
// air / fluid / air pieces.  SurfaceOnly stops after the first fluid piece that
// leaves through the sphere.  Consecutive pieces share their end points.
// ---------------------------------------------------------------------------
// power-nearest site of x (lowest index on ties): cube searches of growing
// half width r until no site outside can be nearer in power distance
__device__ int power_nearest(const Grid &g, const double *__restrict__ psi, double psimax, const double *x) {
    const double hmin = fmin(g.h[0], fmin(g.h[1], g.h[2]));
    double r = hmin;
    int best = -1;
    double bd = 1e300;
    for (int it = 0; it < 64; it++) {
        int lo[3], hi[3];
        for (int a = 0; a < 3; a++) {
            lo[a] = (int)floor((x[a] - r - g.lo[a]) / g.h[a]);
            hi[a] = (int)floor((x[a] + r - g.lo[a]) / g.h[a]);
            lo[a] = lo[a] < 0 ? 0 : (lo[a] >= g.gn[a] ? g.gn[a] - 1 : lo[a]);
            hi[a] = hi[a] < 0 ? 0 : (hi[a] >= g.gn[a] ? g.gn[a] - 1 : hi[a]);
        }
        for (int bx = lo[0]; bx <= hi[0]; bx++)
            for (int by = lo[1]; by <= hi[1]; by++)
                for (int bz = lo[2]; bz <= hi[2]; bz++) {
                    const int lin = (bx * g.gn[1] + by) * g.gn[2] + bz;
                    for (int s = g.bstart[lin]; s < g.bstart[lin + 1]; s++) {
                        const int i = g.sid[s];
                        const double dx = x[0] - g.sx[s], dy = x[1] - g.sy[s], dz = x[2] - g.sz[s];
                        const double pd = dx * dx + dy * dy + dz * dz - psi[i];
                        if (pd < bd || (pd == bd && i < best)) { bd = pd; best = i; }
                    }
                }
        const bool all = lo[0] == 0 && lo[1] == 0 && lo[2] == 0 && hi[0] == g.gn[0] - 1 && hi[1] == g.gn[1] - 1 &&
                         hi[2] == g.gn[2] - 1;
        if (all) break;
        if (best >= 0) {
            // a site at distance > r has power distance > r^2 - psimax
            const double need = bd + psimax;
            if (need <= r * r) break;
            r = fmax(2.0 * r, sqrt(fmax(need, 0.0)) * (1.0 + 1e-12));
        } else {
            r *= 2.0;
        }
    }
    return best;
}

__global__ void k_traverse(Grid g, const double *__restrict__ psi, double psimax, const double *__restrict__ dp,
                           int dnf, int smf, const int32_t *__restrict__ cnf, const double *__restrict__ planes,
                           const int32_t *__restrict__ tags, int64_t m, const double *__restrict__ rays, int mode,
                           int max_seg, int64_t max_steps, int32_t *__restrict__ out_cell, double *__restrict__ out_t0,
                           double *__restrict__ out_t1, uint8_t *__restrict__ out_fluid, int32_t *__restrict__ count,
                           int32_t *__restrict__ status) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        const double o[3] = {rays[6 * r], rays[6 * r + 1], rays[6 * r + 2]};
        const double d[3] = {rays[6 * r + 3], rays[6 * r + 4], rays[6 * r + 5]};
        int nseg = 0, st = 0;
        // the ray inside the (convex) domain: [t0, t1]
        double t0 = 0.0, t1 = 1e300;
        bool miss = false;
        for (int f = 0; f < dnf && !miss; f++) {
            const double nd = dp[4 * f] * d[0] + dp[4 * f + 1] * d[1] + dp[4 * f + 2] * d[2];
            const double gap = dp[4 * f + 3] - (dp[4 * f] * o[0] + dp[4 * f + 1] * o[1] + dp[4 * f + 2] * o[2]);
            if (fabs(nd) < 1e-300) { if (gap < 0.0) miss = true; continue; }
            const double t = gap / nd;
            if (nd > 0.0) t1 = fmin(t1, t); else t0 = fmax(t0, t);
        }
        if (miss || !(t0 < t1)) {
            count[r] = 0;
            status[r] = 1;
            continue;
        }
        const double tm0 = t0 + 1e-9 * (t1 - t0);  // just inside the entry face
        const double x0[3] = {o[0] + tm0 * d[0], o[1] + tm0 * d[1], o[2] + tm0 * d[2]};
        int i = power_nearest(g, psi, psimax, x0);
        int prev = -1;
        double tin = t0;
        for (int64_t step = 0; i >= 0; step++) {
            if (step >= max_steps) { st = 2; break; }
            // exit through the nearest facet facing the ray (not the one entered by)
            double tout = t1;
            int next = -1;
            const int nfi = cnf[i];
            for (int f = 0; f < nfi; f++) {
                const double *pl = planes + ((int64_t)i * smf + f) * 4;
                const int tg = tags[(int64_t)i * smf + f];
                if (tg >= 0 && tg == prev) continue;
                const double nd = pl[0] * d[0] + pl[1] * d[1] + pl[2] * d[2];
                if (!(nd > 1e-300)) continue;
                double t = (pl[3] - (pl[0] * o[0] + pl[1] * o[1] + pl[2] * o[2])) / nd;
                if (t < tin) t = tin;
                if (t < tout || (t == tout && tg >= 0 && (next < 0 || tg < next))) { tout = t; next = tg; }
            }
            if (tout >= t1) { tout = t1; next = -1; }
            // the span's pieces: air / fluid (the chord of B_i) / air
            double ta = 1e300, tb = -1e300;  // chord of the ball B(p_i, sqrt(psi_i))
            bool stop = false;
            {
                const double *pp = g.pts + 3 * (int64_t)i;
                const double wx = o[0] - pp[0], wy = o[1] - pp[1], wz = o[2] - pp[2];
                const double b = d[0] * wx + d[1] * wy + d[2] * wz;
                const double c = wx * wx + wy * wy + wz * wz - psi[i];
                const double disc = b * b - c;
                if (psi[i] > 0.0 && disc > 0.0) {
                    const double sq = sqrt(disc);
                    ta = -b - sq;
                    tb = -b + sq;
                }
            }
            const double fa = fmax(tin, ta), fb = fmin(tout, tb);
            double cut[4];
            int np = 0;
            cut[np++] = tin;
            if (fa < fb) {
                if (fa > tin) cut[np++] = fa;
                if (fb < tout) cut[np++] = fb;
            }
            cut[np++] = tout;
            for (int k = 0; k + 1 < np; k++) {
                const double a = cut[k], bq = cut[k + 1];
                if (!(bq > a)) continue;  // a zero-length span (an edge or vertex crossing)
                const bool fl = fa < fb && a >= fa && bq <= fb;
                if (nseg >= max_seg) { st = 2; stop = true; break; }
                const int64_t q = r * (int64_t)max_seg + nseg++;
                out_cell[q] = i;
                out_t0[q] = a;
                out_t1[q] = bq;
                out_fluid[q] = fl ? 1 : 0;
                if (mode == 1 && fl && bq < tout) { stop = true; break; }  // surface exit
            }
            if (stop || next < 0) break;
            prev = i;
            i = next;
            tin = tout;
        }
        count[r] = nseg;
        status[r] = st;
    }
}

}  // namespace

// defined in pf_runtime.cu
int pf_internal_grid_view(pf_ctx *c, const double **sx, const double **sy, const double **sz, const int **sid,
                          const int **bstart, int *gn, double *lo, double *h);
int pf_internal_domain_view(pf_ctx *c, const double **dp, int *nf, double *tol);

static int render_grid(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax, double extra,
                       Grid &g, void *stream) {
    if (pf_grid_build(ctx, n, pts, psi, 0.0, stream)) return -1;
    if (pf_internal_grid_view(ctx, &g.sx, &g.sy, &g.sz, &g.sid, &g.bstart, g.gn, g.lo, g.h)) return -1;
    g.pts = pts;
    const double hmin = fmin(g.h[0], fmin(g.h[1], g.h[2]));
    g.reach = (int)ceil((rmax + extra) / hmin);
    if (g.reach < 1) g.reach = 1;
    if (g.reach > 8) g.reach = 8;
    return 0;
}

static int upload_cam(const double *cam_host, double **cam, cudaStream_t st) {
    RCK(cudaMallocAsync((void **)cam, 14 * sizeof(double), st));
    RCK(cudaMemcpyAsync(*cam, cam_host, 14 * sizeof(double), cudaMemcpyHostToDevice, st));
    return 0;
}

extern "C" int pf_render_first_hit(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax,
                                   const double *cam_host, int width, int height, int32_t *hit_id,
                                   double *hit_t, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Grid g;
    if (render_grid(ctx, n, pts, psi, rmax, 0.0, g, stream)) return -1;
    double *cam = nullptr;
    if (upload_cam(cam_host, &cam, st)) return -1;
    dim3 blk(16, 8), grd((width + 15) / 16, (height + 7) / 8);
    pf_internal_launches_add(1);
    k_first_hit<<<grd, blk, 0, st>>>(g, psi, width, height, cam, hit_id, hit_t);
    RCK(cudaGetLastError());
    RCK(cudaFreeAsync(cam, st));
    RCK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int pf_render_depth(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax,
                               const double *cam_host, int width, int height, double *depth, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Grid g;
    if (render_grid(ctx, n, pts, psi, rmax, 0.0, g, stream)) return -1;
    double *cam = nullptr;
    if (upload_cam(cam_host, &cam, st)) return -1;
    dim3 blk(16, 8), grd((width + 15) / 16, (height + 7) / 8);
    pf_internal_launches_add(1);
    k_depth<<<grd, blk, 0, st>>>(g, psi, width, height, cam, depth);
    RCK(cudaGetLastError());
    RCK(cudaFreeAsync(cam, st));
    RCK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int pf_render_smooth(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax,
                                double k, double eps, const double *cam_host, int width, int height,
                                const double *raw_t, double *hit_t, double *normal, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!(k > 0.0)) return pf_internal_set_err("pf_render_smooth: blend radius k must be > 0");
    Grid g;
    if (render_grid(ctx, n, pts, psi, rmax, k, g, stream)) return -1;
    double *cam = nullptr;
    if (upload_cam(cam_host, &cam, st)) return -1;
    dim3 blk(16, 8), grd((width + 15) / 16, (height + 7) / 8);
    pf_internal_launches_add(1);
    k_smooth<<<grd, blk, 0, st>>>(g, psi, width, height, cam, k, rmax, g.reach, eps, raw_t, hit_t, normal);
    RCK(cudaGetLastError());
    RCK(cudaFreeAsync(cam, st));
    RCK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int pf_smooth_sdf(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax, double k,
                             int64_t m, const double *xq, double *out, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!(k > 0.0)) return pf_internal_set_err("pf_smooth_sdf: blend radius k must be > 0");
    Grid g;
    if (render_grid(ctx, n, pts, psi, rmax, k, g, stream)) return -1;
    if (m > 0) {
        pf_internal_launches_add(1);
        k_sdf_points<<<(int)((m + 255) / 256 < 4096 ? (m + 255) / 256 : 4096), 256, 0, st>>>(g, psi, m, xq, k, rmax,
                                                                                        g.reach, out);
        RCK(cudaGetLastError());
    }
    RCK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int pf_sample_surface(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax,
                                 int64_t m, const int64_t *cell, const int64_t *max_tries, uint64_t seed,
                                 double *x, double *normal, int32_t *status, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Grid g;
    if (render_grid(ctx, n, pts, psi, rmax, 0.0, g, stream)) return -1;
    const double *dp = nullptr;
    int dnf = 0;
    double tol = 0.0;
    if (pf_internal_domain_view(ctx, &dp, &dnf, &tol)) return -1;
    if (m > 0) {
        pf_internal_launches_add(1);
        k_sample<<<(int)((m + 127) / 128 < 8192 ? (m + 127) / 128 : 8192), 128, 0, st>>>(
            g, pts, psi, m, cell, max_tries, dp, dnf, seed, x, normal, status);
        RCK(cudaGetLastError());
    }
    RCK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int pf_traverse(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double psimax, int smf,
                           const int32_t *cell_nf, const double *planes, const int32_t *tags, int64_t m,
                           const double *rays, int mode, int max_seg, int32_t *out_cell, double *out_t0,
                           double *out_t1, uint8_t *out_fluid, int32_t *count, int32_t *status, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return pf_internal_set_err("pf_traverse: empty scene");
    if (smf <= 0 || max_seg <= 0) return pf_internal_set_err("pf_traverse: bad strides");
    Grid g;
    if (render_grid(ctx, n, pts, psi, 0.0, 0.0, g, stream)) return -1;
    const double *dp = nullptr;
    int dnf = 0;
    double tol = 0.0;
    if (pf_internal_domain_view(ctx, &dp, &dnf, &tol)) return -1;
    if (m > 0) {
        pf_internal_launches_add(1);
        k_traverse<<<(int)((m + 127) / 128 < 8192 ? (m + 127) / 128 : 8192), 128, 0, st>>>(
            g, psi, psimax, dp, dnf, smf, cell_nf, planes, tags, m, rays, mode, max_seg, 8 * n + 8, out_cell, out_t0,
            out_t1, out_fluid, count, status);
        RCK(cudaGetLastError());
    }
    RCK(cudaStreamSynchronize(st));
    return 0;
}
