// pf_render.cu -- first-hit rendering of the fluid surface (SPEC.md:406-463,
// PAPER.md:392-436), thread per pixel.
//
// The fluid is the union of the restricted cells, i.e. the set of points
// whose power-nearest site's ball contains them -- the union of the balls
// B(p_i, sqrt(psi_i)).  The first point of that union along a ray lies on the
// sphere of the ball it enters first, and that point belongs to the ball's
// Laguerre cell (every other site has power distance >= 0 there), so the
// SPEC's first_hit ("nearest ray-sphere hit inside the owning cell") is the
// smallest entry parameter over the balls.  The ray walks the bucket grid
// (3D DDA over the bucket-sorted SoA of pf_grid_build); in each bucket it
// tests the sites of the buckets within the largest ball radius, and stops
// once the best hit lies before the bucket's exit.
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
    const double *sx, *sy, *sz;
    const int *sid, *bstart;
    int gn[3];
    double lo[3], h[3];
    int reach;  // buckets within the largest ball radius
};

// smallest t >= tmin with the ray entering a ball of the sites in bucket b
__device__ void test_bucket(const Grid &g, int bx, int by, int bz, const double *o, const double *d,
                            const double *__restrict__ psi, double tmin, double &best, int &who) {
    if (bx < 0 || by < 0 || bz < 0 || bx >= g.gn[0] || by >= g.gn[1] || bz >= g.gn[2]) return;
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

__global__ void k_first_hit(Grid g, const double *__restrict__ psi, int w, int h, const double *cam,
                            int *__restrict__ hit_id, double *__restrict__ hit_t) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y * blockDim.y + threadIdx.y;
    if (px >= w || py >= h) return;
    // cam: eye[3], forward[3], right[3], up[3], tan(fov/2), aspect
    const double sx = (2.0 * (px + 0.5) / w - 1.0) * cam[12] * cam[13];
    const double sy = (1.0 - 2.0 * (py + 0.5) / h) * cam[12];
    double d[3];
    for (int a = 0; a < 3; a++) d[a] = cam[3 + a] + sx * cam[6 + a] + sy * cam[9 + a];
    const double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int a = 0; a < 3; a++) d[a] /= dn;
    const double o[3] = {cam[0], cam[1], cam[2]};
    // clip the ray to the grid box
    double t0 = 0.0, t1 = 1e300;
    for (int a = 0; a < 3; a++) {
        const double lo = g.lo[a], hi = g.lo[a] + g.gn[a] * g.h[a];
        if (fabs(d[a]) < 1e-300) {
            if (o[a] < lo || o[a] > hi) { t1 = -1.0; break; }
            continue;
        }
        double ta = (lo - o[a]) / d[a], tb = (hi - o[a]) / d[a];
        if (ta > tb) { const double tt = ta; ta = tb; tb = tt; }
        t0 = fmax(t0, ta);
        t1 = fmin(t1, tb);
    }
    double best = 1e300;
    int who = -1;
    if (t0 <= t1) {
        // 3D DDA over the buckets the ray crosses
        int b[3], step[3];
        double tnext[3], tdel[3];
        for (int a = 0; a < 3; a++) {
            const double p = o[a] + t0 * d[a];
            int c = (int)floor((p - g.lo[a]) / g.h[a]);
            b[a] = c < 0 ? 0 : (c >= g.gn[a] ? g.gn[a] - 1 : c);
            if (d[a] > 0.0) {
                step[a] = 1;
                tnext[a] = (g.lo[a] + (b[a] + 1) * g.h[a] - o[a]) / d[a];
                tdel[a] = g.h[a] / d[a];
            } else if (d[a] < 0.0) {
                step[a] = -1;
                tnext[a] = (g.lo[a] + b[a] * g.h[a] - o[a]) / d[a];
                tdel[a] = -g.h[a] / d[a];
            } else {
                step[a] = 0;
                tnext[a] = 1e300;
                tdel[a] = 1e300;
            }
        }
        const int R = g.reach;
        for (int guard = 0; guard < 4 * (g.gn[0] + g.gn[1] + g.gn[2]) + 8; guard++) {
            for (int i = -R; i <= R; i++)
                for (int j = -R; j <= R; j++)
                    for (int k = -R; k <= R; k++) test_bucket(g, b[0] + i, b[1] + j, b[2] + k, o, d, psi, t0, best, who);
            const double texit = fmin(tnext[0], fmin(tnext[1], tnext[2]));
            if (best <= texit || texit > t1) break;
            const int a = tnext[0] <= tnext[1] ? (tnext[0] <= tnext[2] ? 0 : 2) : (tnext[1] <= tnext[2] ? 1 : 2);
            b[a] += step[a];
            if (b[a] < 0 || b[a] >= g.gn[a]) break;
            tnext[a] += tdel[a];
        }
    }
    hit_id[py * w + px] = who;
    hit_t[py * w + px] = who >= 0 ? best : -1.0;
}

}  // namespace

// defined in pf_runtime.cu
int pf_internal_grid_view(pf_ctx *c, const double **sx, const double **sy, const double **sz, const int **sid,
                          const int **bstart, int *gn, double *lo, double *h);

extern "C" int pf_render_first_hit(pf_ctx *ctx, int64_t n, const double *pts, const double *psi, double rmax,
                                   const double *cam_host, int width, int height, int32_t *hit_id,
                                   double *hit_t, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (pf_grid_build(ctx, n, pts, psi, 0.0, stream)) return -1;
    Grid g;
    if (pf_internal_grid_view(ctx, &g.sx, &g.sy, &g.sz, &g.sid, &g.bstart, g.gn, g.lo, g.h)) return -1;
    const double hmin = fmin(g.h[0], fmin(g.h[1], g.h[2]));
    g.reach = (int)ceil(rmax / hmin);
    if (g.reach > 8) g.reach = 8;
    double *cam = nullptr;
    RCK(cudaMallocAsync((void **)&cam, 14 * sizeof(double), st));
    RCK(cudaMemcpyAsync(cam, cam_host, 14 * sizeof(double), cudaMemcpyHostToDevice, st));
    dim3 blk(16, 8), grd((width + 15) / 16, (height + 7) / 8);
    pf_internal_launches_add(1);
    k_first_hit<<<grd, blk, 0, st>>>(g, psi, width, height, cam, hit_id, hit_t);
    RCK(cudaGetLastError());
    RCK(cudaFreeAsync(cam, st));
    RCK(cudaStreamSynchronize(st));
    return 0;
}
