// emu_warp.h -- TEST INFRASTRUCTURE ONLY.  A lock-step host emulation of one
// 32-lane warp, used to run the exact device algorithm of pf_cell.cuh on the
// CPU so the warp-cooperative logic can be checked against the oracle without
// a GPU.  Each lane is a fiber; every collective (ballot / shfl / syncwarp) is
// a rendezvous of all 32 lanes.  The scheduler verifies that all lanes reach
// the same collective (the device code must be warp-convergent at every
// collective) and resumes lanes in a shuffled order each epoch so that a
// missing __syncwarp between a shared-memory write and a cross-lane read
// shows up as a result that depends on the order.
#pragma once
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>

#define PF_DEV static inline
#define PF_DEVNI static
#define PF_NOINL static
static inline int __builtin_ctz_pf(unsigned m) { return __builtin_ctz(m); }
static inline double rsqrt(double x) { return 1.0 / std::sqrt(x); }  // device: MUFU-based rsqrt
static inline double __drcp_rn(double x) { return 1.0 / x; }  // device: correctly rounded reciprocal

extern "C" void emu_swap(void **from_sp, void *to_sp);

namespace pfw {

enum { K_NONE = 0, K_BALLOT = 1, K_SHFL = 2, K_SYNC = 3 };

struct EmuWarp {
    void *sched_sp;
    void *lane_sp[32];
    bool done[32];
    int kind[32];
    uint64_t slot[2][32];
    long epoch[32];
    char *stacks;
    size_t stack_size;
    void (*fn)(void *ctx, int lane);
    void *ctx;
    uint64_t rng;
    long n_collectives;
    int error;
};

extern thread_local EmuWarp *g_w;
extern thread_local int g_lane;

static inline void emu_yield() { emu_swap(&g_w->lane_sp[g_lane], g_w->sched_sp); }

static inline uint64_t deposit_and_wait(int kind, uint64_t v) {
    EmuWarp *w = g_w;
    int l = g_lane;
    long e = w->epoch[l];
    w->slot[e & 1][l] = v;
    w->kind[l] = kind;
    emu_yield();
    w->epoch[l] = e + 1;
    return (uint64_t)e;
}

static inline int lane() { return g_lane; }
static inline unsigned ballot(bool p) {
    long e = (long)deposit_and_wait(K_BALLOT, p ? 1 : 0);
    unsigned m = 0;
    for (int l = 0; l < 32; l++)
        if (g_w->slot[e & 1][l]) m |= 1u << l;
    return m;
}
static inline bool any(bool p) { return ballot(p) != 0; }
static inline void sync() { deposit_and_wait(K_SYNC, 0); }
static inline uint64_t shfl_bits(uint64_t v, int src) {
    long e = (long)deposit_and_wait(K_SHFL, v);
    return g_w->slot[e & 1][src & 31];
}
static inline int shfl(int v, int src) {
    return (int)(int64_t)shfl_bits((uint64_t)(int64_t)v, src);
}
static inline double shfl(double v, int src) {
    uint64_t b;
    memcpy(&b, &v, 8);
    b = shfl_bits(b, src);
    double r;
    memcpy(&r, &b, 8);
    return r;
}
static inline int shfl_xor(int v, int m) { return shfl(v, g_lane ^ m); }
static inline double shfl_xor(double v, int m) { return shfl(v, g_lane ^ m); }
static inline int popc(unsigned m) { return __builtin_popcount(m); }
static inline int atom_add(int *p, int v) {
    int o = *p;
    *p += v;
    return o;
}
static inline unsigned lanemask_lt() { return (1u << g_lane) - 1u; }
static inline int msb(unsigned m) { return 31 - __builtin_clz(m); }
static inline unsigned match_any(int key) {
    long e = (long)deposit_and_wait(K_SHFL, (uint64_t)(int64_t)key);
    unsigned m = 0;
    for (int l = 0; l < 32; l++)
        if ((int)(int64_t)g_w->slot[e & 1][l] == key) m |= 1u << l;
    return m;
}
static inline int atom_add_u8(uint8_t *p) { return (*p)++; }

// run fn(ctx, lane) on 32 fibers to completion; returns 0 or an error code
int emu_run_warp(EmuWarp *w, void (*fn)(void *, int), void *ctx, uint64_t seed);
EmuWarp *emu_new_warp(size_t stack_size);
void emu_free_warp(EmuWarp *w);

}  // namespace pfw
