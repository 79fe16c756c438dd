// pf_warp.cuh -- the handful of warp-collective primitives the cell kernel
// uses.  On the device they are the sm_100a intrinsics.  The cell algorithm
// (pf_cell.cuh) only ever calls these with all 32 lanes converged, which is
// what lets tests/emu compile the same algorithm for a lock-step host warp
// emulator (test infrastructure, never shipped) by providing its own versions
// of exactly these functions.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__) && !defined(PF_EMU)
#define PF_DEV __device__ __forceinline__
#define PF_DEVNI static __device__ __noinline__
// out-of-line device function: one copy of the code however many call sites
// (the cell kernel is instruction-cache bound)
#define PF_NOINL static __device__ __noinline__
#define PF_FULL 0xffffffffu
namespace pfw {
PF_DEV int lane() { return threadIdx.x & 31; }
PF_DEV unsigned ballot(bool p) { return __ballot_sync(PF_FULL, p); }
PF_DEV bool any(bool p) { return __any_sync(PF_FULL, p); }
PF_DEV void sync() { __syncwarp(); }
PF_DEV int shfl(int v, int src) { return __shfl_sync(PF_FULL, v, src); }
PF_DEV double shfl(double v, int src) { return __shfl_sync(PF_FULL, v, src); }
PF_DEV int shfl_xor(int v, int m) { return __shfl_xor_sync(PF_FULL, v, m); }
PF_DEV double shfl_xor(double v, int m) { return __shfl_xor_sync(PF_FULL, v, m); }
PF_DEV int popc(unsigned m) { return __popc(m); }
PF_DEV int atom_add(int *p, int v) { return atomicAdd(p, v); }
// increment a byte counter in shared memory (word-aligned atomic on its word)
PF_DEV int atom_add_u8(uint8_t *p) {
    unsigned *w = (unsigned *)((uintptr_t)p & ~(uintptr_t)3);
    unsigned sh = ((unsigned)((uintptr_t)p & 3)) * 8;
    unsigned old = atomicAdd(w, 1u << sh);
    return (old >> sh) & 0xff;
}
PF_DEV unsigned lanemask_lt() { return (1u << lane()) - 1u; }
PF_DEV int msb(unsigned m) { return 31 - __clz(m); }
PF_DEV unsigned match_any(int key) { return __match_any_sync(PF_FULL, key); }
}  // namespace pfw
PF_DEV int __builtin_ctz_pf(unsigned m) { return __ffs(m) - 1; }
#else
#ifndef PF_EMU
#error "pf_warp.cuh: host compilation requires the test emulator (define PF_EMU)"
#endif
// provided by tests/emu/emu_warp.h
#endif

// the warp reductions inline (PF_WARP_INL=0: one out-of-line copy each;
// inline measured faster: C4 evaluation 36.6 -> 34.1 ms)
#ifndef PF_WARP_INL
#define PF_WARP_INL 1
#endif
#if PF_WARP_INL
#define PF_WRED PF_DEV
#else
#define PF_WRED PF_NOINL
#endif
namespace pfw {
// exact (order-independent) warp reductions
PF_WRED double max_d(double v) {
    for (int m = 16; m > 0; m >>= 1) {
        double o = shfl_xor(v, m);
        v = o > v ? o : v;
    }
    return v;
}
PF_WRED double sum_d(double v) {
    for (int m = 16; m > 0; m >>= 1) v += shfl_xor(v, m);
    return v;
}
PF_WRED int sum_i(int v) {
    for (int m = 16; m > 0; m >>= 1) v += shfl_xor(v, m);
    return v;
}
PF_DEV int max_i(int v) {
    for (int m = 16; m > 0; m >>= 1) {
        int o = shfl_xor(v, m);
        v = o > v ? o : v;
    }
    return v;
}
// inclusive sum over lanes [first, lane] (first = start of this lane's run of
// a segmented reduction); fixed shuffle tree, so the result is deterministic
PF_WRED double seg_sum_d(double v, int first) {
    for (int o = 1; o < 32; o <<= 1) {
        double y = shfl(v, (lane() - o) & 31);
        if (lane() - o >= first) v += y;
    }
    return v;
}
// exclusive prefix over lanes of an int (inline copy for the clip loop,
// given the caller's lane index)
PF_DEV int excl_scan_inl(int v, int L, int *total) {
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = shfl(x, (L - o) & 31);
        if (L >= o) x += y;
    }
    *total = shfl(x, 31);
    return x - v;
}
PF_DEV double max_d_inl(double v) {
    for (int m = 16; m > 0; m >>= 1) {
        double o = shfl_xor(v, m);
        v = o > v ? o : v;
    }
    return v;
}
// exclusive prefix over lanes of an int
PF_WRED int excl_scan_i(int v, int *total) {
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = shfl(x, (lane() - o) & 31);
        if (lane() >= o) x += y;
    }
    *total = shfl(x, 31);
    return x - v;
}
}  // namespace pfw
