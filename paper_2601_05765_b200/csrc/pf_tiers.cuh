// pf_tiers.cuh -- the three capacity instantiations of the cell kernel.
//
//   Fast : shared-memory workspace sized for the cells seen on the paper's
//          scenes (ball-aware maxima measured on dense blocks: nv 38, nf 21,
//          nl 114): 48 vertices, 32 facets, 160 loop
//          entries, 40 candidates per distance shell, 48 crossing entries --
//          9.6 KB of shared memory per build warp, i.e. 24 warps per SM in
//          blocks of 8 (measured on C4: 116 ms at 16 warps with the 64 / 192 /
//          64 capacities, 108 ms at 20, 105 ms at 24).  A cell that exceeds
//          any capacity is queued, untouched, for the exact tier.
//   Mid  : 128 V / 64 F / 448 entries / 64 candidates / 512 pool points in
//          shared memory for the fast tier's overflow; its own overflow goes on.
//   Exact: the reference's own capacities (_kernels.py:24-27) in a
//          global-memory workspace; overflow here reproduces the reference's
//          CLIP_OVERFLOW / FLAG_OVERFLOW outcome.
#pragma once
#include "pf_cell.cuh"

namespace pf {
//                 CV   CF   CL   CC    CE    CP   EXACT
#ifndef PF_FCV
#define PF_FCV 48
#endif
#ifndef PF_FCL
#define PF_FCL 160
#endif
#ifndef PF_FCC
#define PF_FCC 40
#endif
#ifndef PF_FCE
#define PF_FCE 48
#endif
#ifndef PF_FCP
#define PF_FCP 120
#endif
using FastCaps = Caps<PF_FCV, 32, PF_FCL, PF_FCC, PF_FCE, PF_FCP, false>;
// Mid: the fast tier's overflow (mostly the boundary-point pool of cells whose
// sphere meets many facets) in shared memory, 4 warps (48 KB each) per SM.
using MidCaps = Caps<128, 64, 448, 64, 128, 512, false>;
#if PF_FCV == 48 && PF_FCL == 160 && PF_FCC == 40 && PF_FCE == 48
static_assert(sizeof(BWS<FastCaps>) == 9600, "fast build workspace must stay 9600 B: 3 blocks of 8 warps per SM");
#endif
using ExactCaps = Caps<REF_MAX_V, REF_MAX_F, REF_MAX_L, 1024, REF_MAX_L, 4096, true>;
}  // namespace pf
