// pf_tiers.cuh -- the two capacity instantiations of the cell kernel.
//
//   Fast : shared-memory workspace sized for the cells seen on the paper's
//          scenes (ball-aware maxima measured on dense blocks: nv 38, nf 21,
//          nl 114).  A cell that exceeds any capacity is
//          queued, untouched, for the exact tier.
//   Exact: the reference's own capacities (_kernels.py:24-27) in a
//          global-memory workspace; overflow here reproduces the reference's
//          CLIP_OVERFLOW / FLAG_OVERFLOW outcome.
#pragma once
#include "pf_cell.cuh"

namespace pf {
//                 CV   CF   CL   CC    CE    CP   EXACT
using FastCaps = Caps<64, 32, 192, 64, 64, 120, false>;
using ExactCaps = Caps<REF_MAX_V, REF_MAX_F, REF_MAX_L, 1024, REF_MAX_L, 4096, true>;
}  // namespace pf
