// ehmg_stencil3d.cuh -- bandwidth-tuned 3D operator/residual kernel
// (placeholder until the tiled kernel lands; the generic rows serve).
#pragma once
#include "ehmg_core.cuh"
namespace ehmg {
inline bool stencil3d_supported(const Geo&) { return false; }
inline void launch_stencil3d(const Geo&, const OpPar&, const Cell*, const cplx*, const cplx*, cplx*,
                             cudaStream_t) {}
}  // namespace ehmg
