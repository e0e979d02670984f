// swarm_inst.hpp -- the launchers of the fused kernel's instantiations, one
// explicit instantiation each, spread over swarm_inst_*.cu so they compile in
// parallel (swarm_kernel.cu dispatches to them).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

#include "swarm_kernel.cuh"

namespace sepso {
template <class T, bool PATH, bool RING, int MAXT, bool SERVER, bool FAST>
int launch_inst(const SwarmParams& p, const ParamPayload* pl, int problem, cudaStream_t st, size_t* smem_out);
}  // namespace sepso
