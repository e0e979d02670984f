// swarm_inst_latency.cu -- instantiations of the fused kernel (see swarm_inst.hpp).
#include "swarm_kernel_body.cuh"
#include "swarm_inst.hpp"

namespace sepso {
template <class T, bool PATH, bool RING, int MAXT, bool SERVER, bool FAST>
int launch_inst(const SwarmParams& p, const ParamPayload* pl, int problem, cudaStream_t st, size_t* smem_out) {
    return launch_t<T, PATH, RING, MAXT, SERVER, FAST>(p, pl, problem, st, smem_out);
}
template int launch_inst<float, true, false, 896, false, true>(const SwarmParams&, const ParamPayload*, int, cudaStream_t, size_t*);
template int launch_inst<float, true, false, 896, true, true>(const SwarmParams&, const ParamPayload*, int, cudaStream_t, size_t*);
template int launch_inst<float, true, false, 1024, true, false>(const SwarmParams&, const ParamPayload*, int, cudaStream_t, size_t*);
}  // namespace sepso
