// K2 instantiations for shading mode "none" (see sbrc_common.cuh).
#include "sbrc_common.cuh"

void sbrc_march_none(const sbrc_render_params& p, cudaStream_t s) { launch_march_lookup<SBRC_SHADE_NONE>(p, s); }
