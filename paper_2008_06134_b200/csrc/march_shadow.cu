// K2 instantiations for shading mode "shadow" (see sbrc_common.cuh).
#include "sbrc_common.cuh"

void sbrc_march_shadow(const sbrc_render_params& p, cudaStream_t s) { launch_march_lookup<SBRC_SHADE_SHADOW>(p, s); }
