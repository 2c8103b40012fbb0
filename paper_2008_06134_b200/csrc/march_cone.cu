// K2 instantiations for shading mode "cone" (see sbrc_common.cuh).
#include "sbrc_common.cuh"

void sbrc_march_cone(const sbrc_render_params& p, cudaStream_t s) { launch_march_lookup<SBRC_SHADE_CONE>(p, s); }
