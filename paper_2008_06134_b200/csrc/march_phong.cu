// K2 instantiations for shading mode "phong" (see sbrc_common.cuh).
#include "sbrc_common.cuh"

void sbrc_march_phong(const sbrc_render_params& p, cudaStream_t s) { launch_march_lookup<SBRC_SHADE_PHONG>(p, s); }
