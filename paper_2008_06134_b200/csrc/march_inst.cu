// K2 instantiations for one (shading mode, voxel type), chosen with
// -DSBRC_INST_SHADE=<sbrc_shading> -DSBRC_INST_VT=<sbrc_voxel_type>: build.py
// compiles this file once per pair, in parallel (see sbrc_common.cuh).
#include "sbrc_common.cuh"

#if !defined(SBRC_INST_SHADE) || !defined(SBRC_INST_VT)
#error "compile with -DSBRC_INST_SHADE=<sbrc_shading> -DSBRC_INST_VT=<sbrc_voxel_type> (build.py)"
#endif

void SBRC_MARCH_FN(SBRC_INST_SHADE, SBRC_INST_VT)(const sbrc_render_params& p, cudaStream_t s) {
  launch_march_lookup<SBRC_INST_SHADE, SBRC_INST_VT>(p, s);
}

int SBRC_MARCH_VIOL(SBRC_INST_SHADE, SBRC_INST_VT)(unsigned int* acc, int reset) { return tu_violations(acc, reset); }
