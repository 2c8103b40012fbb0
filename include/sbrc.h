/*
 * sbrc.h — C ABI of the B200 slice-based ray-casting hot path.
 *
 * Two entry points replace the two numpy functions of the reference
 * package `slicecast` (arXiv 2008.06134, /root/reference/pkg/src/slicecast):
 *
 *   sbrc_build   <- build_attenuation_buffer(v, tf, cam, spec, compensation_n)
 *                   lightbuffer.py:144-199 (Alg. 1)
 *   sbrc_render  <- render(v, tf, settings, buffer) -> (H, W, 4) float32
 *                   raycaster.py:443-469, with _march_rays :415-440,
 *                   _make_shader :376-412, lookup_light_scalar_many
 *                   lightbuffer.py:256-287, _shell_scalar :239-250,
 *                   _cone_scalar :266-300.
 *
 * Conventions
 *  - Every pointer inside a params struct is a DEVICE pointer; the structs
 *    themselves live in host memory and are copied into the kernel launch.
 *  - The library allocates nothing persistent, keeps no global mutable
 *    state, never synchronises, and enqueues on `stream` (a cudaStream_t,
 *    NULL = legacy default stream). Calls on distinct streams are safe to
 *    issue concurrently (the reference functions are reentrant, raycaster.py:447).
 *  - Return value: SBRC_OK (0) or a negative sbrc_status. Parameters are
 *    validated before launch; launch errors are reported as SBRC_ECUDA.
 *    The Python shim maps EINVAL -> ValueError, ECONFIG -> ConfigError,
 *    ECUDA -> RuntimeError (the reference's exception types).
 *  - Setup quantities are float64 exactly as the reference computes them
 *    (numpy float64); decisions (cube coverage, ray entry/exit, sample
 *    count, early termination) are evaluated in float64 with the numpy
 *    operation order and no FMA contraction, so they match bit for bit.
 */
#ifndef SBRC_H
#define SBRC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBRC_ABI_VERSION 12
#define SBRC_MAX_SHELLS 8   /* ShellKernel radii (raycaster.py:92-109) */
#define SBRC_MAX_ANGLES 16  /* ConeKernel angles (raycaster.py:113-124) */
#define SBRC_LUT_SIZE 256   /* transfer.py:16 */
#define SBRC_MAX_PEERS 8    /* GPUs of one node (image assembly over peer memory) */
#define SBRC_MAX_CLIP 4     /* consumer clip half-spaces of a frustum-culled build */

typedef enum sbrc_status {
  SBRC_OK = 0,
  SBRC_EINVAL = -1,      /* bad parameter (ValueError in the reference)        */
  SBRC_ECONFIG = -2,     /* buffer mode without a buffer (ConfigError, raycaster.py:450) */
  SBRC_ECUDA = -3,       /* CUDA launch / runtime error                        */
  SBRC_EUNSUPPORTED = -4 /* shading mode outside SBRC_SHADE_NONE..SBRC_SHADE_EXTINCTION */
} sbrc_status;

typedef enum sbrc_voxel_type {
  SBRC_VOXEL_F32 = 0, /* already-normalised float32 (volume.py:147-149)          */
  SBRC_VOXEL_U8 = 1,  /* raw u8, normalised at fetch as (float)x / 255.0f (volume.py:143-144) */
  SBRC_VOXEL_U16 = 2  /* raw u16, normalised at fetch as (float)x / 65535.0f (volume.py:145-146) */
} sbrc_voxel_type;

typedef enum sbrc_shading {
  SBRC_SHADE_NONE = 0,   /* "none"        raycaster.py:383-384 */
  SBRC_SHADE_SHADOW = 1, /* "sbrc_shadow" raycaster.py:398-401 */
  SBRC_SHADE_SHELL = 2,  /* "shell"       raycaster.py:402-406 */
  SBRC_SHADE_CONE = 3,   /* "cone"        raycaster.py:407-411 */
  SBRC_SHADE_PHONG = 4,  /* "phong"       raycaster.py:204-228, :385-388 (no buffer) */
  SBRC_SHADE_EXTINCTION = 5 /* "extinction" raycaster.py:312-332, :389-394 (no buffer) */
} sbrc_shading;

typedef enum sbrc_lookup {
  SBRC_LOOKUP_LINEAR = 0, /* lightbuffer.py:277-285 */
  SBRC_LOOKUP_NEAREST = 1 /* lightbuffer.py:274-276 */
} sbrc_lookup;

/* VolumeDataset (volume.py:61-122): voxel (x,y,z) at x + nx*(y + ny*z). */
typedef struct sbrc_volume {
  const void* data;   /* device, nx*ny*nz voxels of voxel_type        */
  int32_t nx, ny, nz;
  int32_t voxel_type; /* sbrc_voxel_type                               */
  double box_lo[3];   /* VolumeDataset.box_lo                          */
  double box_ext[3];  /* box_hi - box_lo, as numpy computes it         */
} sbrc_volume;

/* LightCamera (lightbuffer.py:37-86) + SliceStackSpec (slicing.py:22-33). */
typedef struct sbrc_light_frame {
  int32_t width, height;  /* LightCamera.resolution (W, H)             */
  int32_t n_slices;       /* SliceStackSpec.n_slices                    */
  int32_t _pad;
  double axis_u[3], axis_v[3];
  double light_dir[3];    /* SliceStackSpec.light_dir (normalised)      */
  double u_range[2], v_range[2];
  double d_min, d_max;
  const double* plane_offsets; /* device, n_slices float64 (build only) */
} sbrc_light_frame;

/* Texel quads. The attenuation stack I (n, H, W) (AttenuationBuffer.intensity,
 * lightbuffer.py:114-115) is stored lookup-ready: the float4 at (k, y, x) is
 *   ( I[k][y][x], I[k+][y][x], I[k][y][x+], I[k+][y][x+] ),
 *   k+ = min(k+1, n-1), x+ = min(x+1, W-1),
 * so the two-layer bilinear lookup of lookup_light_scalar_many
 * (lightbuffer.py:238-287) is two 16-byte loads (rows y and y+1) instead of
 * eight scalar gathers. I(k, y, x) is component 0 of quad (k, y, x). */

typedef struct sbrc_build_params {
  sbrc_volume volume;
  sbrc_light_frame light;
  const double* alpha_lut; /* device, 256 float64 = tf.resolve(spec.spacing)[:, 3] */
  double compensation_n;   /* lightbuffer.py:193-196                    */
  int32_t row_begin;       /* light-plane rows [row_begin, row_end) are built; */
  int32_t row_end;         /* full build: 0, height (row-sharded build otherwise) */
  /* output: texel quads (format above) of rows [row_begin, row_end);
   * quad (k, y, x) at quads[4*((y-row_begin)*quad_row_stride + k*quad_layer_stride + x)] */
  float* quads;
  int64_t quad_layer_stride;  /* in float4 units; (n, H, W) layout: H*W, [H][n][W]: W   */
  int64_t quad_row_stride;    /* in float4 units; (n, H, W) layout: W,   [H][n][W]: n*W */
  /* Sparse output. write_sparse = 0: every quad is written. 1: for each
   * texel only the quads of layers a march can read are written — the
   * layers whose slice plane meets the cube inflated by write_reach along
   * the texel's line (world units: the lateral reach of the consumer's
   * lookups plus the bilinear footprint), widened by write_below layers
   * toward the light and write_above away from it (plus two layers of
   * rounding margin each side). Values written are identical to a full
   * build; the other quads are left untouched. */
  double write_reach;
  int32_t write_below, write_above;
  int32_t write_sparse;
  /* output_plain = 1: write the plain float32 stack I[k][y][x] instead of
   * texel quads (strides then in float units) — the row shards a sharded
   * multi-GPU build exchanges (4x fewer bytes than quads), packed into quads
   * afterwards with sbrc_pack_quads. */
  int32_t output_plain;
  /* Consumer clip (frustum-culled build, write_sparse = 1 only): the march
   * that reads this stack samples only points p with
   * clip[i][0]*p.x + clip[i][1]*p.y + clip[i][2]*p.z + clip[i][3] >= 0 for
   * every i < n_clip (half-spaces already widened by the lookups' lateral
   * reach) — e.g. the two planes through the eye that bound one rank's
   * contiguous image rows. Layers outside the clipped texel line (widened
   * by write_below / write_above) are not written, and the slice recurrence
   * of a warp stops after the last layer any of its texels writes: values
   * written are identical to a full build. */
  int32_t n_clip;
  double clip[SBRC_MAX_CLIP][4];
  /* Stack layout: 0 = texel quads (above); 1 = layer pairs: float2
   * (I[k][y][x], I[k+1][y][x]) per texel at the same (k, y, x) offsets, in
   * float2 units (half the bytes; read by an sbrc_shadow march only). */
  int32_t quad_layout;
} sbrc_build_params;

typedef struct sbrc_render_params {
  sbrc_volume volume;
  const double* lut_rgba;  /* device, 256x4 float64 = tf.resolve(settings.step) */
  int32_t width, height;   /* RenderSettings.viewport (W, H)            */
  int32_t shading;         /* sbrc_shading                              */
  int32_t lookup;          /* sbrc_lookup                               */
  /* Camera.rays (raycaster.py:53-68): host computes the basis with numpy */
  double eye[3], forward[3], right[3], up2[3];
  double tan_half, aspect;
  double step;             /* RenderSettings.step                       */
  double et_alpha;         /* RenderSettings.early_termination_alpha    */
  /* attenuation buffer (buffer modes only) */
  sbrc_light_frame light;
  const float* quads;      /* device texel quads of the attenuation stack */
  int64_t quad_layer_stride, quad_row_stride;  /* float4 units */
  float light_color[3];
  float ambient_floor;
  /* ShellKernel: radii/weights (raycaster.py:91-109) */
  int32_t shell_count;
  int32_t cone_axis_samples;      /* ConeKernel.axis_samples              */
  int32_t cone_angle_count;
  /* Speed hint, results are identical either way: 1 = use the kernel that
   * skips the light factor of samples whose (premultiplied) LUT emission is
   * exactly zero — worth it when the volume holds values in the TF's leading
   * zero-emission run (e.g. empty space at 0); 0 = evaluate every factor. */
  int32_t skip_clear;
  double shell_radius[SBRC_MAX_SHELLS];
  double shell_weight[SBRC_MAX_SHELLS];
  double cone_ring;                /* ConeKernel.ring_radius_per_step     */
  double cone_cos[SBRC_MAX_ANGLES], cone_sin[SBRC_MAX_ANGLES];
  /* image-space partition: rows grouped in bands of band_rows; band b is
   * rendered by rank b % world into rank-local row (b / world)*band_rows + r */
  int32_t band_rows, rank, world;
  int32_t local_rows;              /* set by the library (rank-local row count) */
  /* phong / extinction (settings.light, not the buffer's light) */
  double scene_light_dir[3];       /* Light.direction (normalised)        */
  double phong[4];                 /* PhongParams: ambient, diffuse, specular, shininess */
  double voxel_size[3];            /* VolumeDataset.voxel_size (gradient steps, volume.py:210) */
  float* image;                    /* device, rank-local (rows, W, 4) premultiplied rgba; may be
                                      NULL when n_peers > 0 */
  /* Fused image assembly over peer memory: when n_peers > 0 every finished
   * pixel (px, py) is also stored to peer_images[i][py*W + px] (float4) for
   * i < n_peers — the full raster images of all ranks, mapped into this
   * process (CUDA IPC over NVLink). The caller then needs only a barrier. */
  float* peer_images[SBRC_MAX_PEERS];
  int32_t n_peers;
  /* Optional dispatch order (heavy-first scheduling) over the rank-local
   * tiles of sbrc_render_grid, tile = ty * tiles_x + tx;
   * entry i is the tile dispatched i-th. NULL = natural order. n_tiles must
   * equal the tile count; a table sized for another grid is ignored, and so
   * is tile_steps (natural order, no costs recorded). */
  int32_t n_tiles;
  const int32_t* tile_order;
  unsigned long long* sample_count;/* device counter (+= executed samples), may be NULL */
  /* Optional measured tile costs (n_tiles entries over the sbrc_render_grid
   * tiles, zeroed by the caller; only written when n_tiles equals the
   * launch's tile count, with or without tile_order): each block atomically maxes the executed
   * sample count of its longest ray into tile_steps[tile]. Sorted in
   * decreasing order it is the next frame's heavy-first tile_order. */
  unsigned int* tile_steps;
  /* Contiguous partition (row_count > 0): this rank renders raster rows
   * [row_begin, row_begin + row_count) into rank-local rows 0..row_count-1
   * (band_rows / rank / world are then ignored). Used with a frustum-culled
   * build, whose texels only cover one contiguous screen band. */
  int32_t row_begin, row_count;
  /* K2 kernel choice (speed only, results identical): 0 = by the rank-local
   * image size, 1 = the throughput kernel (4 blocks/SM), 2 = the latency
   * kernel (1 block/SM, more registers per warp; ray groups for tiny images)
   * where one exists for the mode. A rank can measure both for its share
   * (FrameRenderer.choose_march_kernel). */
  int32_t march_kernel;
  /* Layout of `quads` (sbrc_build_params.quad_layout): 1 = layer pairs, for
   * shading == SBRC_SHADE_SHADOW and width >= 2 only (the single-lookup
   * march reads half the bytes; results identical). */
  int32_t quad_layout;
} sbrc_render_params;

/* ABI version of the loaded library (== SBRC_ABI_VERSION). */
int sbrc_abi_version(void);

/* Bounds-check counters of a checked build (compiled with SBRC_CHECKED=1):
 * out-of-extent accesses by kind (volume, quad read, quad/plain write,
 * image, peer image, tile table, LUT index, plane offset); reset != 0 zeroes
 * them. SBRC_EUNSUPPORTED in normal builds. Debugging aid, not on the path. */
int sbrc_debug_violations(unsigned int counts[8], int reset);

/* Human-readable text for a status code (static storage). */
const char* sbrc_strerror(int status);

/* sizeof() of the params structs, so a binding can verify its layout. */
int64_t sbrc_struct_size(int which); /* 0 volume, 1 light_frame, 2 build, 3 render, 4 half_angle */

/* K0: repack a raw voxel stream already on the device (no-op copy for f32;
 * u8/u16 stay raw and are normalised at fetch). Replaces load_raw's
 * normalisation (volume.py:141-151) for the device copy. */
int sbrc_volume_check(const sbrc_volume* v);

/* K0: load_raw's float32 min-max normalisation in place (volume.py:147-151):
 * data[i] = fl32(fl32(data[i] - lo) / range), range = fl32(hi - lo) > 0 —
 * numpy's float32 arithmetic, so bit-identical. */
int sbrc_normalize_f32(float* data, int64_t n, float lo, float range, void* stream);

/* K0: widen a raw u8/u16 voxel stream (n voxels, voxel_type SBRC_VOXEL_U8 /
 * U16) to float32 with load_raw's normalisation (volume.py:143-146: IEEE
 * float32 division by 255 / 65535, bit-identical to numpy). */
int sbrc_widen_volume(const void* src, int voxel_type, int64_t n, float* dst, void* stream);

/* Volume layout the kernels of this library read: 0 = linear (nz, ny, nx),
 * 1 = 8^3-cell bricks with a one-voxel apron (an A/B build, SBRC_BRICK=1);
 * sbrc_volume.data must then point at sbrc_brick_pack's output, of
 * sbrc_brick_elems(nx, ny, nz) voxels. */
int sbrc_volume_layout(void);
int64_t sbrc_brick_elems(int nx, int ny, int nz);
int sbrc_brick_pack(const void* src, int voxel_type, int nx, int ny, int nz, void* dst, void* stream);

/* Heavy-first dispatch table from measured tile costs (schedule.TileFeedback):
 * order[0..n) = tile indices by decreasing steps[i], ties by increasing index
 * (deterministic). Device pointers; replaces a stable descending argsort. */
int sbrc_tile_order(const unsigned int* steps, int n, int* order, void* stream);

/* Image assembly of the NCCL path: dst row y (width float4 pixels) = src row
 * perm[y], y < rows (device pointers; perm int64). */
int sbrc_permute_rows(const float* src, const int64_t* perm, float* dst, int rows, int width, void* stream);

/* K1: attenuation build (lightbuffer.py:144-199). */
int sbrc_build(const sbrc_build_params* p, void* stream);

/* K2: ray march (raycaster.py:443-469). Writes the rank-local rows. */
int sbrc_render(const sbrc_render_params* p, void* stream);

/* Repack a plain float32 stack I(k, y, x) = plain[k*plain_layer_stride + y*plain_row_stride + x]
 * (e.g. a host-built reference AttenuationBuffer.intensity uploaded as is) into texel quads. */
int sbrc_pack_quads(const float* plain, int64_t plain_layer_stride, int64_t plain_row_stride,
                    int n, int height, int width, float* quads, int64_t quad_layer_stride,
                    int64_t quad_row_stride, void* stream);

/* Light factor at m float64 world points pts[3*i..] for shading sbrc_shadow /
 * shell / cone (p->shading, p->lookup, kernels, light frame, quads, light
 * colour, ambient floor; the image/volume fields are ignored): out[4*i..] =
 * (scalar, factor_r, factor_g, factor_b) = lookup_light_scalar_many /
 * _shell_scalar / _cone_scalar (lightbuffer.py:256-287, raycaster.py:239-300)
 * followed by _factor_from_intensity (raycaster.py:197-201). eye (3 doubles)
 * orients the cone ring (shade_cone's eye); NULL = the plane_basis fallback. */
int sbrc_light_factor(const sbrc_render_params* p, const double* pts, int64_t m, const double* eye, float* out,
                      void* stream);

/* GPU shadow_oracle_many (raycaster.py:335-366): transmittance from each of
 * m float64 points pts[3*i..] toward the light, a straight march with
 * step-corrected opacity: out[i] = prod (1 - min(a, 1 - 1e-6)).
 * alpha_lut = tf.resolve(oracle_step)[:, 3]; to_light = -light.direction. */
int sbrc_shadow_oracle(const sbrc_volume* v, const double* alpha_lut, const double* pts, int64_t m,
                       const double* to_light, double step, double* out, void* stream);

/* Half-angle slicing baseline (halfangle.py:48-142): n slices perpendicular
 * to the half vector; per slice an eye pass (composite into the float64
 * accumulation image, modulated by the running light transmittance) and a
 * light pass (attenuate it). pass_count = 2n. The host computes the
 * per-frame scalars with numpy exactly as the reference does. */
typedef struct sbrc_half_angle_params {
  sbrc_volume volume;
  const double* lut;          /* device 256x4 float64: the raw TransferFunction.lut */
  const double* plane_offsets;/* device n float64: make_slice_stack(half, n).plane_offsets */
  int32_t width, height;      /* viewport */
  int32_t light_width, light_height;
  int32_t n_slices;
  int32_t front_to_back;      /* 1: "front_to_back", 0: "back_to_front" (_half_vector) */
  double eye[3], forward[3], right[3], up2[3];
  double tan_half, aspect;
  double half[3];             /* half vector */
  double delta;               /* stack.spacing */
  double light_dir[3], axis_u[3], axis_v[3];
  double u_range[2], v_range[2];
  double hl, h_dot_u, h_dot_v, h_dot_e;
  double* eye_accum;          /* device scratch H*W*4 float64 */
  double* light_accum;        /* device scratch Hl*Wl float64 */
  float* image;               /* device out (H, W, 4) float32 */
} sbrc_half_angle_params;

/* Runs the 2n passes on `stream`; *pass_count = 2n. first_slice/last_slice
 * allow running a prefix (light_trace support): passes for k in [first, last). */
int sbrc_half_angle(const sbrc_half_angle_params* p, int first_slice, int last_slice, int init, int finish,
                    int* pass_count, void* stream);

/* Peer-memory plumbing for the fused image assembly (one process per GPU):
 * an IPC-capable allocation, its 64-byte handle, and mapping a peer's handle
 * into this process with lazy peer access (NVLink). These are the only
 * entry points that allocate or map memory. */
int sbrc_ipc_alloc(int64_t bytes, void** ptr);
int sbrc_ipc_free(void* ptr);
int sbrc_ipc_handle(void* ptr, unsigned char handle[64]);
int sbrc_ipc_open(const unsigned char handle[64], void** ptr);
int sbrc_ipc_close(void* ptr);

/* Device address of page-locked host memory (cudaPointerGetAttributes):
 * *dev = the pointer K2 may store to (image = *dev writes the frame straight
 * into host memory over PCIe while the march runs). SBRC_EINVAL if `host`
 * is not page-locked, mapped host memory. */
int sbrc_host_device_pointer(const void* host, void** dev);

/* Block grid of the throughput K2 kernels for (width, height, band_rows,
 * rank, world): grid[0..3] = tiles_x, tiles_y, tile width and height in
 * pixels. Latency mode and ray groups change the grid: build tile_order
 * tables from sbrc_render_grid. */
int sbrc_march_grid(int width, int height, int band_rows, int rank, int world, int grid[4]);

/* The tile grid sbrc_render will launch for *p (block shape, latency mode,
 * and ray groups depend on the params): grid[0..3] =
 * tiles_x, tiles_y, tile width and height in pixels. tile_order tables must
 * index this grid. */
int sbrc_render_grid(const sbrc_render_params* p, int grid[4]);


/* Number of rank-local image rows sbrc_render writes for (height, band_rows, rank, world). */
int sbrc_local_rows(int height, int band_rows, int rank, int world);

#ifdef __cplusplus
}
#endif

#endif /* SBRC_H */
