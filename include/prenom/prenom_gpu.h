/* prenom_gpu.h -- C ABI of the B200-native per-object NeRF trainer.
 *
 * This is the drop-in boundary for PRENOM's object-trainer path
 * (reference: /root/reference/proj/core, namespace noma). The reference has no
 * plugin/FFI layer; its trainer surface is a set of public C++ functions plus
 * the anonymous-namespace loop `train_track` (core/src/mapper.cpp:130-197).
 * Every entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - Plain C types, host pointers unless a name says `_dev`. No torch types.
 *  - Every call returns prenom_status. The status classes mirror the reference
 *    exception classes (core/include/noma/errors.hpp:9-24):
 *      UsageError -> PRENOM_USAGE, DataError -> PRENOM_DATA,
 *      NumericError -> PRENOM_NUMERIC; CUDA failures -> PRENOM_CUDA.
 *    The message of the last failure on the calling thread is returned by
 *    prenom_last_error().
 *  - Parameter vectors use the reference layout exactly (field.cpp:48-62):
 *    hash tables [level][2^T rows][F] fp32, then per hidden layer W[out][in]
 *    row-major followed by b[out], then the 4-wide output layer W[4][in], b[4].
 *  - Density grids are vertex-centred R^3 fp32, x-fastest
 *    (core/include/noma/density_grid.hpp:15-35).
 *  - Images are row-major: rgb [H][W][3] fp32, depth [H][W] fp32 (distance
 *    along the ray, 0 = no return), mask [H][W] u8 (instance id, 0 = bg)
 *    (core/include/noma/image.hpp:11-39).
 *  - Threading: a context is bound to one device; an object handle is not
 *    re-entrant; distinct handles may be driven from distinct host threads
 *    (mirrors "one thread per object", mapper.cpp:572-585).
 *
 * Randomness (the one deliberate departure from the reference): the
 * reference consumes a sequential std::mt19937 in data-dependent order
 * (mapper.cpp:143,151; render.cpp:89-99,216; density_grid.cpp:83-94). Here
 * every draw comes from Philox4x32-10 with
 *     key = { (u32)seed, (u32)(seed >> 32) }
 *     ctr = { c0 = draw index, c1 = ray index, c2 = step, c3 = tag }
 * and the tags below. uniform(x) = (x >> 8) * 2^-24 in [0,1);
 * pick(x, n) = (u32)(((u64)x * n) >> 32) in [0,n).
 *   TAG_FRAME  c0=0 c1=0     out[0]            -> keyframe pick
 *   TAG_PIXEL  c0=0 c1=ray   out[0]            -> pixel pick (object list, or band list for bg slots)
 *   TAG_FINE   c0=s/2 c1=ray out[2(s&1)], out[2(s&1)+1] -> bin draw, in-bin draw of fine sample s
 *   TAG_BG     c0=0 c1=ray   out[0..2]         -> background target colour
 *   TAG_RENDER c0=s/2 c1=ray (c2 = render call) -> fine draws for prenom_render
 *   TAG_INIT   c0=i/4 c1=0 c2=0                 -> device-side init_params draws
 *   TAG_SYNTH  c0=pixel c1=view c2=0 out[0..1] -> depth noise (Box-Muller), out[2] -> missing depth
 * The CPU oracle (oracle/prenom_oracle.c) restates the reference math with
 * exactly these draws, which is what makes bit-exact sample parity possible.
 */
#ifndef PRENOM_GPU_H
#define PRENOM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRENOM_ABI_VERSION 1

typedef enum {
  PRENOM_OK = 0,
  PRENOM_USAGE = 1,   /* noma::UsageError  */
  PRENOM_DATA = 2,    /* noma::DataError   */
  PRENOM_NUMERIC = 3, /* noma::NumericError */
  PRENOM_CUDA = 4
} prenom_status;

enum {
  PRENOM_TAG_FRAME = 1,
  PRENOM_TAG_PIXEL = 2,
  PRENOM_TAG_FINE = 3,
  PRENOM_TAG_BG = 4,
  PRENOM_TAG_RENDER = 5,
  PRENOM_TAG_INIT = 6,
  PRENOM_TAG_SYNTH = 7
};

enum { PRENOM_ACT_EXP_CLAMPED = 0, PRENOM_ACT_SOFTPLUS = 1 };
/* MLP arithmetic of the train step:
 *   FP32      fp32 SIMT GEMMs (1e-4 parity path, no tensor cores);
 *   BF16      tcgen05 kind::f16, bf16 operands, fp32 accumulation (1e-2);
 *   BF16X3    tcgen05 kind::f16 on split operands x = hi + lo (both bf16):
 *             hi*hi + hi*lo + lo*hi, fp32 accumulation -- ~16 significand
 *             bits per product, fp32-class results (1e-4) on tensor cores. */
enum { PRENOM_MLP_FP32 = 0, PRENOM_MLP_BF16 = 1, PRENOM_MLP_BF16X3 = 2 };
enum { PRENOM_KIND_OBJECT = 0, PRENOM_KIND_BACKGROUND = 1 };

/* Mirrors noma::FieldArch (core/include/noma/field.hpp:20-31). */
typedef struct {
  int32_t hash_levels;        /* L */
  int32_t features_per_level; /* F */
  int32_t log2_table_size;    /* T */
  int32_t base_resolution;
  float per_level_scale;
  int32_t hidden_width;       /* W */
  int32_t hidden_layers;      /* H */
  int32_t density_activation; /* PRENOM_ACT_* (noma::DensityActivation) */
} prenom_field_arch;

/* Mirrors noma::Camera (core/include/noma/render.hpp:13-23); pose is
 * camera -> world, R row-major (geom.hpp:44-72, 120-131). */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9];
  float t[3];
} prenom_camera;

/* noma::Pose: world_point = R * local_point + t (geom.hpp:120-131). */
typedef struct {
  float R[9];
  float t[3];
} prenom_pose;

/* Hot keys of MapperConfig / InnerOptions / LossWeights
 * (mapper.hpp:80-103, meta.hpp:14-19, render.hpp:93-96; key names as in
 * commands.cpp:216-244). */
typedef struct {
  int32_t rays_per_iter;      /* "rays"            default 128 (mapper) */
  float bg_fraction;          /* "bg_fraction"     0.25 */
  int32_t samples_per_ray;    /* "samples"         n_fine, 24 (mapper) */
  float lambda_d;             /* "lambda_d"        0.1 */
  float lambda_sigma;         /* "lambda_sigma"    1e-4 */
  int32_t coarse_samples;     /* "coarse_samples"  32 */
  float escape_eps;           /* "escape_eps"      1e-4 */
  int32_t grid_refresh_every; /* "grid_refresh_every" m = 50 (0 = never) */
  float eta;                  /* "eta" Adam lr     1e-2 */
  int32_t prior_sampling;     /* "prior_sampling"  1 */
  int32_t band_px;            /* generate_rays band width, 8 */
  int32_t mlp_precision;      /* PRENOM_MLP_* */
  float adam_beta1, adam_beta2, adam_eps; /* AdamState defaults 0.9/0.999/1e-8 */
} prenom_train_cfg;

/* One train step's batch_loss terms (noma::LossResult, render.hpp:98-104)
 * plus bookkeeping. */
typedef struct {
  double total, color_term, depth_term, sigma_term;
  int64_t n_samples;      /* MLP samples evaluated (non-escaped rays x S) */
  int32_t n_rays_escaped; /* rays with no samples */
  int32_t frame_index;    /* keyframe the step drew its rays from */
} prenom_step_stats;

typedef struct prenom_ctx_s* prenom_ctx_t;
typedef struct prenom_object_s* prenom_object_t;

/* ---- errors / meta ---------------------------------------------------- */
const char* prenom_last_error(void);
int prenom_abi_version(void);
void prenom_default_train_cfg(prenom_train_cfg* out);

/* noma::param_count / hash_param_count / level_resolution / vertex_table_row
 * (field.cpp:113-148). Host-side helpers, no device needed. */
prenom_status prenom_param_count(const prenom_field_arch* arch, size_t* total, size_t* hash);
prenom_status prenom_level_resolution(const prenom_field_arch* arch, int level, int* res);

/* ---- context ------------------------------------------------------------ */
/* Per-GPU context: stream, scratch arena. (No reference counterpart: the
 * reference runs on the calling thread.) */
prenom_status prenom_ctx_create(int device, prenom_ctx_t* out);
prenom_status prenom_ctx_destroy(prenom_ctx_t ctx);
/* cudaStream_t of the context, for callers that time with events. */
prenom_status prenom_ctx_stream(prenom_ctx_t ctx, void** stream);
prenom_status prenom_ctx_synchronize(prenom_ctx_t ctx);
/* Number of product kernels launched on this context so far. */
prenom_status prenom_ctx_launch_count(prenom_ctx_t ctx, int64_t* count);

/* Per-kernel device timing with CUDA events recorded on the context stream
 * around every train-step launch (no reference counterpart; measurement
 * only). prenom_ctx_kernel_times synchronizes, returns the summed
 * milliseconds and launch counts per PRENOM_K_* class, and resets them. */
enum {
  PRENOM_K_SAMPLE = 0,     /* k_sample: rays + prior-CDF sampler        */
  PRENOM_K_FIELD_FWD = 1,  /* k_fwd_tile: encode + MLP forward          */
  PRENOM_K_COMPOSITE = 2,  /* k_composite: compositing + loss + bwd     */
  PRENOM_K_MLP_BWD = 3,    /* k_bwd_tile: MLP backward + d_features     */
  PRENOM_K_ENCODE_BWD = 4, /* k_encode_bwd: table-gradient scatter      */
  PRENOM_K_ADAM = 5,       /* k_adam: dense Adam + grad zero            */
  PRENOM_K_REFRESH = 6,    /* k_field_points: density-grid refresh      */
  PRENOM_K_COUNT = 7
};
prenom_status prenom_ctx_profile(prenom_ctx_t ctx, int enable);
prenom_status prenom_ctx_kernel_times(prenom_ctx_t ctx, double* ms, int64_t* launches);

/* ---- object lifecycle ("create object from a category prior") ----------
 * Replaces train_track's CREATE block (mapper.cpp:133-143):
 *   arch = prior.arch; theta = prior.theta or init_params(arch, seed);
 *   grid = prior.grid or DensityGrid(grid_res, 0); AdamState(lr = eta).
 * theta == NULL -> parameters are drawn on the device from `seed`
 * (same distributions as noma::init_params, field.cpp:150-166, Philox draws).
 * grid == NULL -> zero grid of resolution grid_res (>= 2).
 * box_min/box_max: the metric object-frame box (ObjectTrack::object_box,
 * mapper.hpp:75-77 / Task::object_box, task.hpp:31-33). */
prenom_status prenom_object_create(prenom_ctx_t ctx, const prenom_field_arch* arch,
                                   const float* theta, const float* grid, int grid_res,
                                   uint64_t seed, const prenom_train_cfg* cfg,
                                   const float box_min[3], const float box_max[3],
                                   prenom_object_t* out);
prenom_status prenom_object_destroy(prenom_object_t obj);

/* Training views (train_track reads them from SequenceFrame, mapper.cpp:152-154).
 * All frames share one size. rgb [n][H][W][3], depth [n][H][W], mask [n][H][W].
 * obj_pose: object -> world. The dilation band (render.cpp:17-45) and pixel
 * lists are built once per frame here instead of once per step. */
prenom_status prenom_object_set_frames(prenom_object_t obj, int n_frames,
                                       const prenom_camera* cams, const float* rgb,
                                       const float* depth, const uint8_t* mask,
                                       uint8_t instance_value, const prenom_pose* obj_pose);
/* Replace the pixels of one existing frame (same camera/size); host buffers
 * (pinned for an asynchronous copy) are copied on the sampling stream, after
 * the work already enqueued and before any sampling enqueued later, so a
 * streaming caller's upload of step t+1's keyframe overlaps step t. Used by
 * streaming callers (and bench e2e). */
prenom_status prenom_object_upload_frame(prenom_object_t obj, int frame, const float* rgb,
                                         const float* depth, const uint8_t* mask);
/* Synthetic RGB-D views rendered on the device straight into the object's
 * frames (the device twin of scenes.box_union_scene; stands in for the
 * reference's sdf_render.cpp at cfg5 scale): a union of n_boxes (<= 16)
 * axis-aligned boxes in the scene frame, n views through cams (pixel rays as
 * Camera::pixel_direction, render.hpp:20-22), depth = hit distance +
 * N(0, depth_noise), missing (0) with probability missing_frac (TAG_SYNTH
 * draws), mask instance 1. Band masks and pixel lists are built on the device. */
typedef struct {
  float lo[3], hi[3], albedo[3];
} prenom_box;
prenom_status prenom_object_synth_frames(prenom_object_t obj, int n, const prenom_camera* cams, int n_boxes,
                                         const prenom_box* boxes, float depth_noise, float missing_frac,
                                         uint64_t seed, const prenom_pose* obj_pose);
/* Copy one frame back (any pointer may be NULL): rgb [H][W][3], depth [H][W],
 * and the object / band pixel lists generate_rays draws from (render.cpp:57-66). */
prenom_status prenom_object_get_frame(prenom_object_t obj, int frame, float* rgb, float* depth, int* n_obj_px,
                                      int* n_bg_px, int* obj_px, int* bg_px);

/* ---- train step --------------------------------------------------------
 * n_steps iterations of train_track's loop body (mapper.cpp:150-184):
 * keyframe pick, generate_rays, sample_ray / uniform_samples, field_eval,
 * batch_loss, dense grad zero, field_backward, adam_step, and the grid
 * refresh every grid_refresh_every steps. stats (n_steps entries) may be
 * NULL: the call is then fully asynchronous on the context stream and the
 * stats stay on the device (prenom_object_last_stats reads them). */
prenom_status prenom_train_step(prenom_object_t obj, int n_steps, prenom_step_stats* stats);
prenom_status prenom_object_last_stats(prenom_object_t obj, int n, prenom_step_stats* stats);
/* Streaming train step (same steps as prenom_train_step, nothing synchronizes):
 * the steps' stats and the numeric flag are copied to pinned host memory
 * behind them; *ticket names the call. prefetch_next = 1 also issues the next
 * step's ray sampling after this call's last backward (its keyframe must be
 * resident: upload it first, prenom_object_frame_at tells which). */
prenom_status prenom_train_step_async(prenom_object_t obj, int n_steps, int prefetch_next, uint64_t* ticket);
/* Wait for one async call's stats (the last 4 calls are kept); stats receives
 * its n_steps entries (may be NULL). Returns NUMERIC like train_track's throw. */
prenom_status prenom_wait_stats(prenom_object_t obj, uint64_t ticket, prenom_step_stats* stats);
/* Keyframe index step `step` of this object draws from (TAG_FRAME, mapper.cpp:151). */
prenom_status prenom_object_frame_at(prenom_object_t obj, int64_t step, int* frame);
/* Steps taken so far (AdamState::step). */
prenom_status prenom_object_step(prenom_object_t obj, int64_t* step);
/* Keyframe index the next train step will draw its rays from (TAG_FRAME). */
prenom_status prenom_object_next_frame(prenom_object_t obj, int* frame);
/* Check the device-side numeric flag (NumericError analogue). */
prenom_status prenom_object_check(prenom_object_t obj);

/* ---- render / query ------------------------------------------------------ */
/* "Render": sample + field_eval + composite (render.hpp:79) for explicit
 * object-frame rays. prior_sampling follows the object's cfg; fine draws use
 * TAG_RENDER with c2 = call counter. Escaped rays return colour 0, depth 0. */
prenom_status prenom_render(prenom_object_t obj, int n_rays, const float* origins,
                            const float* dirs, float* rgb_out, float* depth_out);
/* refresh_grid semantics (density_grid.cpp:119-132): sigma at (i,j,k)/(R-1),
 * x-fastest, R^3 floats into out. update_sampling_grid != 0 also installs the
 * result as the object's sampling grid (train_track's refresh). */
prenom_status prenom_density_query(prenom_object_t obj, int R, float* out,
                                   int update_sampling_grid);
/* Mesh extraction, train_track's tail (mapper.cpp:186-187) on the device:
 * density query at R, iso = choose_iso(grid, iso_floor) = max(0.5 max, floor)
 * (density_grid.cpp:134-136) when iso is NaN, then marching_cubes
 * (marching_cubes.cpp:125-180) -- the reference's Mesh exactly: unit-cube
 * vertices, triangles in cell order, vertices numbered by first use after
 * cleanup_mesh (mesh.cpp:30-54). The mesh stays in the object; sizes are
 * returned, prenom_get_mesh copies it out. */
prenom_status prenom_extract_mesh(prenom_object_t obj, int R, float iso, float iso_floor, float* iso_used,
                                  int64_t* n_vertices, int64_t* n_triangles);
/* vertices [n_vertices][3] float, triangles [n_triangles][3] int32 (either may be NULL). */
prenom_status prenom_get_mesh(prenom_object_t obj, float* vertices, int32_t* triangles);
/* The R^3 density lattice the last prenom_extract_mesh ran on (x-fastest), i.e.
 * bake_prior's grid (density_grid.cpp:138-143: refresh_grid then marching_cubes
 * of that grid). res receives R; grid may be NULL. */
prenom_status prenom_get_mesh_grid(prenom_object_t obj, int* res, float* grid);
/* Nearest-neighbour step of noma::chamfer (metrics.cpp:14-22; kd-tree
 * nearest_distance, kdtree.cpp:64-92): min_sq[i] = min_j squared_norm(points[j]
 * - queries[i]) in the reference's float arithmetic (exact minimum). The caller
 * takes sqrt and the two sequential double means (paper_2503_01582_b200.metrics). */
prenom_status prenom_nearest_sq(prenom_ctx_t ctx, int n_queries, const float* queries, int n_points,
                                const float* points, float* min_sq);
/* Batched noma::field_eval (field.cpp:219-225): n points in [0,1]^3. */
prenom_status prenom_field_eval(prenom_object_t obj, int n, const float* xyz, float* sigma,
                                float* rgb);

/* ---- state transfer (save_prior / load_prior sections) ------------------ */
prenom_status prenom_get_params(prenom_object_t obj, float* theta);
prenom_status prenom_set_params(prenom_object_t obj, const float* theta);
prenom_status prenom_get_grid(prenom_object_t obj, int* res, float* grid);
prenom_status prenom_set_grid(prenom_object_t obj, int res, const float* grid);
/* Adam moments (not saved by the reference; for checkpoint/resume). */
prenom_status prenom_get_adam(prenom_object_t obj, float* m, float* v, int64_t* step);
prenom_status prenom_reset_adam(prenom_object_t obj);
/* Restore a checkpointed Adam state (m, v: P floats) and step (resume; the
 * step also keys the Philox draws). Pair with prenom_get_adam / get_params. */
prenom_status prenom_set_adam(prenom_object_t obj, const float* m, const float* v, int64_t step);

/* ---- multi-object ----------------------------------------------------- */
/* Train several objects of one context for n_steps each (no host sync;
 * run_mapper's per-object train_track loop, mapper.cpp:572-585). Objects with
 * the same arch, batch shape (rays, samples, sampler) and tensor-core MLP mode
 * form a group; with grouping on (prenom_ctx_set_grouping) each stage of
 * their step is ONE grouped launch over a
 * per-object descriptor table (sampling, forward, compositing, backward +
 * MLP-gradient reduction, Adam); groups and the other objects run concurrently
 * on lane streams forked from / joined to the context stream. Each object's
 * step is the one prenom_train_step runs (same Philox streams, keyframes and
 * Adam corrections); an object may be listed once. */
prenom_status prenom_train_step_many(prenom_object_t* objs, int n_objs, int n_steps);
/* Grouped launches in prenom_train_step_many: on / off (default: every object
 * on its own launches, the objects concurrently on lane streams).
 * PRENOM_GROUPED=1 sets the default on. */
prenom_status prenom_ctx_set_grouping(prenom_ctx_t ctx, int enable);

/* ---- Reptile (meta.cpp:83-92) -------------------------------------------
 * delta_dev[i] = theta_adapted[i] - theta_meta[i] (device buffer of P floats,
 * e.g. a torch tensor to be all-reduced over NCCL by the caller). Both calls
 * are asynchronous and ordered on the meta object's context stream
 * (prenom_ctx_stream): run the all-reduce on that stream, or synchronize.
 * prenom_reptile_apply: theta_meta <- keep*theta_meta + beta*(theta_meta + delta/n)
 * with keep = 1 - beta, i.e. reptile_update(meta, mean adapted, beta). */
prenom_status prenom_reptile_delta(prenom_object_t meta, prenom_object_t adapted,
                                   float* delta_dev);
prenom_status prenom_reptile_apply(prenom_object_t meta, const float* delta_dev, int n_tasks,
                                   float beta);
/* Copy parameters device-to-device (fresh inner-loop copy: inner_adapt's
 * `ParamVector params = theta`, meta.cpp:31) and reset Adam (meta.cpp:32). */
prenom_status prenom_object_copy_params(prenom_object_t dst, prenom_object_t src);
/* meta <- (1 - beta) * meta + beta * adapted, exactly meta.cpp:83-92 (one task). */
prenom_status prenom_reptile_update(prenom_object_t meta, prenom_object_t adapted, float beta);

/* ---- multi-GPU Reptile: the path's one collective ---------
 * One process per GPU. Rank 0 makes an NCCL unique id, the caller ships its
 * PRENOM_COMM_ID_BYTES bytes to every rank (any transport), and each rank
 * binds a communicator to its context. NCCL is loaded at run time
 * (libnccl.so.2 or $PRENOM_NCCL_LIB); without it these calls fail with
 * PRENOM_CUDA and everything else works. */
#define PRENOM_COMM_ID_BYTES 128
prenom_status prenom_comm_unique_id(uint8_t* id /* PRENOM_COMM_ID_BYTES */);
prenom_status prenom_ctx_init_comm(prenom_ctx_t ctx, int nranks, int rank, const uint8_t* id);
/* nranks = 0 when no communicator is bound; nccl_version as ncclGetVersion. */
prenom_status prenom_ctx_comm_info(prenom_ctx_t ctx, int* nranks, int* rank, int* nccl_version);
/* One Reptile outer step over a meta-batch of n_tasks tasks, n_adapted of
 * them adapted on this rank (meta.cpp:94-120 batched across GPUs):
 *   s = sum over this rank's tasks of (theta_i - theta)       (one kernel)
 *   s = ncclAllReduce(s, sum) over the context's communicator  (if one is bound)
 *   theta <- (1 - beta) theta + beta (theta + s / n_tasks)    = reptile_update
 *                                                (meta, mean adapted, beta)
 * With one task and no communicator it is exactly reptile_update(meta,
 * adapted, beta) (meta.cpp:83-92). Asynchronous on the meta context stream;
 * every rank of the communicator must call it (n_adapted may be 0). */
prenom_status prenom_reptile_step(prenom_object_t meta, const prenom_object_t* adapted,
                                  int n_adapted, int n_tasks, float beta);
/* Philox key of the object's draws (inner_adapt uses mt19937(derive_seed(seed,
 * step)) per meta-step, meta.cpp:111; here: set_seed(derive_seed(...))). */
prenom_status prenom_object_set_seed(prenom_object_t obj, uint64_t seed);

/* ---- single-stage debug / parity entry points ---------------------------
 * Run one stage on caller (host) buffers so unit parity does not depend on
 * the loop. `arch` + `params` describe a field (P floats, reference layout). */
prenom_status prenom_debug_philox(prenom_ctx_t ctx, int n, const uint32_t* ctr_key /* n x 6 */,
                                  uint32_t* out /* n x 4 */);
/* hash_encode (field.cpp:168-172): n points -> n x (L*F) features. */
prenom_status prenom_debug_hash_encode(prenom_ctx_t ctx, const prenom_field_arch* arch,
                                       const float* params, int n, const float* xyz,
                                       float* features);
/* field_eval with cache outputs: sigma[n], rgb[n*3], raw[n*4] (raw may be NULL). */
prenom_status prenom_debug_field_eval(prenom_ctx_t ctx, const prenom_field_arch* arch,
                                      const float* params, int n, const float* xyz,
                                      float* sigma, float* rgb, float* raw, int mlp_precision);
/* (mlp_precision 0: exact per-point kernel; 1 / 2: the tcgen05 train-path tile
 * forward in bf16 / split bf16; 3: the fp32 SIMT train-path tile forward.) */
/* Sum over points of field_backward (field.cpp:227-293) into grad (P floats,
 * overwritten). */
prenom_status prenom_debug_field_backward(prenom_ctx_t ctx, const prenom_field_arch* arch,
                                          const float* params, int n, const float* xyz,
                                          const float* d_sigma, const float* d_rgb, float* grad,
                                          int mlp_precision);
/* Phase trace of the tensor-core backward (set PRENOM_BWD_WAIT bit 8 before the
 * first backward launch): clock64 stamps of CTA 0's first 64 tiles, MLP issuing
 * thread mlp[64][16] (slots 0..10) and first scatter thread scatter[64][4]; and
 * (cta may be NULL) per CTA cta[1024][5]: globaltimer ns at entry, after the
 * prologue, at the end of its tiles and at exit, and its tile count. */
prenom_status prenom_debug_bwd_trace(prenom_ctx_t ctx, int64_t* mlp, int64_t* scatter, int64_t* cta);
/* L2 read bandwidth probe: an L2-resident buffer of mbytes MiB re-read reps times in one
 * launch; *gbs = bytes read / time (the L2 roofline denominator, measured on the box). */
prenom_status prenom_debug_l2_read(prenom_ctx_t ctx, int mbytes, int reps, double* gbs);
/* adam_step (field.cpp:295-310) on n floats; *step in/out. */
prenom_status prenom_debug_adam(prenom_ctx_t ctx, size_t n, float* params, const float* grads,
                                float* m, float* v, int64_t* step, float lr, float beta1,
                                float beta2, float eps);
/* sample_ray / uniform_samples for explicit rays (density_grid.cpp:110-117,
 * render.cpp:104-132): out per ray S = (prior ? n_fine : n_fine) samples;
 * count[r] = 0 when escaped. grid may be NULL when prior == 0.
 * Draws: TAG_FINE with c1 = ray, c2 = step. */
prenom_status prenom_debug_sample_rays(prenom_ctx_t ctx, int n_rays, const float* origins,
                                       const float* dirs, const float box_min[3],
                                       const float box_max[3], int prior, int grid_res,
                                       const float* grid, int n_coarse, int n_fine, float eps,
                                       uint64_t seed, int64_t step, float* depths,
                                       float* deltas, float* positions, int* count,
                                       float* t_entry, float* t_exit);
/* composite + composite_backward + batch_loss for explicit per-sample field
 * outputs (render.cpp:134-243). Rays have S samples each (count[r] = 0 or S).
 * bg_colors: 3 per ray (used for background rays). terms = {total, color,
 * depth, sigma}; d_sigma/d_rgb per sample; color_out/depth_out per ray. */
prenom_status prenom_debug_batch_loss(prenom_ctx_t ctx, int n_rays, int S, const int* kind,
                                      const float* target_rgb, const float* target_depth,
                                      const int* count, const float* deltas,
                                      const float* depths, const float* sigma, const float* rgb,
                                      const float* bg_colors, float lambda_d,
                                      float lambda_sigma, double* terms, float* d_sigma,
                                      float* d_rgb, float* color_out, float* depth_out);
/* generate_rays (render.cpp:47-102) for the object's frame `frame` at `step`:
 * origins/dirs [n][3], kind [n], target_rgb [n][3], target_depth [n] (-1 when
 * absent), pick_px [n] = x + W*y. */
prenom_status prenom_debug_generate_rays(prenom_object_t obj, int frame, int64_t step,
                                         float* origins, float* dirs, int* kind,
                                         float* target_rgb, float* target_depth, int* pick_px);

/* One tcgen05 tile GEMM D[M][N] = A[M][K] * B[N][K]^T (bf16 operands, fp32
 * accumulate in TMEM), operands staged K-major or MN-major: unit test of the
 * tensor-core building blocks the fused MLP kernels use. M in {64,128},
 * N % 8 == 0 (16 for M=128), K % 16 == 0. */
prenom_status prenom_debug_umma_gemm(prenom_ctx_t ctx, int M, int N, int K, int a_mn, int b_mn,
                                     const float* A, const float* B, float* D);

/* marching_cubes (marching_cubes.cpp:125-180) of a caller grid (R^3 floats,
 * x-fastest, host memory) on the device; the result is kept in the context
 * until the next call and copied out by prenom_debug_mesh_get. */
prenom_status prenom_debug_marching_cubes(prenom_ctx_t ctx, int R, const float* grid, float iso,
                                          int64_t* n_vertices, int64_t* n_triangles);
prenom_status prenom_debug_mesh_get(prenom_ctx_t ctx, float* vertices, int32_t* triangles);
/* Host only: the cube-edge triangles of one of the 256 corner configurations
 * (cube_case_triangles, marching_cubes.cpp:115-117) into edges[3 * count];
 * returns count (<= 16), or -1 for a bad config. */
int prenom_mc_case_triangles(int config, int* edges);

#ifdef __cplusplus
}
#endif

#endif /* PRENOM_GPU_H */
