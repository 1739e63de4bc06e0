/*
 * vpb200.h -- C ABI of the B200-native ParaMaP mapping-and-planning hot path.
 *
 * Every entry point takes plain pointers and sizes (no torch types).  Pointers
 * marked (dev) are CUDA device pointers owned by the caller; (host) pointers
 * are read during the call only.  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Nothing here allocates device memory (except SMPC sessions): scratch is passed in
 * as a caller-owned workspace whose size the matching *_workspace_bytes()
 * function reports.  Every function returns VPB_OK (0) or an error code;
 * vpb_last_error() describes the most recent failure on the calling thread.
 *
 * The reference (/root/reference/pkg/src/voxplan, "vp/") has no formal plugin
 * registry: its boundary is a set of module-level numba kernels looked up at
 * call time.  Each entry below names the reference
 * function it replaces; INTEGRATION.md shows the ctypes shim that binds it in
 * place of the numba seam.
 */
#ifndef VPB200_H
#define VPB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPB_OK 0
#define VPB_ERR_ARG 1  /* invalid argument (shape, limit, null pointer) */
#define VPB_ERR_CUDA 2 /* CUDA launch / runtime error */

#define VPB_MAX_JOINTS 16
#define VPB_MAX_SPHERES 64
#define VPB_MAX_PAIRS 256
#define VPB_MAX_MASK_SPHERES 64

int vpb_version(void);
const char *vpb_last_error(void);
/* Number of kernels this library has launched since load (diagnostics). */
uint64_t vpb_launch_count(void);
/* Host -> device upload through a caller-owned pinned staging buffer: copies
 * `bytes` from src_host into pinned (on the host, now) and enqueues the
 * pinned -> dst_dev copy on `stream` (the depth frame of a map update; the
 * caller must not reuse `pinned` before that copy has run). */
int vpb_stage_h2d(void *dst_dev, void *pinned, const void *src_host, int64_t bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* Mapping                                                                   */
/* ------------------------------------------------------------------------ */

/* Pinhole depth camera (vp/mapping.py:143-166, CameraModel). */
typedef struct {
  double fx, fy, cx, cy, d_min, d_max;
  int64_t width, height;
  double pose_r[9], pose_t[3]; /* camera -> world (cam.pose) */
  double w2c_r[9], w2c_t[3];   /* world -> camera (cam.world_to_camera()) */
} vpb_camera;

/* Log-odds constants (vp/mapping.py:41-50, MapParams) and tau. */
typedef struct {
  double l_hit, l_miss, l_min, l_max, l_occ_threshold, tau;
} vpb_map_params;

/* Dense grid state: log_odds f64 and observed u8 over (gx, gy, gz), C order
 * x*gy*gz + y*gz + z (vp/mapping.py:3-4).  occ_bits (optional) is the packed
 * occupancy mask maintained next to the log-odds: bit (z & 31) of word
 * (x*gy + y)*ceil(gz/32) + (z >> 5) is set iff log_odds >= l_occ_threshold. */
typedef struct {
  double *log_odds;   /* (dev) */
  uint8_t *observed;  /* (dev) */
  uint32_t *occ_bits; /* (dev) or NULL */
  int64_t dims[3];
  double origin[3];
  double voxel;
} vpb_grid;

/* Number of uint32 words of the packed occupancy mask of a grid. */
int64_t vpb_occ_words(const int64_t dims[3]);

/* Rebuild occ_bits from log_odds over the whole grid (used after direct
 * writes to log_odds).  Replaces the `grid.occupied_mask()` threshold of
 * vp/mapping.py:113-114 / :601. */
int vpb_occ_bits_from_log_odds(const vpb_grid *grid, double l_occ_threshold,
                               void *stream);

/* Pixels whose back-projection lies inside an inflated mask sphere.
 * Replaces vp/mapping.py:357-380 (_masked_pixels).
 * depth (dev) H x W f64; centers (host) n x 3; radii (host) n; out (dev) u8. */
int vpb_masked_pixels(const double *depth, const vpb_camera *cam,
                      const double *centers, const double *radii,
                      int64_t n_mask, double pad, uint8_t *out, void *stream);

/* Robot-masked voxel-projection fusion over box [lo, lo+n).
 * Replaces vp/mapping.py:266-354 (_fuse_voxels, 29 args) -- bitwise equal
 * log_odds / observed (fp64, reference operation order, no FMA).  When
 * grid->occ_bits is non-NULL it is kept consistent with the new log-odds.
 * depth (dev) H x W f64; pixel_masked (dev) H x W u8; centers/radii (host). */
int vpb_fuse_voxels(const vpb_grid *grid, const int64_t lo[3],
                    const int64_t n[3], const vpb_camera *cam,
                    const double *depth, const uint8_t *pixel_masked,
                    const double *centers, const double *radii,
                    int64_t n_mask, const vpb_map_params *params, void *stream);

/* Masked pixels + fusion in one call: vp/mapping.py:386-455
 * (update_occupancy).  pixel_scratch (dev) holds
 * vpb_pixel_scratch_bytes(W, H) bytes: a per-pixel class byte, two slots for
 * the bounding rectangle of the usable pixels (used to skip whole voxel
 * ranges; consecutive calls on one scratch alternate between them, each call
 * clearing the other) and the usable depth per pixel in fp32.  ZERO-initialise
 * it once at allocation; calls sharing a scratch must be stream-ordered.  (A
 * CUDA graph that captures the call replays one slot: the rectangle then only
 * grows -- the result stays exact, the culling gets looser.) */
int64_t vpb_pixel_scratch_bytes(int64_t width, int64_t height);
int vpb_update_occupancy(const vpb_grid *grid, const int64_t lo[3],
                         const int64_t n[3], const vpb_camera *cam,
                         const double *depth, const double *centers,
                         const double *radii, int64_t n_mask, double mask_pad,
                         const vpb_map_params *params, uint8_t *pixel_scratch,
                         void *stream);

/* Snapshot journal (copy-on-write snapshots of a live grid, vp/mapping.py
 * :125-133 freeze / :713-723 snapshot): while a snapshot of the grid is alive,
 * each update records, before its first write to a 32-voxel word, the word's
 * old log-odds and observed (all 32 z) and its old occupancy word.  A
 * snapshot is then O(1); it is materialised (clone + these undo records,
 * newest update first) only if its grid is read.  All buffers (dev) are
 * caller-owned; count (dev) is the number of records written, capacity the
 * records the buffers hold (the host sizes it so one update cannot overflow:
 * at most one record per word of the box). */
typedef struct {
  int64_t *idx;              /* [capacity] word (x * Ny + y) * ceil(Nz / 32) + z / 32 */
  double *lo;                /* [capacity * 32] old log-odds of the word's z */
  uint8_t *ob;               /* [capacity * 32] old observed */
  uint32_t *occ;             /* [capacity] old occupancy word */
  unsigned long long *count; /* records written (dev) */
  unsigned int *overflow;    /* set if a record did not fit (dev) */
  uint64_t capacity;
  /* segment bookkeeping, done on the device before the update's first record:
   * if reset != 0, count = 0; then starts[seg] = count (starts may be NULL) */
  int64_t *starts;
  int32_t seg;
  int32_t reset;
} vpb_journal;

/* vpb_update_occupancy that also journals the words it modifies
 * (journal == NULL: identical to vpb_update_occupancy). */
int vpb_update_occupancy_journaled(const vpb_grid *grid, const int64_t lo[3],
                                   const int64_t n[3], const vpb_camera *cam,
                                   const double *depth, const double *centers,
                                   const double *radii, int64_t n_mask,
                                   double mask_pad,
                                   const vpb_map_params *params,
                                   uint8_t *pixel_scratch,
                                   const vpb_journal *journal, void *stream);

/* Undo records [first, last) of one update (unique words) written back into
 * grid (a clone of the live grid); call per update, newest first. */
int vpb_journal_restore(const vpb_grid *grid, const vpb_journal *journal,
                        int64_t first, int64_t last, void *stream);

/* Exact squared EDT of the occupied voxels of box [lo, lo+n).
 * Replaces the body of vp/mapping.py:586-613 (edt_3d: threshold, the three
 * _edt_pass_* FH passes of :458-550, and the inf mapping).  Output out_sq
 * (dev) is f32 (n0, n1, n2) C order: exact integer squared voxel distances
 * (exact in f32 up to 2^24), +inf everywhere iff the box holds no source.
 * Source: grid->occ_bits when use_bits != 0 (must be current), else the
 * log-odds threshold.  workspace (dev) >= vpb_edt3d_workspace_bytes(n). */
size_t vpb_edt3d_workspace_bytes(const int64_t n[3]);
int vpb_edt3d(const vpb_grid *grid, const int64_t lo[3], const int64_t n[3],
              double l_occ_threshold, int use_bits, float *out_sq,
              void *workspace, size_t workspace_bytes, void *stream);

/* Distance field view (vp/mapping.py:556-583, DistanceField) consumed by the
 * query and by the rollout kernel.  `sq` holds exact squared voxel distances
 * between voxel centres (+inf = no source), as vpb_edt3d writes them: the
 * fp32 rollout relies on sqrt(sq) being 1-Lipschitz to skip far cells. */
typedef struct {
  const float *sq; /* (dev) (n0, n1, n2), NULL = no field (snap=None) */
  int64_t n[3];
  int64_t lo[3];
  double origin[3];
  double voxel;
  double outside_default;
} vpb_field;

/* Batched distance query: replaces vp/mapping.py:616-710 (_query_metric /
 * query_distance), evaluated in fp64 exactly as the reference.
 * points (dev) count x 3 f64; out (dev) count f64. */
int vpb_query_distance(const vpb_field *field, const double *points,
                       int64_t count, double *out, void *stream);

/* ------------------------------------------------------------------------ */
/* Planner                                                                   */
/* ------------------------------------------------------------------------ */

/* Packed robot + objective (vp/planner.py:461-499 Planner.__init__ packing,
 * vp/planner.py:38-102 PlannerParams) plus the per-call state and goal.
 * Spheres must be sorted by link (the Python host sorts and keeps sph_orig
 * so outputs come back in the caller's sphere order). */
typedef struct {
  int32_t n_joints, n_spheres, n_pairs, horizon;
  double dt;
  double base_r[9], base_t[3];
  double off_r[VPB_MAX_JOINTS * 9], off_t[VPB_MAX_JOINTS * 3];
  double axes[VPB_MAX_JOINTS * 3];
  int32_t sph_link[VPB_MAX_SPHERES];
  int32_t sph_orig[VPB_MAX_SPHERES];
  double sph_loc[VPB_MAX_SPHERES * 3], sph_r[VPB_MAX_SPHERES];
  int32_t pairs[VPB_MAX_PAIRS * 2];
  double goal_r[9], goal_t[3];
  double pose_weight[36], terminal_weight[36];
  double pos_lo[VPB_MAX_JOINTS], pos_hi[VPB_MAX_JOINTS];
  double vel_lo[VPB_MAX_JOINTS], vel_hi[VPB_MAX_JOINTS];
  double acc_lo[VPB_MAX_JOINTS], acc_hi[VPB_MAX_JOINTS];
  double acc_limit[VPB_MAX_JOINTS]; /* |command| clip (vp/planner.py:618) */
  double q_ref[VPB_MAX_JOINTS];
  double q0[VPB_MAX_JOINTS], qd0[VPB_MAX_JOINTS];
  double w_env, w_self, w_q, w_qd, w_qdd, w_s, w_ns, d_act;
  double lam; /* softmin temperature (vp/planner.py:373-384) */
  /* (dev, optional) per-call state [q0 (n), qd0 (n), goal_r (9), goal_t (3)]
   * f64; when set it overrides q0/qd0/goal_* so a captured CUDA graph can be
   * replayed after one small host->device copy. */
  const double *dyn_state;
  /* (dev, optional) device location holding the distance-field pointer; when
   * set it overrides field->sq (same box / dims / origin), so a captured step
   * follows a field that is rebuilt into a new buffer every map update. */
  const float *const *field_sq_dev;
} vpb_problem;

#define VPB_PREC_F32 0 /* production: fp32 arithmetic, fp64 cost sums */
#define VPB_PREC_F64 1 /* parity mode: fp64 end to end */

#define VPB_DTYPE_F32 0
#define VPB_DTYPE_F64 1

/* Rollout + cost evaluation of M control sequences.
 * Replaces vp/batch.py:161-336 (evaluate_batch, 49 args).
 * controls (dev) M x H x n of `dtype`; `nominal` (dev, H x n, same dtype) is
 * added to every sample when non-NULL (controls then hold perturbations);
 * nominal is always f64, controls may be f32 or f64.
 * costs (dev) M f64, terms (dev) M x 6 f64, flags (dev) M u8 (1 = log-map
 * singularity, cost = inf); traj_q/traj_qd (dev, M x (H+1) x n f64) and
 * sphere_pos (dev, M x H x S x 3 f64) are optional (NULL = not stored). */
int vpb_evaluate_batch(const vpb_problem *prob, const vpb_field *field,
                       const void *controls, const void *nominal, int dtype,
                       int64_t M, int precision, double *costs, double *terms,
                       uint8_t *flags, double *traj_q, double *traj_qd,
                       double *sphere_pos, void *stream);

/* Softmin weights (vp/planner.py:373-384): w = exp(-(S - min S)/lam) / sum.
 * costs (dev) M f64 -> weights (dev) M f64; stats (dev, 3 f64) receives
 * [min, Z, nonfinite_count].  Fixed-order reduction (deterministic). */
size_t vpb_soft_weights_workspace_bytes(int64_t M);
int vpb_soft_weights(const double *costs, int64_t M, double lam,
                     double *weights, double *stats, void *workspace,
                     size_t workspace_bytes, void *stream);

/* Weighted mean update (vp/planner.py:387-400): out = nominal + sum_m w_m eps_m.
 * nominal (dev, H*n f64), eps (dev, M x H*n of dtype), weights (dev, M f64). */
size_t vpb_update_controls_workspace_bytes(int64_t M, int64_t hn);
int vpb_update_controls(const double *nominal, const void *eps, int dtype,
                        const double *weights, int64_t M, int64_t hn,
                        double *out, void *workspace, size_t workspace_bytes,
                        void *stream);

/* One SMPC iteration on this device's shard of samples, in ONE kernel launch
 * (vp/planner.py:594-630 smpc_step minus sampling): rollout of nominal + eps
 * (M local samples, eps of `dtype`, nominal f64 H x n) -> per-CTA softmin
 * partials (local min m_c, Z_c = sum exp(-(S-m_c)/lam), N_c = sum w eps) ->
 * fixed-order merges by the last CTA of each group and the last group ->
 * this shard's partial
 *   part_out (dev) = [m_r, Z_r, nonfinite_r, best_index_r, N_r[H*n]]
 * (the record ranks all-gather).  m_offset = global
 * index of local sample 0.  costs (dev, M f64) / flags (dev, M u8) optional. */
size_t vpb_smpc_workspace_bytes(int64_t M, int64_t H, int64_t n);
int64_t vpb_smpc_partial_len(int64_t H, int64_t n);
int vpb_smpc_partial(const vpb_problem *prob, const vpb_field *field,
                     const void *eps, int dtype, const double *nominal,
                     int64_t M, int64_t m_offset, int precision,
                     double *costs, uint8_t *flags, double *part_out,
                     void *workspace, size_t workspace_bytes, void *stream);

/* Single-device SMPC step, fully fused in one launch: the partial above,
 * then (by the last CTA) U* = nominal + N/Z, the clipped command, the
 * shifted warm start and the M = 1 re-evaluation of U* (vp/planner.py:
 * 614-629).  out (dev) layout (vpb_smpc_out_len doubles):
 *   [U* (H*n), command (n), next_nominal (H*n), weighted_cost, terms[6],
 *    best_cost, Z, nonfinite_count, best_index, e_pos, e_ori]
 * (e_pos / e_ori: end-effector errors at the start state, vp/planner.py:
 * 620-629; filled by vpb_ee_errors on the host, NaN from the device step)
 * (weighted_cost = +inf when the re-evaluation hits the log singularity;
 * nonfinite_count = samples flagged at the log singularity + 2^32 x samples
 * with any other non-finite cost: the reference raises DegenerateRotation for
 * the former, ValueError from soft_weights for the latter). */
int64_t vpb_smpc_out_len(int64_t H, int64_t n);
int vpb_smpc_step(const vpb_problem *prob, const vpb_field *field,
                  const void *eps, int dtype, const double *nominal, int64_t M,
                  int precision, double *costs, uint8_t *flags, double *out,
                  void *workspace, size_t workspace_bytes, void *stream);

/* Draw + step in one call: the perturbations of vpb_sample_perturbations
 * (same seed / m_offset / window / sigma -> identical values) go to eps_out
 * (dev, M x H x n, f32 for VPB_PREC_F32, f64 otherwise) and the step runs on
 * them -- the single-device step into `out` or this shard's partial into
 * `part_out` (exactly one non-NULL).  For the compiled robot topology in fp32
 * with window <= 5 the draws happen inside the step kernel (no sampler
 * launch, no read-back of the noise). */
int vpb_smpc_generate(const vpb_problem *prob, const vpb_field *field, uint64_t seed, const uint64_t *seed_dev,
                      int64_t m_offset, int64_t window, const double *sigma, const double *nominal, int64_t M,
                      int precision, double *costs, uint8_t *flags, void *eps_out, double *part_out, double *out,
                      void *workspace, size_t workspace_bytes, void *stream);

/* Debug export of the softmin weights of the last single-device step run on
 * `workspace` (vpb_smpc_step / vpb_smpc_generate with `out`): weights (dev,
 * M f64) receives w_m = exp(-(S_m - min S)/lam) / Z exactly as the fused
 * merge computed them (zeros for the candidates it proved negligible).  Test
 * infrastructure for the weight parity of vp/planner.py:373-384. */
int vpb_smpc_debug_weights(const vpb_problem *prob, int64_t M, const void *workspace, size_t workspace_bytes,
                           double *weights, void *stream);

/* Multi-device finish: merge R rank partials (R x partial_len, dev) in rank
 * order and run the same tail as vpb_smpc_step into `out`. */
size_t vpb_smpc_finish_workspace_bytes(int64_t n_parts, int64_t H, int64_t n);
int vpb_smpc_finish(const vpb_problem *prob, const vpb_field *field,
                    const double *partials, int64_t n_parts,
                    const double *nominal, int precision, double *out,
                    void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* Perturbation sampler (vp/planner.py:182-219)     */
/* ------------------------------------------------------------------------ */
/* Counter-based Philox4x32-10 stream keyed by (seed, sample index), standard
 * normals, moving-average smoothing over `window` (rows scaled 1/sqrt(count)),
 * times sigma[j]; sample 0 is the zero perturbation.  Statistically (not
 * bitwise) equivalent to numpy's Philox stream.  seed_dev (dev, optional)
 * overrides `seed` (graph replays).  m_offset = global index of local sample
 * 0 (sharded sampling).  out (dev) M x H x n of dtype. */
int vpb_sample_perturbations(uint64_t seed, const uint64_t *seed_dev,
                             int64_t m_offset, int64_t M, int64_t H, int64_t n,
                             int64_t window, const double *sigma, int dtype,
                             void *out, void *stream);

/* ------------------------------------------------------------------------ */
/* SMPC session: one host call per step (vp/planner.py:594-630 with host     */
/* buffers).  Owns pinned staging, device buffers and a captured CUDA graph  */
/* (H2D of the per-call block -> sampler -> fused step -> D2H).              */
/* ------------------------------------------------------------------------ */
typedef struct vpb_smpc_session vpb_smpc_session;

/* Length of the step output (same layout as vpb_smpc_step's `out`). */
int64_t vpb_smpc_session_out_len(int64_t H, int64_t n);
/* prob/field (host structs, copied; prob->q0/qd0/goal_* and dyn_state are
 * ignored), M samples, noise window and sigma (n) of the sampler, precision.
 * The field's box, dims, origin and voxel are fixed for the session; its
 * device buffer may change per step (vpb_smpc_session_step's field_sq). */
int vpb_smpc_session_create(const vpb_problem *prob, const vpb_field *field, int64_t M, int64_t window,
                            const double *sigma, int precision, vpb_smpc_session **out);
/* One step: q0, qd0 (n), goal_r (9, row major), goal_t (3), nominal (H x n,
 * NULL = zeros) and the seed are host inputs; field_sq (dev, NULL = the
 * creation-time buffer); out (host, vpb_smpc_session_out_len doubles).  The
 * graph is replayed on `stream` (NULL = the legacy default stream), so it is
 * ordered after the work that produced the field; the call returns when the
 * step is complete. */
int vpb_smpc_session_step(vpb_smpc_session *session, const double *q0, const double *qd0, const double *goal_r,
                          const double *goal_t, const double *nominal, uint64_t seed, const float *field_sq,
                          double *out, void *stream);
/* Asynchronous replay of the step graph on `stream` with the inputs staged
 * by the previous vpb_smpc_session_step (device-side timing, pipelining);
 * the result lands in the session's pinned buffer when the stream reaches
 * it.  Returns without synchronising. */
int vpb_smpc_session_launch(vpb_smpc_session *session, void *stream);
int vpb_smpc_session_destroy(vpb_smpc_session *session);

/* Step diagnostics on the host (vp/planner.py:620-629): end-effector position
 * error and quaternion angle to the goal at configuration q0 (n), in double,
 * following forward_kinematics (vp/robot.py:172-189) and quaternion_angle
 * (vp/geometry.py:368-371).  The step outputs leave their e_pos / e_ori slots
 * to this function (the session fills them). */
int vpb_ee_errors(const vpb_problem *prob, const double *q0, const double *goal_r, const double *goal_t,
                  double *e_pos, double *e_ori);

/* ------------------------------------------------------------------------ */
/* Diagnostics                                                               */
/* ------------------------------------------------------------------------ */
/* Phase timestamps (%globaltimer, ns) of subsequent SMPC launches into a
 * device buffer of >= 2 * ceil(M / 4) + 16 uint64: per CTA [start, candidates
 * done], then [group merges done, global merge done, step done].  NULL turns
 * it off (tools/smpc_trace.py). */
void vpb_debug_smpc_trace(unsigned long long *dev_buffer);

#ifdef __cplusplus
}
#endif

#endif /* VPB200_H */
