// SMPC session: the whole single-device step behind one host call.
//
// Planner.smpc_step (vp/planner.py:594-630) with host buffers in and out: the
// per-call block (start state, goal, seed, field pointer, warm start) is
// written to pinned memory, one captured CUDA graph replays
//   SMPC step: block 0 of the fused step kernel copies the block from the
//   host-mapped buffer to the device while the other CTAs wait on a flag (no
//   copy node: a graph copy node costs ~9 us on B200, the in-kernel copy one
//   PCIe round trip); the perturbations are drawn inside the kernel for the
//   compiled topology; the merging CTA writes the packed result straight into
//   pinned host memory,
// and the call returns after a stream synchronisation.  The session owns its
// device buffers (allocated once at creation), so a step does no allocation,
// no attribute setting and no per-kernel host work.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "vpb_common.cuh"

struct vpb_smpc_session {
  vpb_problem prob;
  vpb_field field;
  int64_t M, H, n, window;
  int precision, dtype;
  double sigma[VPB_MAX_JOINTS];
  cudaStream_t stream;
  cudaGraphExec_t exec;
  vpb::SmpcNode *node;     // fused fp32 path: the step kernel's parameters (per-call state patched in)
  cudaGraphNode_t gnode;   // its kernel node in `exec`
  bool direct;             // re-parameterising the node failed: launch the kernel directly
  cudaEvent_t launched;  // recorded after an asynchronous vpb_smpc_session_launch
  bool inflight;         // a launch() replay may still read h_in / write h_out
  double *h_in, *d_in;  // [dyn (2n + 12) | seed bits | field pointer bits | nominal (H n)]
  double *h_out, *d_out;
  void *eps, *ws;
  size_t ws_bytes;
  int64_t dyn_len, in_len, out_len;
};

namespace {

void release(vpb_smpc_session *s) {
  if (!s) return;
  if (s->inflight) cudaEventSynchronize(s->launched);
  if (s->launched) cudaEventDestroy(s->launched);
  if (s->exec) cudaGraphExecDestroy(s->exec);
  if (s->node) vpb::smpc_session_node_free(s->node);
  if (s->stream) cudaStreamDestroy(s->stream);
  cudaFreeHost(s->h_in);
  cudaFreeHost(s->h_out);
  cudaFree(s->d_in);
  cudaFree(s->d_out);
  cudaFree(s->eps);
  cudaFree(s->ws);
  delete s;
}

int enqueue(vpb_smpc_session *s, bool copies) {
  const int64_t nom = s->dyn_len + 2;
  // the per-call block travels host-mapped -> device inside the fused step
  // kernel (or by a copy that smpc_generate_session enqueues on other paths);
  // the step kernel writes the result straight into the pinned host buffer
  return vpb::smpc_generate_session(&s->prob, &s->field, reinterpret_cast<const uint64_t *>(s->d_in + s->dyn_len),
                                    s->window, s->sigma, s->d_in + nom, s->M, s->precision, s->eps, s->d_out,
                                    s->h_out, s->ws, s->ws_bytes, s->stream, copies ? s->h_in : nullptr, s->d_in,
                                    s->in_len);
}

// Fused fp32 path: replay the one-node graph with this step's parameters
// (or, if the node cannot be re-parameterised, launch the kernel directly).
cudaError_t launch_node(vpb_smpc_session *s, cudaStream_t st, bool reparam) {
  const cudaKernelNodeParams *np = vpb::smpc_session_node_params(s->node);
  if (!s->direct && reparam && cudaGraphExecKernelNodeSetParams(s->exec, s->gnode, np) != cudaSuccess) {
    cudaGetLastError();
    s->direct = true;
  }
  if (s->direct) return cudaLaunchKernel(np->func, np->gridDim, np->blockDim, np->kernelParams, np->sharedMemBytes, st);
  return cudaGraphLaunch(s->exec, st);
}

// 3x3 row-major helpers (host, double)
void mat_mul(const double *a, const double *b, double *c) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

// Rotation3.from_axis_angle (vp/geometry.py:77-83, _so3_exp :284-294)
void so3_exp(const double *axis, double angle, double *r) {
  const double w[3] = {axis[0] * angle, axis[1] * angle, axis[2] * angle};
  const double theta = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  const double k[9] = {0.0, -w[2], w[1], w[2], 0.0, -w[0], -w[1], w[0], 0.0};
  double a, b;
  if (theta < 1e-6) {  // SMALL_ANGLE, vp/geometry.py:22
    a = 1.0 - theta * theta / 6.0;
    b = 0.5 - theta * theta / 24.0;
  } else {
    a = std::sin(theta) / theta;
    b = (1.0 - std::cos(theta)) / (theta * theta);
  }
  double kk[9];
  mat_mul(k, k, kk);
  for (int i = 0; i < 9; ++i) r[i] = (i % 4 == 0 ? 1.0 : 0.0) + a * k[i] + b * kk[i];
}

// UnitQuaternion.from_rotation (Shepperd, vp/geometry.py:232-266), normalised
void quat_from_rotation(const double *m, double q[4]) {
  const double tr = m[0] + m[4] + m[8];
  double s;
  if (tr > 0.0) {
    s = std::sqrt(tr + 1.0) * 2.0;
    q[0] = 0.25 * s, q[1] = (m[7] - m[5]) / s, q[2] = (m[2] - m[6]) / s, q[3] = (m[3] - m[1]) / s;
  } else if (m[0] > m[4] && m[0] > m[8]) {
    s = std::sqrt(1.0 + m[0] - m[4] - m[8]) * 2.0;
    q[0] = (m[7] - m[5]) / s, q[1] = 0.25 * s, q[2] = (m[1] + m[3]) / s, q[3] = (m[2] + m[6]) / s;
  } else if (m[4] > m[8]) {
    s = std::sqrt(1.0 + m[4] - m[0] - m[8]) * 2.0;
    q[0] = (m[2] - m[6]) / s, q[1] = (m[1] + m[3]) / s, q[2] = 0.25 * s, q[3] = (m[5] + m[7]) / s;
  } else {
    s = std::sqrt(1.0 + m[8] - m[0] - m[4]) * 2.0;
    q[0] = (m[3] - m[1]) / s, q[1] = (m[2] + m[6]) / s, q[2] = (m[5] + m[7]) / s, q[3] = 0.25 * s;
  }
  const double nq = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  for (int i = 0; i < 4; ++i) q[i] /= nq;
}

}  // namespace

extern "C" {

int vpb_ee_errors(const vpb_problem *p, const double *q0, const double *goal_r, const double *goal_t, double *e_pos,
                  double *e_ori) {
  VPB_REQUIRE(p && q0 && goal_r && goal_t && e_pos && e_ori, "null argument to vpb_ee_errors");
  // forward_kinematics (vp/robot.py:172-189): T <- T @ offset_i @ rot(axis_i, q_i)
  double R[9], t[3], tmp[9], rot[9];
  memcpy(R, p->base_r, sizeof(R));
  memcpy(t, p->base_t, sizeof(t));
  for (int i = 0; i < p->n_joints; ++i) {
    const double *orr = p->off_r + 9 * i, *ot = p->off_t + 3 * i;
    double tn[3];
    for (int a = 0; a < 3; ++a) tn[a] = R[3 * a] * ot[0] + R[3 * a + 1] * ot[1] + R[3 * a + 2] * ot[2] + t[a];
    mat_mul(R, orr, tmp);
    so3_exp(p->axes + 3 * i, q0[i], rot);
    mat_mul(tmp, rot, R);
    memcpy(t, tn, sizeof(t));
  }
  const double dx = t[0] - goal_t[0], dy = t[1] - goal_t[1], dz = t[2] - goal_t[2];
  *e_pos = std::sqrt(dx * dx + dy * dy + dz * dz);
  // quaternion_angle (vp/geometry.py:368-371)
  double qa[4], qb[4];
  quat_from_rotation(R, qa);
  quat_from_rotation(goal_r, qb);
  double d = std::fabs(qa[0] * qb[0] + qa[1] * qb[1] + qa[2] * qb[2] + qa[3] * qb[3]);
  d = d > 1.0 ? 1.0 : (d < -1.0 ? -1.0 : d);
  *e_ori = 2.0 * std::acos(d);
  return VPB_OK;
}


int64_t vpb_smpc_session_out_len(int64_t H, int64_t n) { return vpb_smpc_out_len(H, n); }

int vpb_smpc_session_create(const vpb_problem *prob, const vpb_field *field, int64_t M, int64_t window,
                            const double *sigma, int precision, vpb_smpc_session **out) {
  VPB_REQUIRE(prob && out && sigma, "null argument to vpb_smpc_session_create");
  VPB_REQUIRE(M >= 1 && prob->horizon >= 1 && prob->n_joints >= 1 && prob->n_joints <= VPB_MAX_JOINTS,
              "bad session shape");
  VPB_REQUIRE(precision == VPB_PREC_F32 || precision == VPB_PREC_F64, "bad precision %d", precision);
  *out = nullptr;
  auto *s = new vpb_smpc_session();
  memset(s, 0, sizeof(*s));
  s->prob = *prob;
  if (field) s->field = *field;
  s->M = M;
  s->H = prob->horizon;
  s->n = prob->n_joints;
  s->window = window;
  s->precision = precision;
  s->dtype = precision == VPB_PREC_F32 ? VPB_DTYPE_F32 : VPB_DTYPE_F64;
  for (int64_t j = 0; j < s->n; ++j) s->sigma[j] = sigma[j];
  s->dyn_len = 2 * s->n + 12;
  s->in_len = s->dyn_len + 2 + s->H * s->n;
  s->out_len = vpb_smpc_out_len(s->H, s->n);
  s->ws_bytes = vpb_smpc_workspace_bytes(M, s->H, s->n);
  const size_t eps_bytes = (size_t)M * s->H * s->n * (s->dtype == VPB_DTYPE_F32 ? 4 : 8);
  int rc = VPB_OK;
#define SESSION_CUDA(call)                                                  \
  do {                                                                      \
    cudaError_t _e = (call);                                                \
    if (_e != cudaSuccess) {                                                \
      vpb::set_error("%s failed: %s", #call, cudaGetErrorString(_e));       \
      release(s);                                                           \
      return VPB_ERR_CUDA;                                                  \
    }                                                                       \
  } while (0)
  SESSION_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  SESSION_CUDA(cudaEventCreateWithFlags(&s->launched, cudaEventDisableTiming));
  SESSION_CUDA(cudaMallocHost(&s->h_in, (size_t)s->in_len * 8));
  SESSION_CUDA(cudaMallocHost(&s->h_out, (size_t)(s->out_len + 1) * 8));  // + the kernel's done flag
  SESSION_CUDA(cudaMalloc(&s->d_in, (size_t)s->in_len * 8));
  SESSION_CUDA(cudaMalloc(&s->d_out, (size_t)s->out_len * 8));
  SESSION_CUDA(cudaMalloc(&s->eps, eps_bytes));
  SESSION_CUDA(cudaMalloc(&s->ws, s->ws_bytes));
  // The warm-up below runs on the session's non-blocking stream: it must not
  // overtake the zeroing of its counters nor the field still being built on
  // the caller's streams (a warm-up on unzeroed counters would spin forever
  // in the merge protocol).  Creation is rare: synchronise the device.
  SESSION_CUDA(cudaDeviceSynchronize());
  SESSION_CUDA(cudaMemsetAsync(s->ws, 0, s->ws_bytes, s->stream));  // counters: zero once, every launch returns them to zero
  memset(s->h_in, 0, (size_t)s->in_len * 8);
  // identity goal so the warm-up launch evaluates a regular pose
  s->h_in[2 * s->n + 0] = s->h_in[2 * s->n + 4] = s->h_in[2 * s->n + 8] = 1.0;
  const float *sq0 = s->field.sq;
  memcpy(s->h_in + s->dyn_len + 1, &sq0, sizeof(sq0));
  s->prob.dyn_state = s->d_in;
  s->prob.field_sq_dev = reinterpret_cast<const float *const *>(s->d_in + s->dyn_len + 1);
  // fused fp32 path: no per-call copy at all -- state, goal, seed, field
  // pointer and nominal ride in the step kernel's launch parameters
  rc = vpb::smpc_session_node(prob, field ? &s->field : nullptr, window, sigma, M, precision, s->eps, s->d_out,
                              s->h_out, s->ws, s->ws_bytes, &s->node);
  if (rc) {
    release(s);
    return rc;
  }
  if (s->node) {
    const double *h = s->h_in;
    vpb::smpc_session_node_patch(s->node, h, h + s->n, h + 2 * s->n, h + 2 * s->n + 9, nullptr, 0, s->field.sq);
    cudaGraph_t g = nullptr;
    SESSION_CUDA(cudaGraphCreate(&g, 0));
    const cudaError_t ae = cudaGraphAddKernelNode(&s->gnode, g, nullptr, 0, vpb::smpc_session_node_params(s->node));
    const cudaError_t ie = ae == cudaSuccess ? cudaGraphInstantiate(&s->exec, g, 0) : ae;
    cudaGraphDestroy(g);
    if (getenv("VPB_SESSION_DIRECT")) s->direct = true;
    if (ie != cudaSuccess) {
      cudaGetLastError();
      s->direct = true;
    }
    SESSION_CUDA(launch_node(s, s->stream, false));  // warm-up
    SESSION_CUDA(cudaStreamSynchronize(s->stream));
    *out = s;
    return VPB_OK;
  }
  // warm-up outside capture (kernel attributes), then capture the step
  SESSION_CUDA(cudaMemcpyAsync(s->d_in, s->h_in, (size_t)s->in_len * 8, cudaMemcpyHostToDevice, s->stream));
  if ((rc = enqueue(s, false))) {
    release(s);
    return rc;
  }
  SESSION_CUDA(cudaStreamSynchronize(s->stream));
  cudaGraph_t graph = nullptr;
  SESSION_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  rc = enqueue(s, true);
  const cudaError_t ce = cudaStreamEndCapture(s->stream, &graph);
  if (rc || ce != cudaSuccess) {
    if (!rc) vpb::set_error("stream capture failed: %s", cudaGetErrorString(ce));
    if (graph) cudaGraphDestroy(graph);
    release(s);
    return rc ? rc : VPB_ERR_CUDA;
  }
  const cudaError_t ie = cudaGraphInstantiate(&s->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    vpb::set_error("graph instantiation failed: %s", cudaGetErrorString(ie));
    release(s);
    return VPB_ERR_CUDA;
  }
#undef SESSION_CUDA
  *out = s;
  return VPB_OK;
}

int vpb_smpc_session_step(vpb_smpc_session *s, const double *q0, const double *qd0, const double *goal_r,
                          const double *goal_t, const double *nominal, uint64_t seed, const float *field_sq,
                          double *out, void *stream) {
  VPB_REQUIRE(s && q0 && qd0 && goal_r && goal_t && out, "null argument to vpb_smpc_session_step");
  if (s->inflight) {  // an asynchronous launch() may still read h_in and set the done flag
    VPB_CUDA(cudaEventSynchronize(s->launched));
    s->inflight = false;
  }
  const int64_t n = s->n;
  double *h = s->h_in;
  memcpy(h, q0, n * 8);
  memcpy(h + n, qd0, n * 8);
  memcpy(h + 2 * n, goal_r, 9 * 8);
  memcpy(h + 2 * n + 9, goal_t, 3 * 8);
  memcpy(h + s->dyn_len, &seed, 8);
  const float *sq = field_sq ? field_sq : s->field.sq;
  memcpy(h + s->dyn_len + 1, &sq, sizeof(sq));
  if (nominal)
    memcpy(h + s->dyn_len + 2, nominal, (size_t)s->H * n * 8);
  else
    memset(h + s->dyn_len + 2, 0, (size_t)s->H * n * 8);
  // replayed on the caller's stream (NULL = the legacy default stream, as
  // everywhere in this ABI): ordered after whatever produced the field
  cudaStream_t st = vpb::as_stream(stream);
  volatile uint64_t *done = reinterpret_cast<volatile uint64_t *>(s->h_out + s->out_len);
  *done = 0;  // the previous launch set it as its last action
  if (s->node) {
    vpb::smpc_session_node_patch(s->node, q0, qd0, goal_r, goal_t, nominal, seed, sq);
    VPB_CUDA(launch_node(s, st, true));
  } else {
    VPB_CUDA(cudaGraphLaunch(s->exec, st));
  }
  double e_pos = 0.0, e_ori = 0.0;  // host diagnostics while the step runs
  vpb_ee_errors(&s->prob, q0, goal_r, goal_t, &e_pos, &e_ori);
  // The kernel's last CTA writes the result into pinned memory and then the
  // done flag (system-scope release): spin on it instead of waking up from a
  // stream synchronisation; the stream is polled now and then so an error
  // (or a kernel variant without the flag) still ends the wait.
  // acquire: the payload loads below must not be satisfied before the flag
  // load (weakly ordered hosts, e.g. Grace)
  for (uint32_t spin = 1; __atomic_load_n(const_cast<const uint64_t *>(done), __ATOMIC_ACQUIRE) == 0; ++spin) {
    if ((spin & 255u) == 0u) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) {
        vpb::set_error("smpc session step: %s", cudaGetErrorString(q));
        return VPB_ERR_CUDA;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);  // also covers the stream-query exit
  vpb::note_launch(1);
  memcpy(out, s->h_out, (size_t)s->out_len * 8);
  const int64_t base = 2 * s->H * n + n;
  out[base + 11] = e_pos;
  out[base + 12] = e_ori;
  return VPB_OK;
}

int vpb_smpc_session_launch(vpb_smpc_session *s, void *stream) {
  VPB_REQUIRE(s, "null session");
  // (replays of this graph are ordered on the stream and none rewrites h_in,
  // so back-to-back launches need no wait; step() waits for the last one)
  cudaStream_t st = vpb::as_stream(stream);
  if (s->node) VPB_CUDA(launch_node(s, st, false));
  else VPB_CUDA(cudaGraphLaunch(s->exec, st));
  VPB_CUDA(cudaEventRecord(s->launched, st));
  s->inflight = true;
  vpb::note_launch(1);
  return VPB_OK;
}

int vpb_smpc_session_destroy(vpb_smpc_session *s) {
  release(s);
  return VPB_OK;
}

}  // extern "C"
