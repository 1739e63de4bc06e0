// Shared helpers for the sm_100a kernels behind include/vpb200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstring>

#include "vpb200.h"

namespace vpb {

// Thread-local last-error message (vpb_last_error).
void set_error(const char *fmt, ...);
void note_launch(int n = 1);

inline int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return VPB_ERR_CUDA;
  }
  note_launch();
  return VPB_OK;
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__host__ __device__ __forceinline__ int64_t vmin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t vmax64(int64_t a, int64_t b) { return a > b ? a : b; }

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// Number of SMs of the current device (cached per process).
int sm_count();

// Programmatic dependent launch on the map update (masked pixels -> fuse;
// the EDT passes opt in via VPB_EDT_PDL): each kernel releases its dependent
// as soon as all of its CTAs run (pdl_release) and waits for its
// predecessor's completion and memory flush (pdl_wait) before touching
// global memory, so the next grid's launch and CTA rasterisation overlap the
// current grid's tail (fusion 31.7 -> 29.7 us).  pdl_wait is a no-op when the
// kernel was not launched with the attribute.  VPB_NO_PDL=1 turns it off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
  return launch_ex(pdl_enabled(), kern, grid, block, smem, st, static_cast<Args &&>(args)...);
}

// Session step (rollout.cu): counters pre-zeroed, result also written to a
// host-mapped buffer by the kernel (session.cu).
// The per-call block [stage_src, + stage_len) (host-mapped) reaches its
// device copy stage_dst either inside the fused kernel (block 0 copies it,
// the other CTAs wait on a flag: no copy node in the session graph) or, on
// the other paths, by a copy enqueued first.
int smpc_generate_session(const vpb_problem *prob, const vpb_field *field, const uint64_t *seed_dev, int64_t window,
                          const double *sigma, const double *nominal, int64_t M, int precision, void *eps_out,
                          double *out, double *out_host, void *workspace, size_t workspace_bytes,
                          cudaStream_t s, const double *stage_src, double *stage_dst, int64_t stage_len);

// Fused fp32 fixed-topology session step with the per-call state in the
// launch parameters (rollout.cu): built once, patched every step, launched as
// a graph kernel node.  *node stays null when the path does not apply.
struct SmpcNode;
int smpc_session_node(const vpb_problem *prob, const vpb_field *field, int64_t window, const double *sigma,
                      int64_t M, int precision, void *eps_out, double *out, double *out_host, void *workspace,
                      size_t workspace_bytes, SmpcNode **node);
void smpc_session_node_patch(SmpcNode *node, const double *q0, const double *qd0, const double *goal_r,
                             const double *goal_t, const double *nominal, uint64_t seed, const float *sq);
const cudaKernelNodeParams *smpc_session_node_params(const SmpcNode *node);
void smpc_session_node_free(SmpcNode *node);

}  // namespace vpb

#define VPB_REQUIRE(cond, ...)      \
  do {                              \
    if (!(cond)) {                  \
      ::vpb::set_error(__VA_ARGS__); \
      return VPB_ERR_ARG;           \
    }                               \
  } while (0)

#define VPB_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::vpb::set_error("%s failed: %s", #call, cudaGetErrorString(_e));      \
      return VPB_ERR_CUDA;                                                   \
    }                                                                        \
  } while (0)
