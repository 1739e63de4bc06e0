// Library-wide state: error strings, launch counter, device properties.
#include <cstdarg>

#include "vpb_common.cuh"

namespace vpb {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
  }
  return cached;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("VPB_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

}  // namespace vpb

extern "C" {

int vpb_version(void) { return 1; }

const char *vpb_last_error(void) { return vpb::g_err; }

uint64_t vpb_launch_count(void) { return vpb::g_launches.load(); }

int vpb_stage_h2d(void *dst_dev, void *pinned, const void *src_host, int64_t bytes, void *stream) {
  VPB_REQUIRE(bytes >= 0 && (bytes == 0 || (dst_dev && pinned && src_host)), "bad vpb_stage_h2d arguments");
  if (bytes == 0) return VPB_OK;
  memcpy(pinned, src_host, (size_t)bytes);
  VPB_CUDA(cudaMemcpyAsync(dst_dev, pinned, (size_t)bytes, cudaMemcpyHostToDevice, vpb::as_stream(stream)));
  return VPB_OK;
}

}  // extern "C"
