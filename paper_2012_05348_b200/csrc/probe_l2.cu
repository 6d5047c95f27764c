// probe_l2.cu — measurement utility, not part of the hot path: the L2 read
// bandwidth that bench.py's L2 roofline divides by ("L2 peak:
// unknown, so measure it"; the D5 row of §2.5).
//
// An L2-resident buffer, sized as a fraction of cudaDevAttrL2CacheSize, is
// streamed `reps` times with 16-byte ld.global.cg loads (cached in L2, not in
// L1) by a grid of SMs x 8 CTAs of 256 threads; GB/s = bytes read / the
// CUDA-event time of the timed passes.  The probe tries a few buffer sizes
// and reports the best, with the size it came from.  It allocates its own
// device memory (unlike the library's query calls).
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdio>

namespace {

__global__ void __launch_bounds__(256) l2_stream(const float4* __restrict__ p, size_t n, int reps, float* sink) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    // four independent 16-B loads in flight per thread per step
    for (; i + 3 * stride < n; i += 4 * stride) {
      const float4 a = __ldcg(p + i), b = __ldcg(p + i + stride);
      const float4 c = __ldcg(p + i + 2 * stride), d = __ldcg(p + i + 3 * stride);
      acc += (a.x + a.w) + (b.y + b.z) + (c.x + c.w) + (d.y + d.z);
    }
    for (; i < n; i += stride) {
      const float4 a = __ldcg(p + i);
      acc += a.x + a.w;
    }
  }
  if (acc == 1.2345e-30f) sink[0] = acc;  // keeps the loads alive; never true for the zero-filled buffer
}

__global__ void fill(float4* p, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

}  // namespace

extern "C" {

// Best L2 read bandwidth (GB/s, 1e9 B/s) over buffer sizes of 1/8, 1/4 and
// 1/2 of the L2; *bytes = the buffer size it was measured on, *l2 = the L2
// size reported by the device.  Returns 0 on success, -1 on a CUDA error
// (message in msg, if non-null, up to 256 bytes).
int cbvh_probe_l2_read_gbs(double* gbs, size_t* bytes, size_t* l2, char* msg) {
  int dev = 0, l2b = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&l2b, cudaDevAttrL2CacheSize, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) {
    if (msg) std::snprintf(msg, 256, "%s", cudaGetErrorString(e));
    return -1;
  }
  const size_t cap = (size_t)l2b / 2;
  float4* buf = nullptr;
  float* sink = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  double best = 0.0;
  size_t best_bytes = 0;
  e = cudaMalloc(&buf, cap);
  if (e == cudaSuccess) e = cudaMalloc(&sink, 64);
  if (e == cudaSuccess) e = cudaEventCreate(&t0);
  if (e == cudaSuccess) e = cudaEventCreate(&t1);
  for (int div = 8; e == cudaSuccess && div >= 2; div /= 2) {
    const size_t nb = (size_t)l2b / div, n = nb / sizeof(float4);
    const int reps = 64;
    fill<<<sms * 4, 256>>>(buf, n);
    for (int w = 0; w < 2; ++w) l2_stream<<<sms * 8, 256>>>(buf, n, 2, sink);  // warm L2
    for (int trial = 0; trial < 3 && e == cudaSuccess; ++trial) {
      cudaEventRecord(t0);
      l2_stream<<<sms * 8, 256>>>(buf, n, reps, sink);
      cudaEventRecord(t1);
      e = cudaEventSynchronize(t1);
      float ms = 0.f;
      if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, t0, t1);
      if (e == cudaSuccess && ms > 0.f) {
        const double g = (double)nb * reps / (ms * 1e-3) / 1e9;
        if (g > best) { best = g; best_bytes = nb; }
      }
    }
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (t0) cudaEventDestroy(t0);
  if (t1) cudaEventDestroy(t1);
  if (sink) cudaFree(sink);
  if (buf) cudaFree(buf);
  if (e != cudaSuccess) {
    if (msg) std::snprintf(msg, 256, "%s", cudaGetErrorString(e));
    return -1;
  }
  *gbs = best;
  *bytes = best_bytes;
  *l2 = (size_t)l2b;
  return 0;
}

}  // extern "C"
