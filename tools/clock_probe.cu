// clock_probe.cu — measurement tool (not product code): one warp on one SM
// samples (globaltimer ns, clock64 cycles) at a fixed interval while other
// kernels run on the same SM, so the SM clock DURING those kernels can be read
// off as d(clock64)/d(globaltimer).  Built by tools/kernel_clock_probe.py's
// recipe (nvcc -shared) into tools/libclock_probe.so.
#include <cuda_runtime.h>

#include <cstdint>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe_kernel(unsigned long long* out, int n, unsigned interval_ns) {
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = gtime();
  for (int i = 0; i < n; ++i) {
    const unsigned long long due = t0 + static_cast<unsigned long long>(i) * interval_ns;
    unsigned long long t;
    while ((t = gtime()) < due) __nanosleep(200);
    out[2 * i] = t;
    out[2 * i + 1] = static_cast<unsigned long long>(clock64());
  }
}

__global__ void stamp_kernel(unsigned long long* out) {
  if (threadIdx.x == 0) out[0] = gtime();
}

extern "C" int clock_probe_launch(void* stream, unsigned long long* out, int n, unsigned interval_ns) {
  // the SM keeps the large-shared-memory configuration the persistent kernels
  // need, so their CTA can stay co-resident with this warp
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       static_cast<int>(cudaSharedmemCarveoutMaxShared));
  probe_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(out, n, interval_ns);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int clock_stamp_launch(void* stream, unsigned long long* out) {
  stamp_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(out);
  return static_cast<int>(cudaGetLastError());
}
