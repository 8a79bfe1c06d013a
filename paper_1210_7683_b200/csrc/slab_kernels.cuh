// slab_kernels.cuh — small HBM-bound kernels around the grid: int8 genotype
// slabs in (GWG_FORMAT_I8) and the order-independent result checksum out.
//
// * i8_pack_kernel: int8 codes as the caller stores them (n x cols,
//   column-major, ld n) -> the int8 tensor-core operand layout [SNP][kp]
//   (zero padded to kp), flagging -128 (the exact int32 slice products assume
//   |code| <= 127).  1 byte per code each way.
// * i8_unpack_kernel: the same codes -> FP64 raw slab (ld ldd) for the FP64
//   path (GWG_SNP_REAL, or n beyond the exact-int8 bound).
// * checksum_kernel: wrapping uint64 sum over a slab-local result buffer of
//   cell_hash(i, j, c, bits(b_ijc)) with global SNP index i — a sum of
//   per-component terms, so it is the same for any slab width, layout, shard
//   split or GPU count (the analogue of the reference's byte-identical output
//   guarantee, proj/include/gwgrid/grid.hpp:35-38, checked without moving the
//   3.2 TB of config 3 through one host).  Reads 8 B per component.
#pragma once

#include <cstdint>

namespace gwg {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// key of cell (i, j); one component's term is mix64((key + c*K3) ^ bits)
__host__ __device__ __forceinline__ uint64_t cell_key(uint64_t i, uint64_t j) {
  return mix64(i * 0xD1B54A32D192ED03ull + j * 0xA24BAED4963EE407ull);
}
__host__ __device__ __forceinline__ uint64_t cell_term(uint64_t key, uint64_t c, uint64_t bits) {
  return mix64((key + c * 0x9FB21C651E98DF25ull) ^ bits);
}

__global__ void __launch_bounds__(256) i8_pack_kernel(const int8_t* __restrict__ x, int32_t n,
                                                      int32_t cols, int32_t kp,
                                                      int8_t* __restrict__ out,
                                                      unsigned long long* __restrict__ bad) {
  bool ok = true;
  for (int c = blockIdx.x; c < cols; c += gridDim.x) {
    const int8_t* col = x + int64_t(c) * n;
    int8_t* dst = out + int64_t(c) * kp;
    if ((n & 3) == 0) {  // 4 codes per load (the column start is 4-byte aligned)
      const int words = kp >> 2, nw = n >> 2;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(col);
      uint32_t* d = reinterpret_cast<uint32_t*>(dst);
      for (int w = threadIdx.x; w < words; w += blockDim.x) {
        const uint32_t v = w < nw ? __ldcs(reinterpret_cast<const unsigned int*>(src) + w) : 0u;
        // a byte equal to 0x80 (-128)
        const uint32_t y = v ^ 0x80808080u;
        ok &= ((y - 0x01010101u) & ~y & 0x80808080u) == 0u;
        d[w] = v;
      }
    } else {
      for (int k = threadIdx.x; k < kp; k += blockDim.x) {
        const int8_t v = k < n ? col[k] : int8_t(0);
        ok &= v != int8_t(-128);
        dst[k] = v;
      }
    }
  }
  if (!ok) *bad = 0;  // error words are reset to all ones
}

__global__ void __launch_bounds__(256) i8_unpack_kernel(const int8_t* __restrict__ x, int32_t n,
                                                        int32_t cols, double* __restrict__ out,
                                                        int64_t ldd) {
  for (int c = blockIdx.x; c < cols; c += gridDim.x) {
    const int8_t* col = x + int64_t(c) * n;
    double* dst = out + int64_t(c) * ldd;
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = double(col[k]);
  }
}

// Cells of a slab-local result buffer: cell (o, q) at (o * inner + q) * p.
// NUMPY layout: o = il (SNP), q = j; STREAM: o = j, q = il.
__global__ void __launch_bounds__(256) checksum_kernel(const double* __restrict__ out,
                                                       int64_t outer, int64_t inner, int32_t p,
                                                       int32_t numpy, int64_t i0,
                                                       unsigned long long* __restrict__ acc) {
  uint64_t sum = 0;
  for (int64_t o = blockIdx.x; o < outer; o += gridDim.x) {
    const double* row = out + o * inner * p;
    for (int64_t q = threadIdx.x; q < inner; q += blockDim.x) {
      const uint64_t i = uint64_t(i0 + (numpy ? o : q));
      const uint64_t j = uint64_t(numpy ? q : o);
      const uint64_t key = cell_key(i, j);
      const double* cell = row + q * p;
      for (int c = 0; c < p; ++c)
        sum += cell_term(key, uint64_t(c), uint64_t(__double_as_longlong(__ldcs(cell + c))));
    }
  }
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if ((threadIdx.x & 31) == 0 && sum) atomicAdd(acc, (unsigned long long)sum);
}

}  // namespace gwg
