// Deterministic block / grid reductions used by every reducing kernel.
// Grid-wide results use the "last block finishes" pattern: each block writes
// its partial, the last block to arrive (atomic ticket) folds the partials in
// block order, so results are bitwise run-to-run reproducible (no float
// atomics anywhere in the library).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace dp {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
// butterfly sum: every lane gets the total
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// sum over the block; result valid in thread 0.  `sh` >= 32 doubles.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (NT > 32) {
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = (threadIdx.x < NT / 32) ? sh[threadIdx.x] : 0.0;
    if (wid == 0) v = warp_sum(v);
    __syncthreads();
  }
  return v;
}
template <int NT>
__device__ __forceinline__ double block_max(double v, double* sh) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (NT > 32) {
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = (threadIdx.x < NT / 32) ? sh[threadIdx.x] : 0.0;
    if (wid == 0) v = warp_max(v);
    __syncthreads();
  }
  return v;
}

// Call from all threads after the block's partials are stored by thread 0.
// Returns true in every thread of the last block to arrive.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  return s_last;
}

// In the last block: fold W partial columns (partial[b*W + k]) over blocks
// b in [0, nb) in a fixed order; result[k] in thread 0 returned via out[k]
// (shared memory, visible to all threads after the call).
template <int NT, int W>
__device__ __forceinline__ void fold_partials(const double* partial, int nb, double* out, double* sh, bool is_max = false) {
#pragma unroll
  for (int k = 0; k < W; ++k) {
    double v = is_max ? 0.0 : 0.0;
    for (int b = threadIdx.x; b < nb; b += NT) {
      double p = __ldcg(partial + (size_t)b * W + k);
      v = is_max ? fmax(v, p) : v + p;
    }
    v = is_max ? block_max<NT>(v, sh) : block_sum<NT>(v, sh);
    if (threadIdx.x == 0) out[k] = v;
    __syncthreads();
  }
}

// In the last block: nv sums over nb partials (partial[b*stride + i]); warp w
// folds values i = w, w + NT/32, ... with lanes striding over blocks, so the
// loads of all values are in flight together.  out[] in shared memory.
template <int NT>
__device__ __forceinline__ void fold_multi(const double* partial, int stride, int nb, int nv, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < nv; i += NT / 32) {
    double acc = 0.0;
    for (int b = lane; b < nb; b += 32) acc += __ldcg(partial + (size_t)b * stride + i);
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
  __syncthreads();
}

// TMA bulk copies (cp.async.bulk, global -> shared) completing on an
// mbarrier (transaction bytes), one elected lane per copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(mb)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mb))
               : "memory");
}

}  // namespace dp

// 256-bit global accesses (sm_100: one full 32-byte sector per lane)
__device__ __forceinline__ void ld256f(const float* p, float o[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
               : "l"(p));
}
__device__ __forceinline__ void st256f(float* p, const float v[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
