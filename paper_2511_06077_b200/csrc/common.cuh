// common.cuh -- shared device helpers of libstca (product path only; never used by oracle/).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

// STCA_DEBUG_SYNC builds: device-side invariant checks that trap with the failed condition (see
// mbar_wait in tc_ptx.cuh); compiled out otherwise.
#ifdef STCA_DEBUG_SYNC
#include <stdio.h>
#define STCA_DCHECK(cond)                                                                                  \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("STCA_DEBUG_SYNC check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)threadIdx.x);                                                           \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define STCA_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace stca {

typedef __nv_bfloat16 bf16;

// storage-type conversions (fp32 accumulation everywhere)
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename S> __device__ __forceinline__ S from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// programmatic dependent launch (launch_pdl): wait for the predecessor grid's results / let the
// successor grid be scheduled
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Device-side attention work item (host plan -> device), 48 bytes.
struct AttnItem {
  int64_t qrow0;     // first query row (row index into U / Y, = target*h + head)
  int64_t key0;      // first key row in the compacted X~ cache
  int64_t part_row;  // -1: single-chunk request (write normalised Y); else partial row of q=0
  int32_t nq;        // query rows in this item
  int32_t klen;      // keys in this item
  int32_t chunk;     // chunk index within the request
  int32_t pad;
};

// Split-K partial row (one query row of one key chunk), 16-byte aligned:
//   O^ = O / l, the chunk's normalised output, d elements of the storage type S (bf16 on the bf16
//   path, exactly what a single-chunk request writes to Y) | m (log2 domain, fp32) | l (fp32) | 8 pad
__host__ __device__ constexpr int part_row_bytes(int d, int elem_bytes) { return d * elem_bytes + 16; }

// Merge item: one multi-chunk request.
struct MergeItem {
  int64_t qrow0;     // first query row of the request
  int64_t part_row;  // partial row of (chunk 0, q = 0)
  int32_t rows;      // m_b * h
  int32_t nchunks;
};

}  // namespace stca
