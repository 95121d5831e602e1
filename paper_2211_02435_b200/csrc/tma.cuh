// tma.cuh — Tensor Memory Accelerator (cp.async.bulk.tensor) and mbarrier helpers for sm_100a.
//
// The population grid [zz][i][y][x] (kernels.cuh layout) is described to the TMA unit as a 4D
// tensor {x: nx, y: ny, i: Q, zz: planes} with byte strides {pitch, pop, plane} x sizeof(real);
// a box {BX, HY, 1, 1} is one population's (TX + 2) x (TY + 2) halo-extended tile of one plane.
// Out-of-range box elements (the periodic wrap at the x / y faces) are zero-filled by the
// hardware and patched by the kernel.
#pragma once
#include <cuda.h>  // CUtensorMap and the cuTensorMapEncodeTiled prototype (the driver entry
                   // point is fetched at run time through cudaGetDriverEntryPoint: no -lcuda)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

namespace lbm {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make the initialised barriers visible to the async proxy (TMA) before first use
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// blocks until the phase with the given parity has completed
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// plain arrival (release.cta): the phase completes when the init count of threads arrived
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// cp.async (LDGSTS): an 4/8-byte global -> shared copy that completes asynchronously, tracked
// per thread by commit / wait groups (no register holds the data in flight)
template <class real>
__device__ __forceinline__ void cp_async(real *dst_smem, const real *src) {
  static_assert(sizeof(real) == 4 || sizeof(real) == 8, "4 or 8 byte elements");
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst_smem)), "l"(src),
               "n"((int)sizeof(real))
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// order this thread's earlier generic-proxy shared-memory accesses before later async-proxy
// (TMA) writes to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// one 4D box of the tensor map into shared memory; completion is signalled on `bar` as
// transaction bytes
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// Host: the tensor map of one population grid (base = element (zz = 0, i = 0, y = 0, x = 0)),
// box {bx, by, 1, 1}.  Returns cudaSuccess or the error of the entry-point lookup / encoding.
template <class real>
inline cudaError_t encode_grid_tmap(CUtensorMap *map, const void *base, int nx, int ny, int q, long long planes,
                                    long long pitch, long long pop, long long plane, int bx, int by) {
  using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q_ = cudaDriverEntryPointSymbolNotFound;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q_);
    if (e != cudaSuccess) return e;
    if (!fn || q_ != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)q, (cuuint64_t)planes};
  const cuuint64_t strides[3] = {(cuuint64_t)(pitch * sizeof(real)), (cuuint64_t)(pop * sizeof(real)),
                                 (cuuint64_t)(plane * sizeof(real))};
  const cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, 1u, 1u};
  const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  const CUresult r = encode(map, sizeof(real) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                            4, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, (getenv("LBM_TMA_L2NONE") ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B),
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace lbm
