// tma_store_probe.cu — standalone probe of the SM-side fp32 store rate on B200 (diagnostics
// for DESIGN.md §6, not part of the library): one persistent CTA per SM, W warps, each warp
// streams boxes of a [rows x cols] fp32 matrix with
//   mode 0: TMA bulk tensor stores from smem (S slots of box bytes per warp, SWIZZLE_NONE)
//   mode 1: coalesced st.global.v4 (each warp writes whole rows, 512 B per instruction)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_store_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int S>
__global__ void k_tma_store(const __grid_constant__ CUtensorMap tm, int box_c, int box_r, int tiles_c, int ntiles,
                            int per_chunk /*0 none, 1 sts, 2 sts+fence, 3 sts+fence per 2 chunks*/) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int box_bytes = box_c * box_r * 4;
  uint8_t* mine = smem + warp * S * box_bytes;
  for (int i = lane; i < S * box_bytes / 4; i += 32) reinterpret_cast<float*>(mine)[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  int k = 0;
  for (int t = blockIdx.x * nw + warp; t < ntiles; t += gridDim.x * nw, ++k) {
    uint8_t* slot = mine + (k % S) * box_bytes;
    if (per_chunk) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
      __syncwarp();
      float4* dst = reinterpret_cast<float4*>(slot);
      for (int i = lane; i < box_bytes / 16; i += 32) dst[i] = make_float4(1.f, 2.f, 3.f, (float)k);
      if (per_chunk == 2 || (per_chunk == 3 && (k & 1))) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    if (lane == 0) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
      const int x = (t % tiles_c) * box_c, y = (t / tiles_c) * box_r;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                   "r"(smem_u32(mine + (k % S) * box_bytes)), "r"(x), "r"(y)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// The GEMM epilogue's write order: CTA b takes tiles u = b, b+148, ... of 128x256 fp32
// (raster 0: m-fastest, 1: n-fastest); warp w (quadrant q = w&3, half h = w>>2) writes
// 32x16 boxes of rows 32q.. : order 0 = its own 128-column half left to right, order 1 =
// the quadrant's two warps interleaved (chunk 2i+h), order 2 = all 8 warps sweep the same
// 32-column window (rows 32w'.. where w' = w&3, column 16*(2i + h)).
template <int S>
__global__ void k_gemm_like(const __grid_constant__ CUtensorMap tm, int m_tiles, int n_tiles, int raster, int order) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, h = warp >> 2;
  uint8_t* mine = smem + warp * S * 2048;
  for (int i = lane; i < S * 512; i += 32) reinterpret_cast<float*>(mine)[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  int k = 0;
  for (int u = blockIdx.x; u < m_tiles * n_tiles; u += gridDim.x) {
    const int mt = raster ? u / n_tiles : u % m_tiles;
    const int nt = raster ? u % n_tiles : u / m_tiles;
    for (int i = 0; i < 8; ++i, ++k) {
      const int cb = order == 0 ? h * 128 + 16 * i : 16 * (2 * i + h);
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                     "r"(smem_u32(mine + (k % S) * 2048)), "r"(nt * 256 + cb), "r"(mt * 128 + 32 * q)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      __syncwarp();
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_stg(float4* out, size_t n4) {
  const float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) out[i] = v;
}

using PFN = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 32256, cols = 4096;
  const size_t bytes = (size_t)rows * cols * 4;
  float* d;
  cudaMalloc(&d, bytes);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  PFN enc = reinterpret_cast<PFN>(fn);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int i = 0; i < 10; ++i) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  printf("{\"probe\":\"stg_fill\",\"GBs\":%.1f}\n", timeit([&] { k_stg<<<148 * 4, 256>>>((float4*)d, bytes / 16); }));
  struct Cfg { int bc, br, warps, slots; };
  std::vector<Cfg> cfgs = {{16, 32, 8, 2}, {16, 32, 8, 4}, {32, 32, 8, 2}, {64, 32, 8, 2}};
  for (int pc = 0; pc < 1; ++pc)
  for (auto c : cfgs) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.bc, (cuuint32_t)c.br};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("{\"probe\":\"tma\",\"box\":[%d,%d],\"error\":\"encode\"}\n", c.bc, c.br);
      continue;
    }
    const int tiles_c = cols / c.bc, ntiles = tiles_c * (rows / c.br);
    const size_t smem = (size_t)c.warps * c.slots * c.bc * c.br * 4;
    auto run = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      return timeit([&] { kern<<<148, c.warps * 32, smem>>>(tm, c.bc, c.br, tiles_c, ntiles, pc); });
    };
    double g = c.slots == 2 ? run(k_tma_store<2>) : run(k_tma_store<4>);
    cudaError_t e = cudaGetLastError();
    printf("{\"probe\":\"tma\",\"per_chunk\":%d,\"box\":[%d,%d],\"warps\":%d,\"slots\":%d,\"GBs\":%.1f,\"err\":\"%s\"}\n",
           pc, c.bc, c.br, c.warps, c.slots, g, cudaGetErrorString(e));
  }
  {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {16, 32};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_gemm_like<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int raster = 0; raster < 2; ++raster)
      for (int order = 0; order < 2; ++order) {
        double g = timeit([&] { k_gemm_like<2><<<148, 256, 32768>>>(tm, rows / 128, cols / 256, raster, order); });
        printf("{\"probe\":\"gemm_like\",\"raster\":%d,\"order\":%d,\"GBs\":%.1f,\"err\":\"%s\"}\n", raster, order, g,
               cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
