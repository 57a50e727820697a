// copy_micro.cu -- measurement only (not part of the library): memory pipelines for the tile
// kernel's access pattern.  x = b over an (n x m) fp64 matrix (row stride m), processed in tiles
// of 32 columns x 256 rows (256-byte row segments, 512 KiB apart for the cfg2 shape), the way
// k_tile streams the slab.  Variants:
//   ldg   each thread loads its 32-row chunk of one column with LDG (all in flight), then STG
//   tma1  TMA load of the tile into a 1-slot smem ring, LDS, STG (k_tile's copy-only mode)
//   tma2  the same with a 2-slot ring (next tile's load issued before this tile's stores)
//   bulk  TMA load into a slot, TMA store from the same slot (no LSU), `slots` in flight
//   d2d   cudaMemcpyAsync of the whole contiguous buffer (reference)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/copy_micro.cu -o /tmp/copy_micro -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                      \
    }                                                                                    \
  } while (0)

constexpr int TC = 32, TR = 256;  // tile: 32 columns x 256 rows

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
               ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* m, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(reinterpret_cast<uint64_t>(m)), "r"(src), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void stcs(double* p, double v) { asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }

// ---- ldg: registers only ----
__global__ void __launch_bounds__(256, 2) k_ldg(const double* __restrict__ b, double* __restrict__ x, long n, long m) {
  const long tiles_c = m / TC, ntiles = tiles_c * (n / TR);
  const int j = threadIdx.x % TC, cl = threadIdx.x / TC;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long r0 = (t / tiles_c) * TR + cl * 32, c0 = (t % tiles_c) * TC + j;
    const double* bp = b + r0 * m + c0;
    double* xp = x + r0 * m + c0;
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __ldcs(bp + k * m);
#pragma unroll
    for (int k = 0; k < 32; ++k) stcs(xp + k * m, v[k]);
  }
}

// ---- tma + LDS/STG, SLOTS-deep ring ----
template <int SLOTS>
__global__ void __launch_bounds__(256, 2) k_tma(const __grid_constant__ CUtensorMap mb, double* __restrict__ x, long n, long m) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* ring = reinterpret_cast<double*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + SLOTS * TC * TR);
  const long tiles_c = m / TC, ntiles = tiles_c * (n / TR);
  const int tid = threadIdx.x, j = tid % TC, cl = tid / TC;
  if (tid < SLOTS) mbar_init(smem_u32(bar + tid), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const uint64_t pol = pol_first();
  auto issue = [&](long it) {
    const long t = blockIdx.x + it * gridDim.x;
    if (t >= ntiles) return;
    const int s = (int)(it % SLOTS);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(smem_u32(bar + s), TC * TR * 8);
    tma_load(smem_u32(ring + s * TC * TR), &mb, (int)((t % tiles_c) * TC), (int)((t / tiles_c) * TR), smem_u32(bar + s), pol);
  };
  if (tid == 0)
    for (int s = 0; s < SLOTS; ++s) issue(s);
  long it = 0;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = (int)(it % SLOTS);
    mbar_wait(smem_u32(bar + s), (uint32_t)((it / SLOTS) & 1));
    const double* tile = ring + s * TC * TR;
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = tile[(cl * 32 + k) * TC + j];
    __syncthreads();
    if (tid == 0) issue(it + SLOTS);
    const long r0 = (t / tiles_c) * TR + cl * 32, c0 = (t % tiles_c) * TC + j;
    double* xp = x + r0 * m + c0;
#pragma unroll
    for (int k = 0; k < 32; ++k) stcs(xp + k * m, v[k]);
  }
}

// ---- bulk: TMA load -> smem -> TMA store, SLOTS tiles of BC columns x BR rows in flight ----
template <int SLOTS, int BC = TC, int BR = TR>
__global__ void __launch_bounds__(32, 1) k_bulk(const __grid_constant__ CUtensorMap mb, const __grid_constant__ CUtensorMap mx, long n, long m) {
  constexpr int TC = BC, TR = BR;
  extern __shared__ __align__(128) unsigned char sm[];
  double* ring = reinterpret_cast<double*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + SLOTS * TC * TR);
  const long tiles_c = m / TC, ntiles = tiles_c * (n / TR);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < SLOTS; ++s) mbar_init(smem_u32(bar + s), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t pol = pol_first();
  auto issue = [&](long it) {
    const long t = blockIdx.x + it * gridDim.x;
    if (t >= ntiles) return;
    const int s = (int)(it % SLOTS);
    mbar_expect_tx(smem_u32(bar + s), TC * TR * 8);
    tma_load(smem_u32(ring + s * TC * TR), &mb, (int)((t % tiles_c) * TC), (int)((t / tiles_c) * TR), smem_u32(bar + s), pol);
  };
  for (int s = 0; s < SLOTS; ++s) issue(s);
  long it = 0;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = (int)(it % SLOTS);
    mbar_wait(smem_u32(bar + s), (uint32_t)((it / SLOTS) & 1));
    tma_store(&mx, smem_u32(ring + s * TC * TR), (int)((t % tiles_c) * TC), (int)((t / tiles_c) * TR));
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the slot is reloaded once its store has read it: keep SLOTS-1 stores in flight
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(SLOTS - 1) : "memory");
    issue(it + SLOTS);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncFn enc, double* p, long n, long m, int bc = TC, int br = TR) {
  CUtensorMap t;
  cuuint64_t gd[2] = {(cuuint64_t)m, (cuuint64_t)n};
  cuuint64_t gs[1] = {(cuuint64_t)m * 8};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br}, es[2] = {1, 1};
  if (enc(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, p, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    std::printf("tensor map failed\n");
    std::exit(1);
  }
  return t;
}

template <class F>
static double timeit(F f, int reps = 30) {
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 8192, m = argc > 2 ? atol(argv[2]) : 65536;
  const double gb = 2.0 * n * m * 8 / 1e9;
  double *b, *x;
  CK(cudaMalloc(&b, n * m * 8));
  CK(cudaMalloc(&x, n * m * 8));
  CK(cudaMemset(b, 0, n * m * 8));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = reinterpret_cast<EncFn>(fp);
  CUtensorMap mb = make_map(enc, b, n, m), mx = make_map(enc, x, n, m);
  auto rep = [&](const char* name, double ms) { std::printf("%-22s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, gb / ms * 1e3); };
  rep("d2d memcpy", timeit([&] { cudaMemcpyAsync(x, b, n * m * 8, cudaMemcpyDeviceToDevice); }));
  for (int cps : {2, 3, 4}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "ldg %d CTA/SM", cps);
    rep(nm, timeit([&] { k_ldg<<<sms * cps, 256>>>(b, x, n, m); }));
  }
  {
    const int sm1 = TC * TR * 8 + 64, sm2 = 2 * TC * TR * 8 + 64;
    CK(cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1));
    CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
    rep("tma1 2 CTA/SM", timeit([&] { k_tma<1><<<sms * 2, 256, sm1>>>(mb, x, n, m); }));
    rep("tma1 3 CTA/SM", timeit([&] { k_tma<1><<<sms * 3, 256, sm1>>>(mb, x, n, m); }));
    rep("tma2 1 CTA/SM", timeit([&] { k_tma<2><<<sms, 256, sm2>>>(mb, x, n, m); }));
  }
  {
    const int s2 = 2 * TC * TR * 8 + 64, s3 = 3 * TC * TR * 8 + 64;
    CK(cudaFuncSetAttribute(k_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
    CK(cudaFuncSetAttribute(k_bulk<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3));
    rep("bulk 2 slots x1", timeit([&] { k_bulk<2><<<sms, 32, s2>>>(mb, mx, n, m); }));
    rep("bulk 3 slots x1", timeit([&] { k_bulk<3><<<sms, 32, s3>>>(mb, mx, n, m); }));
    CUtensorMap mb64 = make_map(enc, b, n, m, 64, 128), mx64 = make_map(enc, x, n, m, 64, 128);
    CUtensorMap mb128 = make_map(enc, b, n, m, 128, 64), mx128 = make_map(enc, x, n, m, 128, 64);
    CUtensorMap mb16 = make_map(enc, b, n, m, 16, 256), mx16 = make_map(enc, x, n, m, 16, 256);
    CK(cudaFuncSetAttribute(k_bulk<2, 64, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
    CK(cudaFuncSetAttribute(k_bulk<2, 128, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
    CK(cudaFuncSetAttribute(k_bulk<2, 16, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
    rep("bulk 512B rows", timeit([&] { k_bulk<2, 64, 128><<<sms, 32, s2>>>(mb64, mx64, n, m); }));
    rep("bulk 1KB rows", timeit([&] { k_bulk<2, 128, 64><<<sms, 32, s2>>>(mb128, mx128, n, m); }));
    rep("bulk 128B rows", timeit([&] { k_bulk<2, 16, 256><<<sms, 32, s2>>>(mb16, mx16, n, m); }));
    rep("bulk 256B x2 CTA/SM", timeit([&] { k_bulk<2><<<2 * sms, 32, s2>>>(mb, mx, n, m); }));
  }
  CK(cudaGetLastError());
  return 0;
}
