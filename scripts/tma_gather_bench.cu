// Config 1 gather (leaf[i] = root[idx[i]], 4,194,304 leaves, 1,048,576 f64
// roots) through the Blackwell TMA row gather (cp.async.bulk.tensor.2d ...
// tile::gather4) instead of LSU loads: the roots are viewed as a 2-D tensor of
// 16-byte rows (2 roots per row); one instruction fetches 4 rows into shared
// memory (32-byte rows of 4 roots: one 128-byte aligned slot per gather4),
// completion on an mbarrier; the CTA then picks each leaf's half of
// its row and stores the tile coalesced. Compared with the LSU gather on the
// same data (cold L2: 256 MB read-flush before every call).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_gather_bench tma_gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

constexpr int kT = 1024;     // leaves per tile
constexpr int kStages = 4;   // tiles in flight per CTA
constexpr int kThr = 128;    // 4 warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(kThr) gather_tma(const __grid_constant__ CUtensorMap tmap, const int* __restrict__ idx,
                                                   double* __restrict__ leaf, long long L) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* rows = reinterpret_cast<uint64_t*>(smem);                   // kStages x kT x 4 words
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kStages * kT * 32);  // kStages mbarriers
  const long long ntiles = (L + kT - 1) / kT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kStages) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + tid)));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const uint64_t tdesc = reinterpret_cast<uint64_t>(&tmap);
  // producer: warp 0; lane l issues the 8 gather4 of rows l*32 .. l*32+31
  auto issue = [&](long long t, int st) {
    if (warp != 0) return;
    // the stage's earlier generic-proxy reads are ordered before the async
    // proxy's writes into it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t b = smem_u32(bar + st);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kT * 32) : "memory");
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long long i0 = t * kT + q * 128 + lane * 4;  // 4 rows per lane, coalesced 16-byte index loads
      int r[4];
      if (i0 + 3 < L) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(idx + i0));
        r[0] = v.x >> 2; r[1] = v.y >> 2; r[2] = v.z >> 2; r[3] = v.w >> 2;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) r[u] = i0 + u < L ? (__ldg(idx + i0 + u) >> 2) : 0;
      }
      const uint32_t dst = smem_u32(rows + (size_t(st) * kT + q * 128 + lane * 4) * 4);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(tdesc), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(b)
          : "memory");
    }
  };
  long long t0 = blockIdx.x;
  const long long step = gridDim.x;
  int k = 0;
  for (int s = 0; s < kStages; ++s)
    if (t0 + s * step < ntiles) issue(t0 + s * step, s);
  uint32_t phase[kStages] = {0, 0, 0, 0};
  for (long long t = t0; t < ntiles; t += step, ++k) {
    const int st = k % kStages;
    const uint32_t b = smem_u32(bar + st);
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(b), "r"(phase[st])
          : "memory");
    phase[st] ^= 1u;
    const uint64_t* tile = rows + size_t(st) * kT * 4;
#pragma unroll
    for (int j = 0; j < kT / kThr; ++j) {
      const int e = j * kThr + tid;
      const long long i = t * kT + e;
      if (i < L) {
        const int q4 = __ldg(idx + i) & 3;
        leaf[i] = __longlong_as_double(static_cast<long long>(tile[e * 4 + q4]));
      }
    }
    __syncthreads();  // stage st consumed
    const long long tn = t + kStages * step;
    if (tn < ntiles) issue(tn, st);
  }
}

__global__ void __launch_bounds__(256, 4) gather_elem(const double* __restrict__ root, const int* __restrict__ idx,
                                                     double* __restrict__ leaf, long long L) {
  const long long base = blockIdx.x * 2048ll + threadIdx.x;
  double v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const long long i = base + u * 256;
    if (i < L) v[u] = root[__ldg(idx + i)];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const long long i = base + u * 256;
    if (i < L) leaf[i] = v[u];
  }
}

__global__ void flush_read(const double4* p, long long n, double* sink) {
  double a = 0;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (long long)gridDim.x * 256) a += p[i].x;
  if (a == 1.2345) *sink = a;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long L = 4194304;
  const int R = 1048576;
  uint64_t s = 12345;
  auto nx = [&]() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  std::vector<int> idx(L);
  for (auto& v : idx) v = static_cast<int>(nx() % R);
  std::vector<double> root(R);
  for (auto& v : root) v = static_cast<double>(nx() >> 11) * 0x1.0p-53;
  double *droot, *dleaf, *sink;
  int* didx;
  double4* flush;
  const long long nf = (256ll << 20) / 32;
  CK(cudaMalloc(&droot, R * 8ll));
  CK(cudaMalloc(&dleaf, L * 8));
  CK(cudaMalloc(&didx, L * 4));
  CK(cudaMalloc(&flush, nf * 32));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(flush, 0, nf * 32));
  CK(cudaMemcpy(droot, root.data(), R * 8ll, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(didx, idx.data(), L * 4, cudaMemcpyHostToDevice));
  EncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  CUtensorMap tmap;
  const cuuint64_t gdim[2] = {4, static_cast<cuuint64_t>(R / 4)};
  const cuuint64_t gstride[1] = {32};
  const cuuint32_t box[2] = {4, 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, droot, gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    std::printf("{\"error\":\"cuTensorMapEncodeTiled %d\"}\n", static_cast<int>(cr));
    return 1;
  }
  const size_t smem = kStages * kT * 32 + kStages * 8;
  CK(cudaFuncSetAttribute(gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  std::vector<double> got(L);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto&& f) {
    std::vector<float> t;
    for (int i = 0; i < 22; ++i) {
      flush_read<<<148 * 8, 256>>>(flush, nf, sink);
      CK(cudaEventRecord(e0));
      f();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (i >= 2) t.push_back(ms * 1000.f);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
  };
  auto check = [&]() {
    CK(cudaMemcpy(got.data(), dleaf, L * 8, cudaMemcpyDeviceToHost));
    for (long long i = 0; i < L; ++i)
      if (got[i] != root[idx[i]]) return false;
    return true;
  };
  CK(cudaMemset(dleaf, 0, L * 8));
  float us = timeit([&] { gather_elem<<<(L + 2047) / 2048, 256>>>(droot, didx, dleaf, L); });
  std::printf("{\"kernel\":\"lsu_elem8\",\"us\":%.2f,\"ok\":%s}\n", us, check() ? "true" : "false");
  for (int per_sm : {1}) {
    CK(cudaMemset(dleaf, 0, L * 8));
    us = timeit([&] { gather_tma<<<148 * per_sm, kThr, smem>>>(tmap, didx, dleaf, L); });
    CK(cudaGetLastError());
    std::printf("{\"kernel\":\"tma_gather4_x%d\",\"us\":%.2f,\"ok\":%s}\n", per_sm, us, check() ? "true" : "false");
  }
  return 0;
}
