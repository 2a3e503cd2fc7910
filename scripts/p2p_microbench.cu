// Microbenchmark of NVLink peer stores on B200 (2 GPUs, one process):
//  1. per-kernel overhead of a graph of empty kernels;
//  2. put bandwidth GPU0 -> GPU1 for message sizes 8 B .. 64 MB with 8-byte
//     and 16-byte stores, with and without a system fence + flag at the end;
//  3. one-way latency: GPU0 stores data+flag, a spinning kernel on GPU1
//     answers with a flag (half round trip).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o p2p_microbench p2p_microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

__global__ void empty_kernel() {}

template <int W>  // bytes per store: 8 or 16
__global__ void put_kernel(const char* __restrict__ src, char* dst, size_t bytes, unsigned long long* flag,
                           unsigned int* count, unsigned long long value, int fence) {
  using V = typename std::conditional<W == 16, uint4, unsigned long long>::type;
  const size_t n = bytes / W;
  const V* s = reinterpret_cast<const V*>(src);
  V* d = reinterpret_cast<V*>(dst);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = s[i];
  if (!fence) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    if (fence == 1) {  // fence.sc.sys per CTA
      __threadfence_system();
      prev = atomicAdd(count, 1u);
    } else if (fence == 2) {  // fence.acq_rel.sys per CTA
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      prev = atomicAdd(count, 1u);
    } else {  // release at gpu scope per CTA; the last CTA releases at sys scope
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(count) : "memory");
    }
    if (prev + 1 == gridDim.x) {
      *count = 0;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
    }
  }
}

// The library's shape: each thread stores E 8-byte elements (lane-strided
// inside a warp's 32*E chunk), one completion flag per launch (mode 3).
template <int E>
__global__ void put_e_kernel(const unsigned long long* __restrict__ src, unsigned long long* dst, size_t n,
                             unsigned long long* flag, unsigned int* count, unsigned long long value) {
  const size_t warp_base = (blockIdx.x * (size_t)blockDim.x + (threadIdx.x & ~31u)) * E;
  const unsigned lane = threadIdx.x & 31;
  unsigned long long v[E];
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const size_t i = warp_base + lane + 32 * u;
    if (i < n) v[u] = src[i];
  }
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const size_t i = warp_base + lane + 32 * u;
    if (i < n) dst[i] = v[u];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(count) : "memory");
    if (prev + 1 == gridDim.x) {
      *count = 0;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
    }
  }
}

__global__ void spin_then_signal(const unsigned long long* my_flag, unsigned long long want,
                                 unsigned long long* peer_flag, unsigned long long value) {
  if (threadIdx.x != 0) return;
  unsigned long long v;
  do {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory");
  } while (v < want);
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flag), "l"(value) : "memory");
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("need 2 GPUs\n");
    return 0;
  }
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  const size_t maxb = size_t(64) << 20;
  char *src0, *dst1;
  unsigned long long *flag0, *flag1;
  unsigned int* cnt0;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&dst1, maxb));
  CK(cudaMalloc(&flag1, 4096));
  CK(cudaMemset(flag1, 0, 4096));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&src0, maxb));
  CK(cudaMemset(src0, 1, maxb));
  CK(cudaMalloc(&flag0, 4096));
  CK(cudaMemset(flag0, 0, 4096));
  CK(cudaMalloc(&cnt0, 4096));
  CK(cudaMemset(cnt0, 0, 4096));
  cudaStream_t s0;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));

  // 1. empty kernel chain in a graph
  {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    const int K = 200;
    CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < K; ++i) empty_kernel<<<1, 32, 0, s0>>>();
    CK(cudaStreamEndCapture(s0, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s0));
    CK(cudaStreamSynchronize(s0));
    CK(cudaEventRecord(a, s0));
    CK(cudaGraphLaunch(ge, s0));
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    std::printf("{\"test\": \"empty_kernel_graph\", \"us_per_kernel\": %.3f}\n", ms * 1e3 / K);
    // eager
    CK(cudaEventRecord(a, s0));
    for (int i = 0; i < K; ++i) empty_kernel<<<1, 32, 0, s0>>>();
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    std::printf("{\"test\": \"empty_kernel_eager\", \"us_per_kernel\": %.3f}\n", ms * 1e3 / K);
  }

  // 2. put bandwidth
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long seq = 0;
  for (size_t bytes = 2097152; bytes <= 2097152; bytes *= 4) {
    for (int w : {16}) {
      for (int fence : {0, 1, 2, 3}) {
        for (int grid_mode : {0}) {  // 0: 1 element per thread, 1: grid = 4 x SMs (grid-stride)
          const size_t elems = (bytes + w - 1) / w;
          int grid = grid_mode == 0 ? (int)std::min<size_t>((elems + 255) / 256, 1 << 20) : 4 * sms;
          if (grid < 1) grid = 1;
          const int reps = 20;
          cudaGraph_t g;
          cudaGraphExec_t ge;
          CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeGlobal));
          for (int r = 0; r < reps; ++r) {
            ++seq;
            if (w == 8)
              put_kernel<8><<<grid, 256, 0, s0>>>(src0, dst1, bytes < 8 ? 8 : bytes, flag1, cnt0, seq, fence);
            else
              put_kernel<16><<<grid, 256, 0, s0>>>(src0, dst1, bytes < 16 ? 16 : bytes, flag1, cnt0, seq, fence);
          }
          CK(cudaStreamEndCapture(s0, &g));
          CK(cudaGraphInstantiate(&ge, g, 0));
          CK(cudaGraphLaunch(ge, s0));
          CK(cudaStreamSynchronize(s0));
          CK(cudaEventRecord(a, s0));
          CK(cudaGraphLaunch(ge, s0));
          CK(cudaEventRecord(b, s0));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          const double us = ms * 1e3 / reps;
          std::printf("{\"test\": \"put\", \"bytes\": %zu, \"store_bytes\": %d, \"fence_flag\": %d, \"grid\": %d, "
                      "\"us\": %.3f, \"GBps\": %.1f}\n",
                      bytes, w, fence, grid, us, bytes / (us * 1e-6) / 1e9);
          CK(cudaGraphExecDestroy(ge));
          CK(cudaGraphDestroy(g));
        }
      }
    }
  }

  // 2b. the library's per-thread element count
  for (size_t bytes : {size_t(262144), size_t(2097152), size_t(8388608)}) {
    const size_t n = bytes / 8;
    for (int E : {1, 2, 4, 8}) {
      const int grid = (int)((n + 256 * E - 1) / (256 * E));
      const int reps = 20;
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeGlobal));
      for (int r = 0; r < reps; ++r) {
        ++seq;
        auto* sp = reinterpret_cast<const unsigned long long*>(src0);
        auto* dp = reinterpret_cast<unsigned long long*>(dst1);
        if (E == 1) put_e_kernel<1><<<grid, 256, 0, s0>>>(sp, dp, n, flag1, cnt0, seq);
        if (E == 2) put_e_kernel<2><<<grid, 256, 0, s0>>>(sp, dp, n, flag1, cnt0, seq);
        if (E == 4) put_e_kernel<4><<<grid, 256, 0, s0>>>(sp, dp, n, flag1, cnt0, seq);
        if (E == 8) put_e_kernel<8><<<grid, 256, 0, s0>>>(sp, dp, n, flag1, cnt0, seq);
      }
      CK(cudaStreamEndCapture(s0, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, s0));
      CK(cudaStreamSynchronize(s0));
      CK(cudaEventRecord(a, s0));
      CK(cudaGraphLaunch(ge, s0));
      CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      const double us = ms * 1e3 / reps;
      std::printf("{\"test\": \"put_e\", \"bytes\": %zu, \"elems_per_thread\": %d, \"grid\": %d, \"us\": %.3f, \"GBps\": %.1f}\n",
                  bytes, E, grid, us, bytes / (us * 1e-6) / 1e9);
      CK(cudaGraphExecDestroy(ge));
      CK(cudaGraphDestroy(g));
    }
  }

  // 3. flag ping-pong latency (spinning kernels on distinct GPUs)
  {
    cudaStream_t s1;
    CK(cudaSetDevice(1));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaSetDevice(0));
    CK(cudaMemset(flag0, 0, 4096));
    CK(cudaSetDevice(1));
    CK(cudaMemset(flag1, 0, 4096));
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(0));
    CK(cudaDeviceSynchronize());
    const int K = 200;
    // GPU1: for i: wait flag1 >= i, then flag0 = i.  GPU0: for i: flag1 = i, wait flag0 >= i.
    // One kernel per step per side, stream-ordered: measures flag RTT + kernel turnaround.
    CK(cudaSetDevice(1));
    for (int i = 1; i <= K; ++i) spin_then_signal<<<1, 32, 0, s1>>>(flag1 + 8, i, flag0 + 8, i);
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(a, s0));
    for (int i = 1; i <= K; ++i) spin_then_signal<<<1, 32, 0, s0>>>(flag0 + 8, i - 1, flag1 + 8, i);
    spin_then_signal<<<1, 32, 0, s0>>>(flag0 + 8, K, flag0 + 16, 1);
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    std::printf("{\"test\": \"flag_pingpong_kernel_per_step\", \"half_rtt_us\": %.3f}\n", ms * 1e3 / (2 * K));
    CK(cudaSetDevice(1));
    CK(cudaDeviceSynchronize());
  }
  std::printf("{\"test\": \"done\"}\n");
  return 0;
}
