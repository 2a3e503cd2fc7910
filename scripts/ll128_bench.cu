// NVLink exchange microbenchmark on 2 B200s (one process, peer access):
// the p2p Bcast shape — every GPU puts a message into the peer's staging and
// unpacks the peer's message into its own destination, ONE launch per
// exchange per GPU, K exchanges captured in a CUDA graph per GPU.
//
//   proto 0 "flag":  8-byte stores into the peer, GPU-scope CTA arrival + one
//                    st.release.sys message flag; receiver CTAs ld.acquire.sys
//                    the flag, then copy (round-1 library protocol).
//   proto 1 "ll128": 128-byte lines of 15 data words + 1 flag word (message
//                    number), written with one 16-byte store per lane (8 lanes
//                    per line, NCCL's LL128 layout); no fence, no message flag:
//                    receiver warps poll each line's flag word and unpack the
//                    line as soon as it is valid. Staging double-buffered by
//                    message parity; the credit (receiver consumed message
//                    m-2) is a relaxed store off the critical path.
//
// Verify mode: the data word of position p in message m is (m << 40) ^ p and
// every receiver checks every word it unpacks (torn or stale lines show up).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ll128_bench ll128_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) {                                                                  \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
      std::exit(1);                                                                           \
    }                                                                                         \
  } while (0)

typedef unsigned long long u64;

struct Chan {
  const u64* src;       // local source words
  u64* dst;             // local destination words
  u64* peer_stage;      // peer's staging (2 parities)
  const u64* my_stage;  // my staging (2 parities)
  u64* peer_free;       // peer's credit flag for me
  const u64* my_free;   // my credit flag (written by peer)
  u64* peer_arrive;     // proto 0: peer's arrival flag
  const u64* my_arrive;
  u64* sent;            // local message counters
  u64* recvd;
  unsigned* put_count;  // CTA arrival counters
  unsigned* all_count;
  unsigned long long* errors;
  long long n;          // data words per message
  long long lines;      // ll128 lines per message
  long long stage_words_per_parity;
  int nput;             // put CTAs (the rest receive)
  int verify;
  u64* trace;           // optional: 8 words per launch (see ll128_body)
  u64* trace_idx;       // launch counter (advanced by the last CTA)
};

__device__ __forceinline__ u64 gns() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ u64 ld_acq_sys(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_vol(const u64* p) {
  u64 v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(u64* p, u64 v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rlx_sys(u64* p, u64 v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned arrive(unsigned* c) {
  unsigned prev;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(c) : "memory");
  return prev;
}
__device__ __forceinline__ void st_v2_vol(u64* p, u64 a, u64 b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_v2_vol(const u64* p, u64& a, u64& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

__device__ __forceinline__ u64 word(const Chan& c, u64 m, long long p) {
  return c.verify ? ((m << 40) ^ static_cast<u64>(p)) : c.src[p];
}

// ------------------------------------------------------------- proto 0
__global__ void __launch_bounds__(256) flag_kernel(const __grid_constant__ Chan c) {
  __shared__ u64 sm;
  const bool put = blockIdx.x < c.nput;
  if (threadIdx.x == 0) sm = put ? *c.sent + 1 : *c.recvd + 1;
  __syncthreads();
  const u64 m = sm;
  if (put) {
    if (threadIdx.x == 0)
      while (ld_acq_sys(c.my_free) + 1 < m) __nanosleep(32);  // peer consumed message m-1
    __syncthreads();
    u64* d = c.peer_stage;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < c.n; i += 256ll * c.nput) d[i] = word(c, m, i);
    __syncthreads();
    if (threadIdx.x == 0 && arrive(c.put_count) + 1 == static_cast<unsigned>(c.nput)) {
      *c.put_count = 0;
      *c.sent = m;
      st_rel_sys(c.peer_arrive, m);
    }
  } else {
    if (threadIdx.x == 0)
      while (ld_acq_sys(c.my_arrive) < m) __nanosleep(32);
    __syncthreads();
    const int b = blockIdx.x - c.nput, nb = gridDim.x - c.nput;
    for (long long i = b * 256ll + threadIdx.x; i < c.n; i += 256ll * nb) {
      const u64 v = c.my_stage[i];
      c.dst[i] = v;
      if (c.verify && v != ((m << 40) ^ static_cast<u64>(i))) atomicAdd(c.errors, 1ull);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && arrive(c.all_count) + 1 == gridDim.x) {
    *c.all_count = 0;
    *c.recvd = m - (put ? 0 : 0);
    st_rel_sys(c.peer_free, *c.recvd);
  }
}

// ------------------------------------------------------------- proto 1
// line L of message m (parity m&1): words [L*16, L*16+15), word 15 = m.
// Warp q, iteration u, lane l covers line 4*(IT*q + u) + l/8, words
// 2*(l%8), 2*(l%8)+1. IT line groups per warp (loads first, then stores).
template <int IT, bool REL>
__device__ __forceinline__ void ll128_body(const Chan& c) {
  const u64 t_start = gns();
  __shared__ u64 sm;
  __shared__ u64* tslot;
  if (threadIdx.x == 0) tslot = c.trace ? c.trace + 8 * (*c.trace_idx % 4096) : nullptr;
  const int lines_per_cta = 8 * 4 * IT;
  const bool put = blockIdx.x < c.nput;
  if (threadIdx.x == 0) sm = put ? *c.sent + 1 : *c.recvd + 1;
  __syncthreads();
  const u64 m = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = lane & 7;
  const long long par = static_cast<long long>(m & 1) * c.stage_words_per_parity;
  const int b = put ? blockIdx.x : blockIdx.x - c.nput;
  const long long L0 = (long long)b * lines_per_cta + warp * 4 * IT + (lane >> 3);
  if (put) {
    if (threadIdx.x == 0)
      while (ld_vol(c.my_free) + 2 < m) __nanosleep(32);  // peer consumed message m-2 (same parity)
    __syncthreads();
    u64 a[IT], v[IT];
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const long long L = L0 + 4 * u;
      const long long p0 = L * 15 + 2 * j;
      a[u] = (L < c.lines && p0 < c.n) ? word(c, m, p0) : 0;
      v[u] = j == 7 ? m : ((L < c.lines && p0 + 1 < c.n) ? word(c, m, p0 + 1) : 0);
    }
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const long long L = L0 + 4 * u;
      if (L < c.lines) st_v2_vol(c.peer_stage + par + L * 16 + 2 * j, a[u], v[u]);
    }
    __syncthreads();
    if (tslot && threadIdx.x == 0) {
      atomicMax(tslot + 0, ~t_start);
      atomicMax(tslot + 1, gns());
    }
    if (threadIdx.x == 0 && arrive(c.put_count) + 1 == static_cast<unsigned>(c.nput)) {
      *c.put_count = 0;
      *c.sent = m;
    }
  } else {
    u64 a[IT], v[IT];
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int u = 0; u < IT; ++u) {
        const long long L = L0 + 4 * u;
        a[u] = 0;
        v[u] = m;
        if (L < c.lines) ld_v2_vol(c.my_stage + par + L * 16 + 2 * j, a[u], v[u]);
      }
#pragma unroll
      for (int u = 0; u < IT; ++u) {
        const u64 f = __shfl_sync(0xffffffffu, v[u], (lane & ~7) | 7);  // every lane
        ok = ok && f == m;
      }
      if (__all_sync(0xffffffffu, ok)) break;
      __nanosleep(20);
    }
    if (tslot && (threadIdx.x & 31) == 0) atomicMax(tslot + 3, gns());
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const long long L = L0 + 4 * u;
      if (L >= c.lines) break;
      const long long p0 = L * 15 + 2 * j;
      if (p0 < c.n) {
        c.dst[p0] = a[u];
        if (c.verify && a[u] != ((m << 40) ^ static_cast<u64>(p0))) atomicAdd(c.errors, 1ull);
      }
      if (j != 7 && p0 + 1 < c.n) {
        c.dst[p0 + 1] = v[u];
        if (c.verify && v[u] != ((m << 40) ^ static_cast<u64>(p0 + 1))) atomicAdd(c.errors, 1ull);
      }
    }
  }
  __syncthreads();
  if (tslot && threadIdx.x == 0) atomicMax(tslot + 4, gns());
  if (threadIdx.x == 0 && arrive(c.all_count) + 1 == gridDim.x) {
    *c.all_count = 0;
    *c.recvd = m;
    if (tslot) {
      atomicMax(tslot + 5, gns());
      *c.trace_idx = *c.trace_idx + 1;
    }
    if (REL)
      st_rel_sys(c.peer_free, m);
    else
      st_rlx_sys(c.peer_free, m);  // credit for message m (read 2 messages later)
  }
}

template <int IT, bool REL>
__global__ void __launch_bounds__(256) ll128_kernel(const __grid_constant__ Chan c) { ll128_body<IT, REL>(c); }

struct ChanPad {  // the library's launch parameter block is ~5 KB
  Chan c;
  char pad[5120];
};
__global__ void __launch_bounds__(256) ll128_kernel_pad(const __grid_constant__ ChanPad c) { ll128_body<4, false>(c.c); }

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    std::printf("need 2 GPUs\n");
    return 1;
  }
  const int K = 50;
  const int verify_iters = argc > 1 ? std::atoi(argv[1]) : 2000;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
  }
  const long long maxn = (32ll << 20) / 8;
  const long long maxlines = (maxn + 14) / 15;
  struct Dev {
    u64 *src, *dst, *stage, *flags;
    unsigned* counts;
    unsigned long long* errors;
    cudaStream_t s;
  } D[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&D[d].src, maxn * 8));
    CK(cudaMalloc(&D[d].dst, maxn * 8));
    CK(cudaMalloc(&D[d].stage, 2 * maxlines * 128));
    CK(cudaMalloc(&D[d].flags, 64 * 8));
    CK(cudaMalloc(&D[d].counts, 64 * 4));
    CK(cudaMalloc(&D[d].errors, 8));
    CK(cudaMemset(D[d].src, 1, maxn * 8));
    CK(cudaStreamCreateWithFlags(&D[d].s, cudaStreamNonBlocking));
  }
  auto reset = [&]() {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemset(D[d].stage, 0, 2 * maxlines * 128));
      CK(cudaMemset(D[d].flags, 0, 64 * 8));
      CK(cudaMemset(D[d].counts, 0, 64 * 4));
      CK(cudaMemset(D[d].errors, 0, 8));
      CK(cudaDeviceSynchronize());
    }
  };
  auto chan = [&](int d, long long n, int verify, int proto) {
    Chan c{};
    const int p = 1 - d;
    c.src = D[d].src;
    c.dst = D[d].dst;
    c.peer_stage = D[p].stage;
    c.my_stage = D[d].stage;
    c.peer_free = D[p].flags + 0;
    c.my_free = D[d].flags + 0;
    c.peer_arrive = D[p].flags + 1;
    c.my_arrive = D[d].flags + 1;
    c.sent = D[d].flags + 2;
    c.recvd = D[d].flags + 3;
    c.put_count = D[d].counts;
    c.all_count = D[d].counts + 1;
    c.errors = D[d].errors;
    c.n = n;
    c.lines = (n + 14) / 15;
    c.stage_words_per_parity = maxlines * 16;
    c.verify = verify;
    const long long per_cta = proto == 0 ? 256 * 8 : proto == 2 ? 8 * 4 * 15 : 8 * 4 * 4 * 15;  // words per CTA
    c.nput = static_cast<int>(std::max(1ll, (n + per_cta - 1) / per_cta));
    if (proto == 0) c.nput = std::min(c.nput, 592);  // grid-stride loops
    return c;
  };
  auto launch = [&](int d, const Chan& c, int proto) {
    if (proto == 0) {
      flag_kernel<<<2 * c.nput, 256, 0, D[d].s>>>(c);
    } else if (proto == 1) {
      ll128_kernel<4, false><<<2 * c.nput, 256, 0, D[d].s>>>(c);
    } else if (proto == 2) {
      ll128_kernel<1, false><<<2 * c.nput, 256, 0, D[d].s>>>(c);
    } else if (proto == 3) {
      ll128_kernel<4, true><<<2 * c.nput, 256, 0, D[d].s>>>(c);
    } else {
      ChanPad cp{};
      cp.c = c;
      ll128_kernel_pad<<<2 * c.nput, 256, 0, D[d].s>>>(cp);
    }
  };
  const char* pname[5] = {"flag", "ll128", "ll128_it1", "ll128_release_ack", "ll128_5KB_params"};
  // 1. integrity: many exchanges with changing data, every word checked
  for (int proto = 0; proto < 5; proto += 1) {
    for (long long bytes : {8ll, 4096ll, 262144ll, 2097152ll}) {
      reset();
      const long long n = bytes / 8;
      Chan c0 = chan(0, n, 1, proto), c1 = chan(1, n, 1, proto);
      for (int it = 0; it < verify_iters; ++it) {
        CK(cudaSetDevice(0));
        launch(0, c0, proto);
        CK(cudaSetDevice(1));
        launch(1, c1, proto);
      }
      unsigned long long e[2];
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&e[d], D[d].errors, 8, cudaMemcpyDeviceToHost));
      }
      std::printf("{\"test\":\"integrity\",\"proto\":\"%s\",\"bytes\":%lld,\"iters\":%d,\"errors\":[%llu,%llu]}\n",
                  pname[proto], bytes, verify_iters, e[0], e[1]);
    }
  }
  // 2. latency / bandwidth: K exchanges per graph, per exchange time
  for (int proto = 0; proto < 5; ++proto) {
    for (long long bytes = 8; bytes <= (32ll << 20); bytes *= 4) {
      reset();
      const long long n = bytes / 8;
      Chan c[2] = {chan(0, n, 0, proto), chan(1, n, 0, proto)};
      cudaGraphExec_t ge[2];
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(D[d].s, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < K; ++k) launch(d, c[d], proto);
        CK(cudaStreamEndCapture(D[d].s, &g));
        CK(cudaGraphInstantiate(&ge[d], g, 0));
      }
      std::vector<float> t;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEvent_t e0, e1;
        CK(cudaSetDevice(0));
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, D[0].s));
        CK(cudaGraphLaunch(ge[0], D[0].s));
        CK(cudaEventRecord(e1, D[0].s));
        CK(cudaSetDevice(1));
        CK(cudaGraphLaunch(ge[1], D[1].s));
        CK(cudaSetDevice(0));
        CK(cudaEventSynchronize(e1));
        CK(cudaSetDevice(1));
        CK(cudaDeviceSynchronize());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep) t.push_back(ms * 1000.f / K);
      }
      std::sort(t.begin(), t.end());
      const double us = t[t.size() / 2];
      std::printf("{\"test\":\"exchange\",\"proto\":\"%s\",\"bytes\":%lld,\"us\":%.2f,\"GBps\":%.1f,\"ctas\":%d}\n",
                  pname[proto], bytes, us, bytes / (us * 1e-6) / 1e9, 2 * c[0].nput);
    }
  }
  // 3. timeline of 20 exchanges at 2 MB (proto ll128), globaltimer marks
  {
    reset();
    const long long n = (2ll << 20) / 8;
    u64 *tr[2], *ti[2];
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMalloc(&tr[d], 4096 * 64));
      CK(cudaMemset(tr[d], 0, 4096 * 64));
      CK(cudaMalloc(&ti[d], 8));
      CK(cudaMemset(ti[d], 0, 8));
    }
    Chan c[2] = {chan(0, n, 0, 1), chan(1, n, 0, 1)};
    for (int d = 0; d < 2; ++d) {
      c[d].trace = tr[d];
      c[d].trace_idx = ti[d];
    }
    cudaGraphExec_t ge[2];
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(D[d].s, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < 20; ++k) launch(d, c[d], 1);
      CK(cudaStreamEndCapture(D[d].s, &g));
      CK(cudaGraphInstantiate(&ge[d], g, 0));
    }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaGraphLaunch(ge[d], D[d].s));
    }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
      std::vector<u64> h(20 * 8);
      CK(cudaMemcpy(h.data(), tr[d], h.size() * 8, cudaMemcpyDeviceToHost));
      const u64 t0 = ~h[0];
      for (int k = 0; k < 20; ++k) {
        const u64* w = h.data() + 8 * k;
        std::printf("{\"trace\":%d,\"launch\":%d,\"put_start\":%.2f,\"put_end\":%.2f,\"recv_ready\":%.2f,\"cta_end\":%.2f,\"end\":%.2f}\n",
                    d, k, (double)(~w[0] - t0) / 1e3, (double)(w[1] - t0) / 1e3, (double)(w[3] - t0) / 1e3,
                    (double)(w[4] - t0) / 1e3, (double)(w[5] - t0) / 1e3);
      }
    }
  }
  return 0;
}
