// Random 8-byte gather / fold microbenchmark on one B200 (BASELINE configs 1
// and 4 shapes): leaf[i] = root[idx[i]] (Bcast REPLACE) and root[r] = fold
// of its leaves in ascending leaf order (Reduce SUM, bit-exact order).
//
//   elem     one element per item, 8 items per thread (round-1 kernel shape)
//   csr      thread per root over a root-sorted CSR (round-1 Reduce kernel)
//   2phase   transposition through an L2-resident scratch S: phase A works
//            on ROOT buckets (roots staged in shared memory), phase B on LEAF
//            chunks (leaves staged in shared memory); each phase reads and
//            writes only coalesced runs, the random access happens in SMEM.
//            Bcast: A gathers roots -> S (chunk-major), B scatters S -> leaf.
//            Reduce: A' gathers leaves -> S (bucket-major), B' folds per root
//            from SMEM in leaf order (bit-identical to the sequential fold).
// Host-built plans (the library builds them at SetUp). Times: CUDA events,
// L2 flushed (256 MB read) before every timed call, median of 20.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bench gather_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

static uint64_t sm64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------------ kernels
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

template <int U>
__global__ void __launch_bounds__(256) gather_persist(const double* __restrict__ root, const int* __restrict__ idx,
                                                     double* __restrict__ leaf, long long L) {
  const long long stride = (long long)gridDim.x * 256 * U;
  for (long long b = blockIdx.x * 256ll * U + threadIdx.x; b < L; b += stride) {
    double v[U];
    int ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ix[u] = b + u * 256 < L ? __ldg(idx + b + u * 256) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = root[ix[u]];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + u * 256 < L) leaf[b + u * 256] = v[u];
  }
}

// thread per root, 8 entries in flight (round-1 csr_kernel shape)
__global__ void __launch_bounds__(256, 4) csr_fold(double* root, const int* __restrict__ off, const int* __restrict__ ent,
                                                  const double* __restrict__ leaf, int R) {
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r >= R) return;
  const int lo = off[r], hi = off[r + 1];
  double acc = root[r];
  int en[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) en[q] = lo + q < hi ? __ldg(ent + lo + q) : 0;
  for (int j = lo; j < hi; j += 8) {
    double c[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (j + q < hi) c[q] = leaf[en[q]];
    int nx[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) nx[q] = j + 8 + q < hi ? __ldg(ent + j + 8 + q) : 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (j + q >= hi) break;
      acc = __dadd_rn(acc, c[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) en[q] = nx[q];
  }
  root[r] = acc;
}

// ---- two-phase Bcast
// A: CTA per root bucket (RB roots in smem); entries of the bucket in
// (chunk, leaf) order; S[posA[e]] = tile[rootA[e]].
__global__ void __launch_bounds__(256) bcast_A(const double* __restrict__ root, int R, int RB,
                                               const int* __restrict__ eoff, const uint16_t* __restrict__ rootA,
                                               const int* __restrict__ posA, double* __restrict__ S) {
  extern __shared__ double tile[];
  const int b = blockIdx.x;
  const int r0 = b * RB, nr = min(RB, R - r0);
  for (int i = threadIdx.x; i < nr; i += 256) tile[i] = root[r0 + i];
  __syncthreads();
  const int lo = eoff[b], hi = eoff[b + 1];
  for (int e = lo + threadIdx.x; e < hi; e += 256) S[__ldg(posA + e)] = tile[__ldg(rootA + e)];
}

// B: CTA per leaf chunk (LC leaves in smem); chunk region of S in bucket
// order; tile[permB[k]] = S[k]; tile -> leaf (coalesced). Full chunks only.
__global__ void __launch_bounds__(256) bcast_B(const double* __restrict__ S, int LC, long long L,
                                               const uint16_t* __restrict__ permB, double* __restrict__ leaf) {
  extern __shared__ double tile[];
  const long long c0 = (long long)blockIdx.x * LC;
  const int n = (int)min((long long)LC, L - c0);
  for (int k = threadIdx.x; k < n; k += 256) tile[__ldg(permB + c0 + k)] = S[c0 + k];
  __syncthreads();
  double2* out = reinterpret_cast<double2*>(leaf + c0);
  const double2* t2 = reinterpret_cast<const double2*>(tile);
  for (int k = threadIdx.x; k < n / 2; k += 256) out[k] = t2[k];
}

// ---- two-phase Reduce
// A': CTA per leaf chunk: tile = leaf chunk; S[posR[k]] = tile[permR[k]] for
// the chunk's entries in (bucket, leaf) order.
__global__ void __launch_bounds__(256) reduce_A(const double* __restrict__ leaf, int LC, long long L,
                                                const uint16_t* __restrict__ permR, const int* __restrict__ posR,
                                                double* __restrict__ S) {
  extern __shared__ double tile[];
  const long long c0 = (long long)blockIdx.x * LC;
  const int n = (int)min((long long)LC, L - c0);
  const double2* in = reinterpret_cast<const double2*>(leaf + c0);
  double2* t2 = reinterpret_cast<double2*>(tile);
  for (int k = threadIdx.x; k < n / 2; k += 256) t2[k] = in[k];
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += 256) S[__ldg(posR + c0 + k)] = tile[__ldg(permR + c0 + k)];
}

// B': CTA per root bucket: region of S (entries of the bucket's roots in
// leaf order) -> smem; thread per root folds its entries (bucket CSR, local
// u16 offsets) in order.
__global__ void __launch_bounds__(256) reduce_B(double* root, const int* __restrict__ rb, const int* __restrict__ sb,
                                                const int* __restrict__ roff, const uint16_t* __restrict__ rent,
                                                const double* __restrict__ S) {
  extern __shared__ double tile[];
  const int b = blockIdx.x;
  const int s0 = sb[b], ns = sb[b + 1] - s0;
  for (int k = threadIdx.x; k < ns; k += 256) tile[k] = S[s0 + k];
  __syncthreads();
  for (int r = rb[b] + threadIdx.x; r < rb[b + 1]; r += 256) {
    double acc = root[r];
    const int lo = roff[r], hi = roff[r + 1];
    for (int j = lo; j < hi; ++j) acc = __dadd_rn(acc, tile[__ldg(rent + j)]);
    root[r] = acc;
  }
}

// ---- improved two-phase (ILP: each thread issues all its loads first)
// A2: CTA per root bucket; entries padded to a multiple of 8 per bucket (pad
// entries write to a dummy slot); thread handles 8 consecutive entries with
// 16-byte index loads.
__global__ void __launch_bounds__(512) bcast_A2(const double* __restrict__ root, int R, int RB,
                                                const int* __restrict__ eoff, const uint16_t* __restrict__ rootA,
                                                const int* __restrict__ posA, double* __restrict__ S) {
  extern __shared__ double tile[];
  const int b = blockIdx.x;
  const int r0 = b * RB, nr = min(RB, R - r0);
  for (int i = threadIdx.x; i < nr; i += 512) tile[i] = root[r0 + i];
  __syncthreads();
  const int lo = eoff[b], hi = eoff[b + 1];  // multiples of 8
  for (int e = lo + threadIdx.x * 8; e < hi; e += 512 * 8) {
    const uint4 ra = *reinterpret_cast<const uint4*>(rootA + e);
    const int4 p0 = *reinterpret_cast<const int4*>(posA + e);
    const int4 p1 = *reinterpret_cast<const int4*>(posA + e + 4);
    const uint16_t* r = reinterpret_cast<const uint16_t*>(&ra);
    const int pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) S[pp[q]] = tile[r[q]];
  }
}

// B2: CTA per leaf chunk (LC leaves), 512 threads, 16 loads in flight each.
template <int LC>
__global__ void __launch_bounds__(512) bcast_B2(const double* __restrict__ S, long long L,
                                                const uint16_t* __restrict__ permB, double* __restrict__ leaf) {
  extern __shared__ double tile[];
  const long long c0 = (long long)blockIdx.x * LC;
  constexpr int J = LC / 512;
  double v[J];
  uint16_t pk[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int k = j * 512 + threadIdx.x;
    pk[j] = __ldg(permB + c0 + k);
    v[j] = S[c0 + k];
  }
#pragma unroll
  for (int j = 0; j < J; ++j) tile[pk[j]] = v[j];
  __syncthreads();
  double2* out = reinterpret_cast<double2*>(leaf + c0);
  const double2* t2 = reinterpret_cast<const double2*>(tile);
#pragma unroll
  for (int j = 0; j < LC / 2 / 512; ++j) out[j * 512 + threadIdx.x] = t2[j * 512 + threadIdx.x];
}

// A'2: CTA per leaf chunk: tile = leaf chunk; S[posR[k]] = tile[permR[k]].
template <int LC>
__global__ void __launch_bounds__(512) reduce_A2(const double* __restrict__ leaf, const uint16_t* __restrict__ permR,
                                                 const int* __restrict__ posR, double* __restrict__ S) {
  extern __shared__ double tile[];
  const long long c0 = (long long)blockIdx.x * LC;
  const double2* in = reinterpret_cast<const double2*>(leaf + c0);
  double2* t2 = reinterpret_cast<double2*>(tile);
  constexpr int J = LC / 512;
  uint16_t pk[J];
  int ps[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    pk[j] = __ldg(permR + c0 + j * 512 + threadIdx.x);
    ps[j] = __ldg(posR + c0 + j * 512 + threadIdx.x);
  }
#pragma unroll
  for (int j = 0; j < LC / 2 / 512; ++j) t2[j * 512 + threadIdx.x] = in[j * 512 + threadIdx.x];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < J; ++j) S[ps[j]] = tile[pk[j]];
}

// B'2: CTA per root bucket, 512 threads.
__global__ void __launch_bounds__(512) reduce_B2(double* root, const int* __restrict__ rb, const int* __restrict__ sb,
                                                 const int* __restrict__ roff, const uint16_t* __restrict__ rent,
                                                 const double* __restrict__ S) {
  extern __shared__ double tile[];
  const int b = blockIdx.x;
  const int s0 = sb[b], ns = sb[b + 1] - s0;
  for (int k = threadIdx.x; k < ns; k += 512) tile[k] = S[s0 + k];
  __syncthreads();
  for (int r = rb[b] + threadIdx.x; r < rb[b + 1]; r += 512) {
    double acc = root[r];
    const int lo = roff[r], hi = roff[r + 1];
    for (int j = lo; j < hi; ++j) acc = __dadd_rn(acc, tile[__ldg(rent + j)]);
    root[r] = acc;
  }
}

__global__ void flush_read(const double4* p, long long n, double* sink) {
  double a = 0;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (long long)gridDim.x * 256) a += p[i].x;
  if (a == 1.2345) *sink = a;
}

// ------------------------------------------------------------------ driver
struct Timer {
  double4* flush;
  long long nf;
  double* sink;
  cudaEvent_t e0, e1;
  Timer() {
    nf = (256ll << 20) / 32;
    CK(cudaMalloc(&flush, nf * 32));
    CK(cudaMemset(flush, 0, nf * 32));
    CK(cudaMalloc(&sink, 8));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
  }
  template <class F>
  double run(F&& f, int reps = 20) {
    std::vector<float> t;
    for (int i = 0; i < reps + 2; ++i) {
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
  }
};

static void config(const char* name, long long L, int R, int RB, int LC, Timer& T) {
  uint64_t s = 12345;
  std::vector<int> idx(L);
  for (long long i = 0; i < L; ++i) idx[i] = (int)(sm64(s) % (uint64_t)R);
  std::vector<double> hroot(R), hleaf(L);
  for (int r = 0; r < R; ++r) hroot[r] = (double)(sm64(s) >> 11) * 0x1.0p-53;
  for (long long i = 0; i < L; ++i) hleaf[i] = (double)(sm64(s) >> 11) * 0x1.0p-53;
  // CSR by root (ascending leaf)
  std::vector<int> off(R + 1, 0), ent(L);
  for (long long i = 0; i < L; ++i) off[idx[i] + 1]++;
  for (int r = 0; r < R; ++r) off[r + 1] += off[r];
  {
    std::vector<int> cur(off.begin(), off.end() - 1);
    for (long long i = 0; i < L; ++i) ent[cur[idx[i]]++] = (int)i;
  }
  // expected results
  std::vector<double> want_leaf(L), want_root(hroot);
  for (long long i = 0; i < L; ++i) want_leaf[i] = hroot[idx[i]];
  for (long long i = 0; i < L; ++i) want_root[idx[i]] += hleaf[i];

  double *droot, *dleaf, *dS, *dout;
  int *didx, *doff, *dent;
  CK(cudaMalloc(&droot, R * 8ll));
  CK(cudaMalloc(&dout, R * 8ll));
  CK(cudaMalloc(&dleaf, L * 8));
  CK(cudaMalloc(&dS, L * 8));
  CK(cudaMalloc(&didx, L * 4));
  CK(cudaMalloc(&doff, (R + 1) * 4ll));
  CK(cudaMalloc(&dent, L * 4));
  CK(cudaMemcpy(didx, idx.data(), L * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(doff, off.data(), (R + 1) * 4ll, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dent, ent.data(), L * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(droot, hroot.data(), R * 8ll, cudaMemcpyHostToDevice));
  std::vector<double> got(std::max<long long>(L, R));
  auto check_leaf = [&](const char* what) {
    CK(cudaMemcpy(got.data(), dleaf, L * 8, cudaMemcpyDeviceToHost));
    const bool ok = std::memcmp(got.data(), want_leaf.data(), L * 8) == 0;
    return ok;
  };
  const double bcast_bytes = 0.0;  // filled per config
  (void)bcast_bytes;
  // distinct roots
  long long distinct = 0;
  for (int r = 0; r < R; ++r) distinct += off[r + 1] > off[r];
  const double bb = distinct * 8.0 + L * 12.0;          // Bcast algorithmic
  const double rbytes = L * 12.0 + distinct * 16.0;    // Reduce algorithmic
  auto line = [&](const char* op, const char* kern, double us, double bytes, bool ok) {
    std::printf("{\"config\":\"%s\",\"op\":\"%s\",\"kernel\":\"%s\",\"us\":%.2f,\"GBps\":%.0f,\"ok\":%s}\n", name, op,
                kern, us, bytes / (us * 1e-6) / 1e9, ok ? "true" : "false");
  };
  const int nb_elem = (int)((L + 2047) / 2048);
  double us;
  us = T.run([&] { gather_elem<<<nb_elem, 256>>>(droot, didx, dleaf, L); });
  line("bcast", "elem8", us, bb, check_leaf("elem"));
  for (int k : {4, 8, 16}) {
    CK(cudaMemset(dleaf, 0, L * 8));
    us = T.run([&] { gather_persist<8><<<148 * k, 256>>>(droot, didx, dleaf, L); });
    char nm[32];
    std::snprintf(nm, sizeof nm, "persist8_x%d", k);
    line("bcast", nm, us, bb, check_leaf(nm));
  }
  CK(cudaMemset(dleaf, 0, L * 8));
  us = T.run([&] { gather_persist<16><<<148 * 4, 256>>>(droot, didx, dleaf, L); });
  line("bcast", "persist16_x4", us, bb, check_leaf("p16"));

  // ---- two-phase bcast plan
  const int nb = (R + RB - 1) / RB;
  const int nc = (int)((L + LC - 1) / LC);
  // entries per (chunk, bucket), S positions: chunk-major, bucket order inside a chunk, leaf order inside
  std::vector<int> cnt((size_t)nc * nb, 0);
  for (long long i = 0; i < L; ++i) cnt[(size_t)(i / LC) * nb + idx[i] / RB]++;
  std::vector<long long> cpos((size_t)nc * nb);
  {
    long long acc = 0;
    for (size_t k = 0; k < cpos.size(); ++k) {
      cpos[k] = acc;
      acc += cnt[k];
    }
  }
  std::vector<uint16_t> permB(L);
  std::vector<int> eoff(nb + 1, 0), posA(L);
  std::vector<uint16_t> rootA(L);
  {
    std::vector<long long> cur(cpos);
    std::vector<int> bcount(nb, 0);
    for (long long i = 0; i < L; ++i) bcount[idx[i] / RB]++;
    for (int b = 0; b < nb; ++b) eoff[b + 1] = eoff[b] + bcount[b];
    std::vector<int> bcur(eoff.begin(), eoff.end() - 1);
    // leaves in ascending order: per bucket the entries come out in (chunk, leaf) order
    for (long long i = 0; i < L; ++i) {
      const int b = idx[i] / RB;
      const size_t k = (size_t)(i / LC) * nb + b;
      const long long p = cur[k]++;
      permB[p] = (uint16_t)(i % LC);
      const int e = bcur[b]++;
      posA[e] = (int)p;
      rootA[e] = (uint16_t)(idx[i] - b * RB);
    }
  }
  int *deoff, *dposA;
  uint16_t *drootA, *dpermB;
  CK(cudaMalloc(&deoff, (nb + 1) * 4));
  CK(cudaMalloc(&dposA, L * 4));
  CK(cudaMalloc(&drootA, L * 2));
  CK(cudaMalloc(&dpermB, L * 2));
  CK(cudaMemcpy(deoff, eoff.data(), (nb + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dposA, posA.data(), L * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drootA, rootA.data(), L * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpermB, permB.data(), L * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(bcast_A, cudaFuncAttributeMaxDynamicSharedMemorySize, RB * 8));
  CK(cudaFuncSetAttribute(bcast_B, cudaFuncAttributeMaxDynamicSharedMemorySize, LC * 8));
  CK(cudaMemset(dleaf, 0, L * 8));
  cudaEvent_t m0, m1, m2;
  CK(cudaEventCreate(&m0));
  CK(cudaEventCreate(&m1));
  CK(cudaEventCreate(&m2));
  float ta = 0, tb = 0;
  us = T.run([&] {
    CK(cudaEventRecord(m0));
    bcast_A<<<nb, 256, RB * 8>>>(droot, R, RB, deoff, drootA, dposA, dS);
    CK(cudaEventRecord(m1));
    bcast_B<<<nc, 256, LC * 8>>>(dS, LC, L, dpermB, dleaf);
    CK(cudaEventRecord(m2));
  });
  CK(cudaEventSynchronize(m2));
  CK(cudaEventElapsedTime(&ta, m0, m1));
  CK(cudaEventElapsedTime(&tb, m1, m2));
  line("bcast", "2phase", us, bb, check_leaf("2phase"));
  {
    // padded copies of the bucket entry lists (dummy slot at L)
    std::vector<int> eoff8(nb + 1, 0);
    for (int b = 0; b < nb; ++b) eoff8[b + 1] = eoff8[b] + ((eoff[b + 1] - eoff[b] + 7) / 8) * 8;
    std::vector<uint16_t> rootA8(eoff8[nb], 0);
    std::vector<int> posA8(eoff8[nb], (int)L);
    for (int b = 0; b < nb; ++b)
      for (int e = eoff[b]; e < eoff[b + 1]; ++e) {
        rootA8[eoff8[b] + e - eoff[b]] = rootA[e];
        posA8[eoff8[b] + e - eoff[b]] = posA[e];
      }
    int *deoff8, *dposA8;
    uint16_t* drootA8;
    double* dS8;
    CK(cudaMalloc(&deoff8, (nb + 1) * 4));
    CK(cudaMalloc(&dposA8, eoff8[nb] * 4ll));
    CK(cudaMalloc(&drootA8, eoff8[nb] * 2ll));
    CK(cudaMalloc(&dS8, (L + 8) * 8));
    CK(cudaMemcpy(deoff8, eoff8.data(), (nb + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dposA8, posA8.data(), eoff8[nb] * 4ll, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(drootA8, rootA8.data(), eoff8[nb] * 2ll, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(bcast_A2, cudaFuncAttributeMaxDynamicSharedMemorySize, RB * 8));
    CK(cudaFuncSetAttribute(bcast_B2<8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8));
    if (L % 8192 == 0) {
      CK(cudaMemset(dleaf, 0, L * 8));
      // B2 needs chunk-major S with chunks of 8192: rebuild permB for LC=8192
      const int LC2 = 8192, nc2 = (int)(L / LC2);
      std::vector<int> cnt2((size_t)nc2 * nb, 0);
      for (long long i = 0; i < L; ++i) cnt2[(size_t)(i / LC2) * nb + idx[i] / RB]++;
      std::vector<long long> cur2((size_t)nc2 * nb);
      long long acc = 0;
      for (size_t k = 0; k < cur2.size(); ++k) { cur2[k] = acc; acc += cnt2[k]; }
      std::vector<uint16_t> permB2(L);
      std::vector<int> bcur(eoff8.begin(), eoff8.end() - 1);
      for (long long i = 0; i < L; ++i) {
        const int b = idx[i] / RB;
        const long long p = cur2[(size_t)(i / LC2) * nb + b]++;
        permB2[p] = (uint16_t)(i % LC2);
        const int e = bcur[b]++;
        posA8[e] = (int)p;
      }
      CK(cudaMemcpy(dposA8, posA8.data(), eoff8[nb] * 4ll, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dpermB, permB2.data(), L * 2, cudaMemcpyHostToDevice));
      us = T.run([&] {
        CK(cudaEventRecord(m0));
        bcast_A2<<<nb, 512, RB * 8>>>(droot, R, RB, deoff8, drootA8, dposA8, dS8);
        CK(cudaEventRecord(m1));
        bcast_B2<8192><<<nc2, 512, 8192 * 8>>>(dS8, L, dpermB, dleaf);
        CK(cudaEventRecord(m2));
      });
      CK(cudaEventSynchronize(m2));
      CK(cudaEventElapsedTime(&ta, m0, m1));
      CK(cudaEventElapsedTime(&tb, m1, m2));
      line("bcast", "2phase_v2", us, bb, check_leaf("2phase_v2"));
      std::printf("{\"config\":\"%s\",\"two_phase_bcast_v2\":{\"A_us\":%.2f,\"B_us\":%.2f}}\n", name, ta * 1000, tb * 1000);
    }
    cudaFree(deoff8); cudaFree(dposA8); cudaFree(drootA8); cudaFree(dS8);
  }
  std::printf("{\"config\":\"%s\",\"two_phase_bcast\":{\"A_us\":%.2f,\"B_us\":%.2f,\"buckets\":%d,\"chunks\":%d}}\n", name,
              ta * 1000, tb * 1000, nb, nc);

  // ---- reduce: CSR thread per root
  CK(cudaMemcpy(dleaf, hleaf.data(), L * 8, cudaMemcpyHostToDevice));
  auto check_root = [&]() {
    CK(cudaMemcpy(got.data(), dout, R * 8ll, cudaMemcpyDeviceToHost));
    return std::memcmp(got.data(), want_root.data(), R * 8ll) == 0;
  };
  us = T.run([&] {
    CK(cudaMemcpyAsync(dout, droot, R * 8ll, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(m0));
    csr_fold<<<(R + 255) / 256, 256>>>(dout, doff, dent, dleaf, R);
    CK(cudaEventRecord(m1));
  });
  CK(cudaEventSynchronize(m1));
  CK(cudaEventElapsedTime(&ta, m0, m1));
  line("reduce", "csr_thread", ta * 1000, rbytes, check_root());

  // ---- reduce: two-phase. Buckets = root ranges with <= SB entries (smem),
  // S bucket-major (entries of a bucket in leaf order), chunks of LC leaves.
  const int SB = 16384;
  std::vector<int> rb{0};
  {
    int acc = 0;
    for (int r = 0; r < R; ++r) {
      const int d = off[r + 1] - off[r];
      if (acc + d > SB && r > rb.back()) {
        rb.push_back(r);
        acc = 0;
      }
      acc += d;
    }
    rb.push_back(R);
  }
  const int nbr = (int)rb.size() - 1;
  std::vector<int> bucket_of(R);
  for (int b = 0; b < nbr; ++b)
    for (int r = rb[b]; r < rb[b + 1]; ++r) bucket_of[r] = b;
  std::vector<int> sb(nbr + 1, 0);
  for (int b = 0; b < nbr; ++b) sb[b + 1] = sb[b] + (off[rb[b + 1]] - off[rb[b]]);
  // S position of leaf i: bucket base + rank of i among the bucket's leaves (leaf order)
  std::vector<int> posS(L);
  {
    std::vector<int> cur(sb.begin(), sb.end() - 1);
    for (long long i = 0; i < L; ++i) posS[i] = cur[bucket_of[idx[i]]]++;
  }
  // A': chunk entries in (bucket, leaf) order: permR (local leaf) + posR
  std::vector<uint16_t> permR(L);
  std::vector<int> posR(L);
  for (long long c0 = 0; c0 < L; c0 += LC) {
    const long long n = std::min<long long>(LC, L - c0);
    std::vector<int> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return bucket_of[idx[c0 + a]] < bucket_of[idx[c0 + b]]; });
    for (long long k = 0; k < n; ++k) {
      permR[c0 + k] = (uint16_t)ord[k];
      posR[c0 + k] = posS[c0 + ord[k]];
    }
  }
  // B': per root, its entries' local offsets in the bucket's S region (ascending leaf)
  std::vector<uint16_t> rent(L);
  for (int r = 0; r < R; ++r)
    for (int j = off[r]; j < off[r + 1]; ++j) rent[j] = (uint16_t)(posS[ent[j]] - sb[bucket_of[r]]);
  int *drb, *dsb, *dposR;
  uint16_t *dpermR, *drent;
  CK(cudaMalloc(&drb, (nbr + 1) * 4));
  CK(cudaMalloc(&dsb, (nbr + 1) * 4));
  CK(cudaMalloc(&dposR, L * 4));
  CK(cudaMalloc(&dpermR, L * 2));
  CK(cudaMalloc(&drent, L * 2));
  CK(cudaMemcpy(drb, rb.data(), (nbr + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsb, sb.data(), (nbr + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dposR, posR.data(), L * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpermR, permR.data(), L * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drent, rent.data(), L * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(reduce_A, cudaFuncAttributeMaxDynamicSharedMemorySize, LC * 8));
  CK(cudaFuncSetAttribute(reduce_B, cudaFuncAttributeMaxDynamicSharedMemorySize, SB * 8));
  us = T.run([&] {
    CK(cudaMemcpyAsync(dout, droot, R * 8ll, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(m0));
    reduce_A<<<nc, 256, LC * 8>>>(dleaf, LC, L, dpermR, dposR, dS);
    CK(cudaEventRecord(m1));
    reduce_B<<<nbr, 256, SB * 8>>>(dout, drb, dsb, doff, drent, dS);
    CK(cudaEventRecord(m2));
  });
  CK(cudaEventSynchronize(m2));
  CK(cudaEventElapsedTime(&ta, m0, m1));
  CK(cudaEventElapsedTime(&tb, m1, m2));
  line("reduce", "2phase", (ta + tb) * 1000, rbytes, check_root());
  if (LC == 8192 && L % 8192 == 0) {
    CK(cudaFuncSetAttribute(reduce_A2<8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8));
    CK(cudaFuncSetAttribute(reduce_B2, cudaFuncAttributeMaxDynamicSharedMemorySize, SB * 8));
    us = T.run([&] {
      CK(cudaMemcpyAsync(dout, droot, R * 8ll, cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(m0));
      reduce_A2<8192><<<nc, 512, 8192 * 8>>>(dleaf, dpermR, dposR, dS);
      CK(cudaEventRecord(m1));
      reduce_B2<<<nbr, 512, SB * 8>>>(dout, drb, dsb, doff, drent, dS);
      CK(cudaEventRecord(m2));
    });
    CK(cudaEventSynchronize(m2));
    CK(cudaEventElapsedTime(&ta, m0, m1));
    CK(cudaEventElapsedTime(&tb, m1, m2));
    line("reduce", "2phase_v2", (ta + tb) * 1000, rbytes, check_root());
    std::printf("{\"config\":\"%s\",\"two_phase_reduce_v2\":{\"A_us\":%.2f,\"B_us\":%.2f}}\n", name, ta * 1000, tb * 1000);
  }
  std::printf("{\"config\":\"%s\",\"two_phase_reduce\":{\"A_us\":%.2f,\"B_us\":%.2f,\"buckets\":%d}}\n", name, ta * 1000,
              tb * 1000, nbr);
  cudaFree(droot); cudaFree(dout); cudaFree(dleaf); cudaFree(dS); cudaFree(didx); cudaFree(doff); cudaFree(dent);
  cudaFree(deoff); cudaFree(dposA); cudaFree(drootA); cudaFree(dpermB);
  cudaFree(drb); cudaFree(dsb); cudaFree(dposR); cudaFree(dpermR); cudaFree(drent);
}

int main() {
  Timer T;
  config("cfg1", 4194304, 1048576, 4096, 8192, T);
  config("cfg4", 16777216, 65536, 4096, 8192, T);
  return 0;
}
