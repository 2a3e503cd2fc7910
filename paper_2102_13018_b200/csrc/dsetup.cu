// Device-side SetGraph + SetUp: the planner of
// starforest.cpp run on the GPU for graphs that already live in HBM.
//
// Reference: /root/reference/proj/src/starforest.cpp:29-161 (the same
// contract and error messages as the host planner), pattern.cpp:13-64 for the
// classification. The host planner (starforest.cpp StarForest::setup,
// pattern.cpp Pattern::analyze) is the specification; this file reproduces
// its results — group ranks, items, order and patterns — with:
//   validation / order checks   one pass, first offending position by atomicMin
//   leaf-index order            CUB stable radix sort of (leaf index, ordinal)
//                               only when the indices are not increasing
//   grouping by root rank       CUB stable radix sort on ceil(log2 P) key bits
//   discovery payload           gather off[ords]; the self segment never
//                               leaves HBM, remote segments go device to device
//                               over NCCL between processes (through the host
//                               control plane otherwise)
//   pattern classification      device find-first passes for contiguity and
//                               the Affine3D inference + full verification;
//                               distinct counts by bitmap or sorted uniques
// Everything is synchronous on cudaStreamPerThread (SetUp is collective and
// blocking in the reference too). Group items stay in HBM; host copies are
// made on demand by host_graph() for host-side consumers.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "sfg.hpp"

namespace sfg {

namespace {

constexpr int kT = 256;
constexpr int64_t kI32Max = (int64_t(1) << 31) - 1;
using u64 = unsigned long long;

cudaStream_t dstream() { return cudaStreamPerThread; }

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + kT - 1) / kT;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * 8)));
}

// Planner buffers come from the device's stream-ordered pool, which keeps
// freed memory mapped (release threshold = max): a 1 GB cudaMalloc/cudaFree
// costs 4-16 ms / up to 0.6 s on B200 (scripts/malloc_probe.py), the pool
// hands it back in microseconds once it has grown.
void ensure_pool() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  SFG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  SFG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = UINT64_MAX;
  SFG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done.push_back(dev);
}

template <class T>
T* dalloc(int64_t n) {
  void* p = nullptr;
  if (n > 0) {
    ensure_pool();
    SFG_CUDA(cudaMallocAsync(&p, static_cast<size_t>(n) * sizeof(T), dstream()));
  }
  return static_cast<T*>(p);
}

void dfree(void* p) {
  if (p) cudaFreeAsync(p, dstream());
}

template <class T>
T read1(const T* d) {
  T v{};
  SFG_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, dstream()));
  SFG_CUDA(cudaStreamSynchronize(dstream()));
  return v;
}

__device__ __forceinline__ u64 warp_min(u64 v) {
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide min of one value per thread into *out (atomicMin).
__device__ __forceinline__ void block_min_to(u64 v, u64* out) {
  __shared__ u64 red[kT / 32];
  v = warp_min(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    u64 w = threadIdx.x < kT / 32 ? red[threadIdx.x] : ~0ull;
    w = warp_min(w);
    if (threadIdx.x == 0 && w != ~0ull) atomicMin(out, w);
  }
  __syncthreads();
}

__global__ void k_fill(u64* p, int k, u64 v) {
  if (static_cast<int>(threadIdx.x) < k) p[threadIdx.x] = v;
}

// First position at which pred(i) holds, or n: grid-stride, per-thread
// first hit, block min, one atomicMin per block.
template <class Pred>
__global__ void __launch_bounds__(kT) k_find_first(int64_t n, Pred pred, u64* out) {
  u64 first = ~0ull;
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT)
    if (pred(i)) {
      first = static_cast<u64>(i);
      break;
    }
  block_min_to(first, out);
}

// Scratch for find-first results (one per forest call site, small).
struct Scratch {
  u64* v = nullptr;
  Scratch() { SFG_CUDA(cudaMalloc(&v, 8 * sizeof(u64))); }
  ~Scratch() { cudaFree(v); }
};

template <class Pred>
int64_t find_first(int64_t n, Pred pred, Scratch& sc) {
  if (n <= 0) return n;
  k_fill<<<1, 32, 0, dstream()>>>(sc.v, 1, static_cast<u64>(n));
  k_find_first<<<grid_for(n), kT, 0, dstream()>>>(n, pred, sc.v);
  SFG_CUDA(cudaGetLastError());
  const u64 r = read1(sc.v);
  return static_cast<int64_t>(std::min<u64>(r, static_cast<u64>(n)));
}

__global__ void k_iota(int64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) p[i] = i;
}

template <class T>
__global__ void k_gather(const T* __restrict__ src, const int64_t* __restrict__ idx, T* __restrict__ dst,
                         int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT)
    dst[i] = src[idx[i]];
}

// first[k] = first position of key k in the sorted keys (untouched if absent).
__global__ void k_key_starts(const int32_t* keys, int64_t n, int64_t* first) {
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT)
    if (i == 0 || keys[i] != keys[i - 1]) first[keys[i]] = i;
}

__global__ void k_minmax(const int64_t* idx, int64_t n, long long* mm) {
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    lo = min(lo, static_cast<long long>(idx[i]));
    hi = max(hi, static_cast<long long>(idx[i]));
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}

// Distinct values by bitmap over [lo, lo + 32*words): count bits newly set.
__global__ void k_bitmap_distinct(const int64_t* idx, int64_t n, int64_t lo, uint32_t* bits, u64* count,
                                  u64* repeat) {
  u64 fresh = 0, rep = 0;
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const uint64_t x = static_cast<uint64_t>(idx[i] - lo);
    const uint32_t b = 1u << (x & 31);
    const uint32_t old = atomicOr(&bits[x >> 5], b);
    if (old & b)
      rep = 1;
    else
      ++fresh;
  }
  for (int o = 16; o; o >>= 1) {
    fresh += __shfl_xor_sync(0xffffffffu, fresh, o);
    rep |= __shfl_xor_sync(0xffffffffu, rep, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (count && fresh) atomicAdd(count, fresh);
    if (repeat && rep) atomicOr(repeat, rep);
  }
}

__global__ void k_count_uniques(const int64_t* sorted, int64_t n, u64* count) {
  u64 c = 0;
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT)
    c += (i == 0 || sorted[i] != sorted[i - 1]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void k_narrow(const int64_t* src, int64_t n, int32_t* dst, u64* bad) {
  u64 first = ~0ull;
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const int64_t v = src[i];
    if (v > kI32Max && first == ~0ull) first = static_cast<u64>(i);
    dst[i] = static_cast<int32_t>(v);
  }
  block_min_to(first, bad);
}

// CUB radix sort of (key, value) pairs, stable, on bits [0, end_bit).
template <class K, class V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int end_bit) {
  size_t tmp = 0;
  SFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, end_bit, dstream()));
  void* t = nullptr;
  SFG_CUDA(cudaMallocAsync(&t, tmp, dstream()));
  SFG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, vout, n, 0, end_bit, dstream()));
  SFG_CUDA(cudaFreeAsync(t, dstream()));
}

template <class K>
void sort_keys(const K* kin, K* kout, int64_t n) {
  size_t tmp = 0;
  SFG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, n, 0, int(sizeof(K) * 8), dstream()));
  void* t = nullptr;
  SFG_CUDA(cudaMallocAsync(&t, tmp, dstream()));
  SFG_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, kin, kout, n, 0, int(sizeof(K) * 8), dstream()));
  SFG_CUDA(cudaFreeAsync(t, dstream()));
}

int64_t count_distinct_dev(const int64_t* idx, int64_t n, int64_t lo, int64_t hi, Scratch& sc) {
  if (n < 2) return n;
  const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
  k_fill<<<1, 32, 0, dstream()>>>(sc.v, 1, 0);
  if (span <= 4 * static_cast<uint64_t>(n) + 4096) {
    const int64_t words = static_cast<int64_t>((span + 31) / 32);
    uint32_t* bits = nullptr;
    SFG_CUDA(cudaMallocAsync(&bits, static_cast<size_t>(words) * 4, dstream()));
    SFG_CUDA(cudaMemsetAsync(bits, 0, static_cast<size_t>(words) * 4, dstream()));
    k_bitmap_distinct<<<grid_for(n), kT, 0, dstream()>>>(idx, n, lo, bits, sc.v, nullptr);
    SFG_CUDA(cudaFreeAsync(bits, dstream()));
  } else {
    int64_t* sorted = nullptr;
    SFG_CUDA(cudaMallocAsync(&sorted, static_cast<size_t>(n) * 8, dstream()));
    sort_keys(idx, sorted, n);
    k_count_uniques<<<grid_for(n), kT, 0, dstream()>>>(sorted, n, sc.v);
    SFG_CUDA(cudaFreeAsync(sorted, dstream()));
  }
  SFG_CUDA(cudaGetLastError());
  return static_cast<int64_t>(read1(sc.v));
}

// Pattern::analyze (pattern.cpp:230-299, infer_affine, no extents) over a
// list in HBM; indexed patterns keep the list there (Pattern::didx).
Pattern analyze_dev(const int64_t* idx, int64_t n, Scratch& sc) {
  if (n == 0) return Pattern::contiguous_range(0, 0);
  const int64_t start = read1(idx);
  const int64_t run = find_first(n, [=] __device__(int64_t i) { return idx[i] != start + i; }, sc);
  if (run == n) return Pattern::contiguous_range(start, n);

  if (start >= 0) {
    const int64_t dx = run;
    if (n % dx == 0) {
      const int64_t rows = n / dx;
      const int64_t s1 = read1(idx + dx) - start;
      if (s1 >= dx) {
        // dy = first row r >= 1 not at start + r*s1 (capped at rows)
        const int64_t dy = 1 + find_first(
                                   rows - 1,
                                   [=] __device__(int64_t r) {
                                     return idx[(r + 1) * dx] != start + (r + 1) * s1;
                                   },
                                   sc);
        if (rows % dy == 0) {
          const int64_t dz = rows / dy;
          const int64_t s2 = dz > 1 ? read1(idx + dy * dx) - start : dy * s1;
          const bool planes_ok = dz == 1 || s2 >= (dy - 1) * s1 + dx;
          if (planes_ok && dx < (int64_t(1) << 31) && dy < (int64_t(1) << 31)) {
            const int64_t plane = dx * dy;
            const int64_t bad = find_first(
                n,
                [=] __device__(int64_t i) {
                  const int64_t r = i / dx, x = i - r * dx;
                  const int64_t k = i / plane, j = r - k * dy;
                  return idx[i] != start + k * s2 + j * s1 + x;
                },
                sc);
            if (bad == n) {
              Pattern p;
              p.kind = Pattern::affine;
              p.count = n;
              p.start = start;
              p.dx = dx;
              p.dy = dy;
              p.dz = dz;
              p.s1 = s1;
              p.s2 = s2;
              p.bound = start + (dz - 1) * s2 + (dy - 1) * s1 + dx;
              p.distinct = n;
              return p;
            }
          }
        }
      }
    }
  }

  Pattern p;
  p.kind = Pattern::indexed;
  p.count = n;
  p.didx = idx;
  long long* mm = reinterpret_cast<long long*>(sc.v + 2);
  const long long init[2] = {LLONG_MAX, LLONG_MIN};
  SFG_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, dstream()));
  k_minmax<<<grid_for(n), kT, 0, dstream()>>>(idx, n, mm);
  SFG_CUDA(cudaGetLastError());
  long long got[2];
  SFG_CUDA(cudaMemcpyAsync(got, mm, sizeof(got), cudaMemcpyDeviceToHost, dstream()));
  SFG_CUDA(cudaStreamSynchronize(dstream()));
  p.start = got[0];
  p.bound = got[1] + 1;
  p.distinct = count_distinct_dev(idx, n, got[0], got[1], sc);
  p.has_duplicates = p.distinct < n;
  return p;
}

// ---------------------------------------------------------------- CSR build
// Root-sorted CSR of every contribution (StarForest::ensure_csr): one stable
// radix sort of (root, entry) pairs given in fold order, run-length encoding
// for the root list, binary searches for the self/remote split and the L2
// piece table, and a compaction for the remote-only view.

__global__ void k_csr_fill(const int64_t* keys, const int64_t* vals, int64_t n, int64_t base, int32_t* kout,
                           int32_t* vout, u64* bad) {
  u64 first = ~0ull;
  for (int64_t i = blockIdx.x * int64_t(kT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    kout[i] = static_cast<int32_t>(keys[i]);
    if (vals) {
      const int64_t v = vals[i];
      if (v > kI32Max && first == ~0ull) first = static_cast<u64>(i);
      vout[i] = static_cast<int32_t>(v);
    } else {
      vout[i] = static_cast<int32_t>(-(base + i) - 1);
    }
  }
  block_min_to(first, bad);
}

// Per root q: split = first remote (negative) entry; ptab row = first self
// entry at or beyond b * piece for b = 1..cols (self entries ascend).
__global__ void k_csr_split(const int32_t* off, const int32_t* ent, int64_t nq, int32_t* split, int32_t* ptab,
                            int cols, int64_t piece) {
  for (int64_t q = blockIdx.x * int64_t(kT) + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kT) {
    int32_t lo = off[q], hi = off[q + 1];
    while (lo < hi) {
      const int32_t mid = lo + (hi - lo) / 2;
      if (ent[mid] >= 0) lo = mid + 1; else hi = mid;
    }
    split[q] = lo;
    for (int b = 1; b <= cols; ++b) {
      int32_t a = off[q], e = lo;
      const int64_t v = b * piece;
      while (a < e) {
        const int32_t mid = a + (e - a) / 2;
        if (ent[mid] < v) a = mid + 1; else e = mid;
      }
      ptab[q * cols + (b - 1)] = a;
    }
  }
}

__global__ void k_csr_remote_counts(const int32_t* off, const int32_t* split, int64_t nq, int32_t* flag,
                                    int32_t* rcnt) {
  for (int64_t q = blockIdx.x * int64_t(kT) + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kT) {
    const int32_t r = off[q + 1] - split[q];
    flag[q] = r > 0;
    rcnt[q] = r;
  }
}

__global__ void k_csr_remote_view(const int32_t* roots, const int32_t* off, const int32_t* split,
                                  const int32_t* ent, int64_t nq, const int32_t* fpos, const int32_t* rpos,
                                  int32_t* rroots, int32_t* roffs, int32_t* rent, int32_t* clo, int32_t* chi,
                                  uint32_t* cbits, u64* centries) {
  u64 ce = 0;
  for (int64_t q = blockIdx.x * int64_t(kT) + threadIdx.x; q < nq; q += int64_t(gridDim.x) * kT) {
    const int32_t a = split[q], b = off[q + 1];
    if (a == b) continue;
    const int32_t k = fpos[q], p = rpos[q];
    rroots[k] = roots[q];
    roffs[k] = p;
    for (int32_t j = a; j < b; ++j) rent[p + (j - a)] = ent[j];
    if (clo) {
      clo[k] = off[q];
      chi[k] = b;
      ce += static_cast<u64>(b - off[q]);
      if (a > off[q]) atomicOr(&cbits[roots[q] >> 5], 1u << (roots[q] & 31));
    }
  }
  for (int o = 16; o; o >>= 1) ce += __shfl_xor_sync(0xffffffffu, ce, o);
  if ((threadIdx.x & 31) == 0 && ce) atomicAdd(centries, ce);
}

template <class T>
void excl_sum(const T* in, T* out, int64_t n) {
  size_t tmp = 0;
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, dstream()));
  void* t = nullptr;
  SFG_CUDA(cudaMallocAsync(&t, tmp, dstream()));
  SFG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, dstream()));
  SFG_CUDA(cudaFreeAsync(t, dstream()));
}

}  // namespace

DevGraph::~DevGraph() {
  if (device >= 0) cudaSetDevice(device);
  cudaDeviceSynchronize();
  int64_t* bufs[] = {local, off, ords, ridx != ords && ridx != local ? ridx : nullptr, loffs};
  for (int64_t* b : bufs)
    if (b) dfree(b);
  if (rank) dfree(rank);
}

void* dev_pool_alloc(size_t bytes) { return dalloc<char>(static_cast<int64_t>(bytes)); }
void dev_pool_free(void* p) { dfree(p); }

void dev_narrow_index(const int64_t* src, int64_t n, int32_t* dst) {
  if (n <= 0) return;
  Scratch sc;
  k_fill<<<1, 32, 0, dstream()>>>(sc.v, 1, ~0ull);
  k_narrow<<<grid_for(n), kT, 0, dstream()>>>(src, n, dst, sc.v);
  SFG_CUDA(cudaGetLastError());
  SFG_REQUIRE(read1(sc.v) == ~0ull, "index exceeds the int32 range of device plans");
}

bool dev_keys_sorted(const int64_t* items, const int64_t* src, int64_t n) {
  if (n <= 1) return true;
  Scratch sc;
  const int64_t bad = src == nullptr
                          ? find_first(n - 1, [=] __device__(int64_t i) { return items[i] > items[i + 1]; }, sc)
                          : find_first(
                                n - 1, [=] __device__(int64_t i) { return src[items[i]] > src[items[i + 1]]; }, sc);
  return bad == n - 1;
}

bool dev_any_repeat(const std::vector<std::pair<const int64_t*, int64_t>>& lists, int64_t bound) {
  if (bound <= 0) return false;
  Scratch sc;
  const int64_t words = (bound + 31) / 32;
  uint32_t* bits = dalloc<uint32_t>(words);
  SFG_CUDA(cudaMemsetAsync(bits, 0, static_cast<size_t>(words) * 4, dstream()));
  k_fill<<<1, 32, 0, dstream()>>>(sc.v, 1, 0);
  for (const auto& [p, n] : lists)
    if (n > 0) k_bitmap_distinct<<<grid_for(n), kT, 0, dstream()>>>(p, n, 0, bits, nullptr, sc.v);
  SFG_CUDA(cudaGetLastError());
  const bool rep = read1(sc.v) != 0;
  dfree(bits);
  return rep;
}

// set_graph (starforest.cpp:29-76) with the arrays in device memory: the
// same validation order and messages as StarForest::set_graph.
void StarForest::set_graph_device(int64_t nroots, int64_t nleaves, const int64_t* leaf_local,
                                  const int32_t* remote_rank, const int64_t* remote_off) {
  SFG_REQUIRE(state_ == SfState::created || state_ == SfState::graph_set,
              "set_graph requires a created or graph-set star forest");
  SFG_REQUIRE(nroots >= 0 && nleaves >= 0, "set_graph: negative root or leaf count");
  SFG_REQUIRE(nleaves == 0 || (remote_rank != nullptr && remote_off != nullptr),
              "set_graph: leaf_remote length does not match nleaves");
  SFG_REQUIRE(comm_->has_device(), "set_graph_device needs a communicator with a device");
  comm_->bind_device();
  const int64_t n = nleaves;
  Scratch sc;
  auto g = std::make_unique<DevGraph>();
  g->device = comm_->device();

  int64_t bound = n;
  bool contiguous = true;
  if (leaf_local != nullptr && n > 0) {
    const int64_t* L = leaf_local;
    const bool increasing =
        find_first(n, [=] __device__(int64_t i) { return i > 0 && L[i] <= L[i - 1]; }, sc) == n;
    contiguous = find_first(n, [=] __device__(int64_t i) { return L[i] != i; }, sc) == n;
    g->ascending = increasing;
    if (increasing) {
      SFG_REQUIRE(read1(L) >= 0, "set_graph: negative leaf index");
      bound = read1(L + n - 1) + 1;
    } else {
      int64_t* sorted = dalloc<int64_t>(n);
      sort_keys(L, sorted, n);
      const int64_t lo = read1(sorted);
      if (lo < 0) {
        dfree(sorted);
        fail("set_graph: negative leaf index");
      }
      const int64_t dup = find_first(n, [=] __device__(int64_t i) { return i > 0 && sorted[i] == sorted[i - 1]; }, sc);
      if (dup < n) {
        const int64_t v = read1(sorted + dup);
        dfree(sorted);
        fail("set_graph: duplicate leaf index " + std::to_string(v) + " violates the forest property");
      }
      bound = read1(sorted + n - 1) + 1;
      dfree(sorted);
    }
  } else if (leaf_local != nullptr) {
    bound = 0;
  }
  const int nranks = comm_->size();
  const int32_t* R = remote_rank;
  const int64_t* O = remote_off;
  const int64_t bad = find_first(
      n, [=] __device__(int64_t i) { return R[i] < 0 || R[i] >= nranks || O[i] < 0; }, sc);
  if (bad < n) {
    const int32_t r = read1(R + bad);
    SFG_REQUIRE(r >= 0 && r < nranks, "set_graph: root rank " + std::to_string(r) + " outside communicator");
    fail("set_graph: negative root offset");
  }

  // Own copies, like the host set_graph (the caller may free its arrays).
  auto copy = [&](auto*& dst, const auto* src) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(src)>>;
    dst = dalloc<T>(n);
    if (n) SFG_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(n) * sizeof(T), cudaMemcpyDeviceToDevice, dstream()));
  };
  if (leaf_local != nullptr && !contiguous) copy(g->local, leaf_local);
  copy(g->rank, remote_rank);
  copy(g->off, remote_off);
  SFG_CUDA(cudaStreamSynchronize(dstream()));

  nroots_ = nroots;
  nleaves_ = nleaves;
  leaf_bound_ = bound;
  contiguous_leaves_ = contiguous;
  has_local_ = leaf_local != nullptr;
  leaf_local_.clear();
  remote_rank_.clear();
  remote_off_.clear();
  root_groups_.clear();
  leaf_groups_.clear();
  self_first_ = false;
  multi_.reset();
  dev_.reset();
  staging_.clear();
  dg_ = std::move(g);
  state_ = SfState::graph_set;
}

// StarForest::setup (starforest.cpp:82-161) on the device.
void StarForest::setup_device() {
  comm_->bind_device();
  DevGraph& g = *dg_;
  const int me = comm_->rank();
  const int P = comm_->size();
  const int64_t n = nleaves_;
  Scratch sc;
  const bool trace = std::getenv("SFG_TRACE_SETUP") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    SFG_CUDA(cudaStreamSynchronize(dstream()));
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dsetup] %-28s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  };
  const int gs = grid_for(n);

  // Edge order: ascending leaf index (starforest.cpp:86-90), then stable by
  // root rank — ords[i] = leaf ordinal of the i-th edge.
  int64_t* ord = nullptr;  // leaf-index order, nullptr = identity
  if (!g.ascending && n > 0) {
    int64_t* iota = dalloc<int64_t>(n);
    int64_t* keys = dalloc<int64_t>(n);
    ord = dalloc<int64_t>(n);
    k_iota<<<gs, kT, 0, dstream()>>>(iota, n);
    sort_pairs(g.local, keys, iota, ord, n, 64);
    SFG_CUDA(cudaStreamSynchronize(dstream()));
    dfree(iota);
    dfree(keys);
  }
  std::vector<int64_t> start(static_cast<size_t>(P) + 1, 0), cnt(static_cast<size_t>(P), 0);
  if (P == 1 || n == 0) {
    if (ord) {
      g.ords = ord;
    } else {
      g.ords = dalloc<int64_t>(n);
      if (n) k_iota<<<gs, kT, 0, dstream()>>>(g.ords, n);
    }
    cnt[0] = P == 1 ? n : 0;  // n == 0: every group empty
  } else {
    int32_t* kin = dalloc<int32_t>(n);
    int32_t* kout = dalloc<int32_t>(n);
    int64_t* vin = ord;
    if (!vin) {
      vin = dalloc<int64_t>(n);
      k_iota<<<gs, kT, 0, dstream()>>>(vin, n);
    }
    k_gather<<<gs, kT, 0, dstream()>>>(g.rank, vin, kin, n);
    g.ords = dalloc<int64_t>(n);
    int bits = 0;
    while ((1 << bits) < P) ++bits;
    sort_pairs(kin, kout, vin, g.ords, n, bits);
    int64_t* first = dalloc<int64_t>(P);
    std::vector<int64_t> host_first(static_cast<size_t>(P), -1);
    SFG_CUDA(cudaMemcpyAsync(first, host_first.data(), static_cast<size_t>(P) * 8, cudaMemcpyHostToDevice,
                             dstream()));
    k_key_starts<<<gs, kT, 0, dstream()>>>(kout, n, first);
    SFG_CUDA(cudaMemcpyAsync(host_first.data(), first, static_cast<size_t>(P) * 8, cudaMemcpyDeviceToHost,
                             dstream()));
    SFG_CUDA(cudaStreamSynchronize(dstream()));
    dfree(first);
    dfree(kin);
    dfree(kout);
    dfree(vin);
    int64_t next = n;
    for (int r = P - 1; r >= 0; --r) {
      if (host_first[static_cast<size_t>(r)] < 0) continue;
      cnt[static_cast<size_t>(r)] = next - host_first[static_cast<size_t>(r)];
      next = host_first[static_cast<size_t>(r)];
    }
  }
  for (int r = 0; r < P; ++r) start[static_cast<size_t>(r) + 1] = start[static_cast<size_t>(r)] + cnt[static_cast<size_t>(r)];
  SFG_CUDA(cudaGetLastError());
  mark("order + group by rank");

  if (g.local) {
    g.ridx = dalloc<int64_t>(n);
    if (n) k_gather<<<gs, kT, 0, dstream()>>>(g.local, g.ords, g.ridx, n);
  } else {
    g.ridx = g.ords;
  }
  // Discovery payload: root offsets in edge order (starforest.cpp:96-107).
  int64_t* payload = dalloc<int64_t>(n);
  if (n) k_gather<<<gs, kT, 0, dstream()>>>(g.off, g.ords, payload, n);
  SFG_CUDA(cudaGetLastError());
  SFG_CUDA(cudaStreamSynchronize(dstream()));
  mark("payload");

  // Discovery exchange: the counts over the host control plane (8 bytes per
  // peer), then the lists themselves device to device when the control
  // plane can move device memory (NCCL between processes), else staged
  // through the host. The self list never leaves HBM. Leaf groups' items are
  // laid out back to back: self first, then the received lists in ascending
  // rank.
  const int64_t nself = cnt[static_cast<size_t>(me)];
  std::vector<int64_t> lstart(static_cast<size_t>(P), 0), lcnt(static_cast<size_t>(P), 0);
  lcnt[static_cast<size_t>(me)] = nself;
  if (P == 1) {
    g.loffs = payload;
    mark("discovery exchange");
  } else {
    std::vector<std::vector<uint8_t>> csend(static_cast<size_t>(P));
    for (int r = 0; r < P; ++r) {
      if (r == me) continue;
      csend[static_cast<size_t>(r)].resize(8);
      std::memcpy(csend[static_cast<size_t>(r)].data(), &cnt[static_cast<size_t>(r)], 8);
    }
    auto crecv = comm_->ctrl().alltoallv(std::move(csend));
    int64_t total = nself;
    for (int r = 0; r < P; ++r) {
      if (r == me) continue;
      const auto& b = crecv[static_cast<size_t>(r)];
      SFG_REQUIRE(b.size() == 8, "malformed setup payload");
      std::memcpy(&lcnt[static_cast<size_t>(r)], b.data(), 8);
      lstart[static_cast<size_t>(r)] = total;
      total += lcnt[static_cast<size_t>(r)];
    }
    g.loffs = dalloc<int64_t>(total);
    if (nself)
      SFG_CUDA(cudaMemcpyAsync(g.loffs, payload + start[static_cast<size_t>(me)], static_cast<size_t>(nself) * 8,
                               cudaMemcpyDeviceToDevice, dstream()));
    std::vector<int64_t> soff(static_cast<size_t>(P)), sbytes(static_cast<size_t>(P)),
        roff(static_cast<size_t>(P)), rbytes(static_cast<size_t>(P));
    for (int r = 0; r < P; ++r) {
      const size_t i = static_cast<size_t>(r);
      soff[i] = start[i] * 8;
      sbytes[i] = r == me ? 0 : cnt[i] * 8;
      roff[i] = lstart[i] * 8;
      rbytes[i] = r == me ? 0 : lcnt[i] * 8;
    }
    SFG_CUDA(cudaStreamSynchronize(dstream()));
    const bool on_device = comm_->ctrl().alltoallv_device(reinterpret_cast<const uint8_t*>(payload), soff, sbytes,
                                                          reinterpret_cast<uint8_t*>(g.loffs), roff, rbytes);
    if (!on_device) {
      std::vector<std::vector<uint8_t>> send(static_cast<size_t>(P));
      for (int r = 0; r < P; ++r) {
        const size_t i = static_cast<size_t>(r);
        if (r == me || sbytes[i] == 0) continue;
        send[i].resize(static_cast<size_t>(sbytes[i]));
        SFG_CUDA(cudaMemcpyAsync(send[i].data(), payload + start[i], send[i].size(), cudaMemcpyDeviceToHost,
                                 dstream()));
      }
      SFG_CUDA(cudaStreamSynchronize(dstream()));
      auto recv = comm_->ctrl().alltoallv(std::move(send));
      for (int r = 0; r < P; ++r) {
        const size_t i = static_cast<size_t>(r);
        if (r == me) continue;
        SFG_REQUIRE(static_cast<int64_t>(recv[i].size()) == rbytes[i], "malformed setup payload");
        if (rbytes[i])
          SFG_CUDA(cudaMemcpyAsync(g.loffs + lstart[i], recv[i].data(), recv[i].size(), cudaMemcpyHostToDevice,
                                   dstream()));
      }
      SFG_CUDA(cudaStreamSynchronize(dstream()));
    }
    mark(on_device ? "discovery exchange (device)" : "discovery exchange (host)");
    dfree(payload);
  }
  mark("receive");

  // Groups in ascending rank, offsets validated (starforest.cpp:116-123),
  // then the self group rotated to the head and every list classified.
  std::vector<Group> roots, leaves;
  for (int r = 0; r < P; ++r) {
    if (cnt[static_cast<size_t>(r)] == 0) continue;
    Group gr;
    gr.rank = r;
    gr.ditems = g.ords + start[static_cast<size_t>(r)];
    gr.pat.count = cnt[static_cast<size_t>(r)];
    roots.push_back(gr);
  }
  const int64_t nr = nroots_;
  for (int r = 0; r < P; ++r) {
    const int64_t m = lcnt[static_cast<size_t>(r)];
    if (m == 0) continue;
    const int64_t* items = g.loffs + lstart[static_cast<size_t>(r)];
    const int64_t bad = find_first(m, [=] __device__(int64_t i) { return items[i] >= nr; }, sc);
    SFG_REQUIRE(bad == m, "setup: leaf on rank " + std::to_string(r) + " references root offset " +
                              std::to_string(bad < m ? read1(items + bad) : 0) + " but this rank has only " +
                              std::to_string(nroots_) + " roots");
    Group gl;
    gl.rank = r;
    gl.ditems = items;
    gl.pat.count = m;
    leaves.push_back(gl);
  }
  mark("validate");
  auto self_to_head = [me](std::vector<Group>& v) {
    auto it = std::find_if(v.begin(), v.end(), [me](const Group& x) { return x.rank == me; });
    if (it != v.end()) std::rotate(v.begin(), it, it + 1);
  };
  self_to_head(roots);
  self_to_head(leaves);
  self_first_ = !roots.empty() && roots.front().rank == me;
  for (auto& gr : roots) {
    const int64_t* ip = g.ridx + (gr.ditems - g.ords);
    gr.pat = analyze_dev(ip, gr.pat.count, sc);
  }
  mark("analyze root groups");
  for (auto& gl : leaves) gl.pat = analyze_dev(gl.ditems, gl.pat.count, sc);
  mark("analyze leaf groups");

  root_groups_ = std::move(roots);
  leaf_groups_ = std::move(leaves);
  g.host_ready = false;
  state_ = SfState::set_up;
  prepare_default();
}

// Host copies of a device-set graph and its groups, for the host-side
// consumers (degrees, multi-SF, algebra, CSR build, group export).
void StarForest::host_graph() const {
  if (!dg_ || dg_->host_ready) return;
  comm_->bind_device();
  const DevGraph& g = *dg_;
  const size_t n = static_cast<size_t>(nleaves_);
  auto down = [](auto& dst, const auto* src, size_t cnt) {
    dst.resize(cnt);
    if (cnt)
      SFG_CUDA(cudaMemcpyAsync(dst.data(), src, cnt * sizeof(*src), cudaMemcpyDeviceToHost, dstream()));
  };
  if (g.local) down(leaf_local_, g.local, n);
  down(remote_rank_, g.rank, n);
  down(remote_off_, g.off, n);
  if (state_ == SfState::set_up) {
    for (auto* gs : {&root_groups_, &leaf_groups_})
      for (auto& gr : *gs) {
        down(gr.items, gr.ditems, static_cast<size_t>(gr.count()));
        if (gr.pat.kind == Pattern::indexed) down(gr.pat.idx, gr.pat.didx, static_cast<size_t>(gr.count()));
      }
  }
  SFG_CUDA(cudaStreamSynchronize(dstream()));
  dg_->host_ready = true;
}

void dev_csr_fill(const int64_t* keys, const int64_t* vals, int64_t n, int64_t base, int32_t* kout,
                  int32_t* vout) {
  if (n <= 0) return;
  Scratch sc;
  k_fill<<<1, 32, 0, dstream()>>>(sc.v, 1, ~0ull);
  k_csr_fill<<<grid_for(n), kT, 0, dstream()>>>(keys, vals, n, base, kout, vout, sc.v);
  SFG_CUDA(cudaGetLastError());
  SFG_REQUIRE(read1(sc.v) == ~0ull, "leaf index exceeds the int32 range of device plans");
}

void dev_build_csr(DevPlan& d, int32_t* key, int32_t* val, int64_t total, int64_t n_self, int64_t nroots,
                   int64_t leaf_bound, bool self) {
  SFG_REQUIRE(total <= kI32Max, "CSR exceeds the int32 range of device plans");
  Scratch sc;
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < nroots) ++bits;
  int32_t* skey = dalloc<int32_t>(total);
  int32_t* ent = dalloc<int32_t>(total);
  if (total) sort_pairs(key, skey, val, ent, total, bits);
  // roots + run lengths
  int32_t* roots = dalloc<int32_t>(total + 1);
  int32_t* cnts = dalloc<int32_t>(total + 1);
  int64_t nq = 0;
  if (total) {
    int64_t* nruns = reinterpret_cast<int64_t*>(sc.v + 4);
    size_t tmp = 0;
    SFG_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp, skey, roots, cnts, nruns, total, dstream()));
    void* t = nullptr;
    SFG_CUDA(cudaMallocAsync(&t, tmp, dstream()));
    SFG_CUDA(cub::DeviceRunLengthEncode::Encode(t, tmp, skey, roots, cnts, nruns, total, dstream()));
    SFG_CUDA(cudaFreeAsync(t, dstream()));
    nq = read1(nruns);
  }
  dfree(skey);
  // offs: exclusive sum over nq + 1 counts (the extra one set to 0 -> total)
  int32_t* offs = dalloc<int32_t>(nq + 1);
  SFG_CUDA(cudaMemsetAsync(cnts + nq, 0, sizeof(int32_t), dstream()));
  excl_sum(cnts, offs, nq + 1);

  constexpr int64_t kPiece = int64_t(1) << 21;
  const int64_t np_max = (leaf_bound + kPiece - 1) / kPiece;
  const int64_t mean_deg = nq ? total / nq : 0;
  const bool tiled = np_max >= 3 && mean_deg >= 8 && n_self > 0;
  const int cols = tiled ? static_cast<int>(np_max - 1) : 0;
  int32_t* split = dalloc<int32_t>(nq);
  int32_t* ptab = dalloc<int32_t>(nq * cols);
  if (nq) k_csr_split<<<grid_for(nq), kT, 0, dstream()>>>(offs, ent, nq, split, ptab, cols, kPiece);

  // remote-only view
  int32_t* flag = dalloc<int32_t>(nq + 1);
  int32_t* rcnt = dalloc<int32_t>(nq + 1);
  int32_t* fpos = dalloc<int32_t>(nq + 1);
  int32_t* rpos = dalloc<int32_t>(nq + 1);
  SFG_CUDA(cudaMemsetAsync(flag + nq, 0, sizeof(int32_t), dstream()));
  SFG_CUDA(cudaMemsetAsync(rcnt + nq, 0, sizeof(int32_t), dstream()));
  if (nq) k_csr_remote_counts<<<grid_for(nq), kT, 0, dstream()>>>(offs, split, nq, flag, rcnt);
  excl_sum(flag, fpos, nq + 1);
  excl_sum(rcnt, rpos, nq + 1);
  const int64_t rn = read1(fpos + nq);
  const int64_t rtotal = read1(rpos + nq);
  const int64_t nbits = self ? (nroots + 31) / 32 : 0;
  const int64_t ncl = self ? rn : 0;

  const int64_t words = nq + (nq + 1) + nq + total + rn + (rn + 1) + rtotal + nq * cols + 2 * ncl + nbits;
  if (words) SFG_CUDA(cudaMalloc(&d.csr_blob, static_cast<size_t>(words) * 4));
  int32_t* p = static_cast<int32_t*>(d.csr_blob);
  auto take = [&](int64_t n) {
    int32_t* q = p;
    p += n;
    return q;
  };
  auto d2d = [&](int32_t* dst, const int32_t* src, int64_t n) {
    if (n) SFG_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToDevice, dstream()));
  };
  d.csr_roots = take(nq);
  d2d(d.csr_roots, roots, nq);
  d.csr_off = take(nq + 1);
  d2d(d.csr_off, offs, nq + 1);
  d.csr_split = take(nq);
  d2d(d.csr_split, split, nq);
  d.csr_ent = take(total);
  d2d(d.csr_ent, ent, total);
  d.rcsr_roots = take(rn);
  d.rcsr_off = take(rn + 1);
  d.rcsr_ent = take(rtotal);
  d.csr_ptab = take(nq * cols);
  d2d(d.csr_ptab, ptab, nq * cols);
  if (!tiled) d.csr_ptab = nullptr;
  d.ccsr_lo = take(ncl);
  d.ccsr_hi = take(ncl);
  uint32_t* cb = reinterpret_cast<uint32_t*>(take(nbits));
  if (nbits) SFG_CUDA(cudaMemsetAsync(cb, 0, static_cast<size_t>(nbits) * 4, dstream()));
  d.coupled_bits = self ? cb : nullptr;
  d2d(d.rcsr_off + rn, rpos + nq, 1);
  k_fill<<<1, 32, 0, dstream()>>>(sc.v, 1, 0);
  if (nq)
    k_csr_remote_view<<<grid_for(nq), kT, 0, dstream()>>>(roots, offs, split, ent, nq, fpos, rpos, d.rcsr_roots,
                                                          d.rcsr_off, d.rcsr_ent, self ? d.ccsr_lo : nullptr,
                                                          self ? d.ccsr_hi : nullptr, cb, sc.v);
  SFG_CUDA(cudaGetLastError());
  d.ccsr_entries += static_cast<int64_t>(read1(sc.v));
  for (int32_t* b : {ent, roots, cnts, offs, split, ptab, flag, rcnt, fpos, rpos})
    if (b) dfree(b);
  if (tiled) {
    d.csr_np_max = static_cast<int32_t>(np_max);
    d.csr_piece_leaves = kPiece;
  }
  d.csr_n = nq;
  d.csr_self_entries = self ? n_self : 0;
  d.csr_remote_entries = total - d.csr_self_entries;
  d.rcsr_n = rn;
}

}  // namespace sfg
