// sm_100a kernels for the star-forest data path.
//
// One launch executes a table of segments (see kernels.hpp). Each CTA owns a
// contiguous block of kThreads*kItems work items of one segment; every thread
// first resolves all its indices and issues all its loads (kItems independent
// loads in flight per thread), then applies the reduction and stores. The
// index maps are evaluated with 32-bit magic-number division so an Affine3D
// pattern (a 3-D subblock of a ghosted box) costs a few integer ops per
// element and no index traffic.
//
// Reference semantics (what every segment type must reproduce):
//   ops:      /root/reference/proj/src/pack.cpp:19-45  (MAX is `if (b > a) a = b`)
//   pack:     /root/reference/proj/src/pack.cpp:111-121
//   unpack:   /root/reference/proj/src/pack.cpp:138-173
//   scatter:  /root/reference/proj/src/pack.cpp:220-256
//   fetch:    /root/reference/proj/src/ops.cpp:110-158, 521-563
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "kernels.hpp"


namespace sfg {
namespace {

enum : int {
  OP_REPLACE = 0,
  OP_SUM = 1,
  OP_PROD = 2,
  OP_MAX = 3,
  OP_MIN = 4,
  OP_LAND = 5,
  OP_LOR = 6,
  OP_BAND = 7,
  OP_BOR = 8
};

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.s;
}

__device__ __forceinline__ int64_t pat_index(const DPat& p, int64_t i) {
  if (p.kind == PAT_CONTIG) return p.start + i;
  if (p.kind == PAT_INDEXED) return static_cast<int64_t>(__ldg(p.idx + i));
  const uint32_t ui = static_cast<uint32_t>(i);
  const uint32_t row = fdiv(ui, p.dx);
  const uint32_t x = ui - row * p.dx.d;
  const uint32_t z = fdiv(row, p.dy);
  const uint32_t y = row - z * p.dy.d;
  return p.start + static_cast<int64_t>(x) + static_cast<int64_t>(y) * p.s1 +
         static_cast<int64_t>(z) * p.s2;
}

template <class T>
struct Unsigned {
  using type = T;
};
template <>
struct Unsigned<int32_t> {
  using type = uint32_t;
};
template <>
struct Unsigned<int64_t> {
  using type = uint64_t;
};

// a (op)= b with the reference's exact semantics; integer arithmetic wraps.
template <class T, int OP>
__device__ __forceinline__ T apply_op(T a, T b) {
  if constexpr (OP == OP_REPLACE) {
    return b;
  } else if constexpr (OP == OP_SUM) {
    if constexpr (std::is_same_v<T, double>)
      return __dadd_rn(a, b);
    else
      return static_cast<T>(static_cast<typename Unsigned<T>::type>(a) +
                            static_cast<typename Unsigned<T>::type>(b));
  } else if constexpr (OP == OP_PROD) {
    if constexpr (std::is_same_v<T, double>)
      return __dmul_rn(a, b);
    else
      return static_cast<T>(static_cast<typename Unsigned<T>::type>(a) *
                            static_cast<typename Unsigned<T>::type>(b));
  } else if constexpr (OP == OP_MAX) {
    return (b > a) ? b : a;
  } else if constexpr (OP == OP_MIN) {
    return (b < a) ? b : a;
  } else if constexpr (OP == OP_LAND) {
    return (a && b) ? T(1) : T(0);
  } else if constexpr (OP == OP_LOR) {
    return (a || b) ? T(1) : T(0);
  } else if constexpr (OP == OP_BAND) {
    if constexpr (std::is_integral_v<T>) return a & b;
    return a;
  } else {
    if constexpr (std::is_integral_v<T>) return a | b;
    return a;
  }
}

struct ItemMap {
  int64_t bl;
  bool small;
  FastDiv f;
  __device__ __forceinline__ void split(int64_t e, int64_t& i, int64_t& k) const {
    if (bl == 1) {
      i = e;
      k = 0;
    } else if (small) {
      i = fdiv(static_cast<uint32_t>(e), f);
      k = e - i * bl;
    } else {
      i = e / bl;
      k = e - i * bl;
    }
  }
};

__device__ __forceinline__ bool skipped(const uint32_t* bits, int64_t v) {
  return bits != nullptr && ((__ldg(bits + (v >> 5)) >> (v & 31)) & 1u);
}

// dst[dpat(i)] (op)= src[spat(i)] over this CTA's items.
template <class T, int OP, class PP>
__device__ __forceinline__ void run_pair(const DSeg& s, const PP& P, int64_t blk) {
  const T* __restrict__ src = static_cast<const T*>(P.bufs[s.src_buf]);
  T* dst = static_cast<T*>(P.bufs[s.dst_buf]);
  const int64_t total = s.n * P.bl;
  const ItemMap im{P.bl, total < (int64_t(1) << 31), P.bldiv};
  const int64_t base = blk * (kThreads * kItems) + threadIdx.x;
  T v[kItems];
  T d[kItems];
  int64_t di[kItems];
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    const int64_t e = base + static_cast<int64_t>(u) * kThreads;
    di[u] = -1;
    if (e < total) {
      int64_t i, k;
      im.split(e, i, k);
      const int64_t si = pat_index(s.src, i) * P.bl + k;
      const int64_t dv = pat_index(s.dst, i);
      if constexpr (OP != OP_REPLACE) {
        if (skipped(s.skip_dst, dv)) continue;
      }
      di[u] = dv * P.bl + k;
      v[u] = src[si];
      if constexpr (OP != OP_REPLACE) d[u] = dst[di[u]];
    }
  }
#pragma unroll
  for (int u = 0; u < kItems; ++u) {
    if (di[u] < 0) continue;
    if constexpr (OP == OP_REPLACE) {
      dst[di[u]] = v[u];
    } else {
      dst[di[u]] = apply_op<T, OP>(d[u], v[u]);
    }
  }
}

// Row mode: both patterns are contiguous or Affine3D and share runs of
// `s.run` positions that are contiguous on both sides. Each warp owns 32*kItems
// consecutive elements of the CTA's chunk; index maps are evaluated once per
// run (not per element), then the lanes stream the run with kItems
// independent loads in flight each.
template <class T, int OP, class PP>
__device__ __forceinline__ void run_pair_rows(const DSeg& s, const PP& P, int64_t blk) {
  const T* __restrict__ src = static_cast<const T*>(P.bufs[s.src_buf]);
  T* dst = static_cast<T*>(P.bufs[s.dst_buf]);
  const int64_t bl = P.bl;
  const int64_t total = s.n * bl;
  const ItemMap im{bl, total < (int64_t(1) << 31), P.bldiv};
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int64_t e = blk * (kThreads * kItems) + static_cast<int64_t>(warp) * (32 * kItems);
  const int64_t wend = min(e + 32 * kItems, total);
  while (e < wend) {
    int64_t pos, k;
    im.split(e, pos, k);
    const uint32_t r = fdiv(static_cast<uint32_t>(pos), s.rundiv);
    const int64_t in_run = pos - static_cast<int64_t>(r) * s.run;
    const int64_t len = min((s.run - in_run) * bl - k, wend - e);
    const T* sp = src + pat_index(s.src, pos) * bl + k;
    const int64_t d0 = pat_index(s.dst, pos) * bl + k;  // element index of dp[0]
    T* dp = dst + d0;
    T v[kItems];
    T d[kItems];
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const int64_t i = lane + 32 * u;
      if (i < len) {
        v[u] = sp[i];
        if constexpr (OP != OP_REPLACE) d[u] = dp[i];
      }
    }
    // Coupled roots (skip_dst): one bitmap word per lane covers the whole run
    // (<= 32 * kItems vertices, bl == 1); only runs that contain a coupled
    // root test their elements, the others store unconditionally.
    uint32_t skipw = 0;
    bool any_skip = false;
    int64_t w0 = 0;
    if constexpr (OP != OP_REPLACE) {
      if (s.skip_dst != nullptr) {
        if (bl == 1) {
          w0 = d0 >> 5;
          const int64_t w1 = (d0 + len - 1) >> 5;
          if (w0 + lane <= w1) skipw = __ldg(s.skip_dst + w0 + lane);
          any_skip = __any_sync(0xffffffffu, skipw != 0);
        } else {
          any_skip = true;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const int64_t i = lane + 32 * u;
      bool keep = i < len;
      if constexpr (OP != OP_REPLACE) {
        if (any_skip) {
          const int64_t vx = bl == 1 ? d0 + i : (d0 + i) / bl;
          const uint32_t word = bl == 1 ? __shfl_sync(0xffffffffu, skipw, static_cast<int>((vx >> 5) - w0) & 31)
                                        : __ldg(s.skip_dst + (vx >> 5));
          keep = keep && !((word >> (vx & 31)) & 1u);
        }
      }
      if (keep) {
        if constexpr (OP == OP_REPLACE)
          dp[i] = v[u];
        else
          dp[i] = apply_op<T, OP>(d[u], v[u]);
      }
    }
    e += len;
  }
}

// Root-sorted fold in the reference order (self leaves ascending, then remote
// groups ascending rank, each in ascending leaf order). Sequential per root,
// so floating-point results are bit-identical to the CPU reference.
// Sequential fold of contributions [lo, hi) of one root item by one thread,
// kB contributions in flight (entries, then values, then the dependent fold).
template <class T, int OP, int kB, bool FETCH>
__device__ __forceinline__ T csr_thread_range(const DSeg& s, const T* leaf, T* stage, T* aux,
                                              int64_t bl, int64_t k, int32_t lo, int32_t hi, T acc) {
  if constexpr (FETCH) {
    // entries, then values, then the fold storing every contribution's
    // fetched value (the pipelined form below measured slower here: the
    // scattered fetched-value stores dominate, 227 vs 267 us on config 4)
    for (int32_t j = lo; j < hi; j += kB) {
      int32_t en[kB];
      T c[kB];
#pragma unroll
      for (int q = 0; q < kB; ++q) en[q] = j + q < hi ? __ldg(s.csr_ent + j + q) : 0;
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (j + q < hi)
          c[q] = en[q] >= 0 ? leaf[static_cast<int64_t>(en[q]) * bl + k]
                            : stage[static_cast<int64_t>(-en[q] - 1) * bl + k];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        if (j + q >= hi) break;
        if (en[q] >= 0)
          aux[static_cast<int64_t>(en[q]) * bl + k] = acc;
        else
          stage[static_cast<int64_t>(-en[q] - 1) * bl + k] = acc;
        acc = apply_op<T, OP>(acc, c[q]);
      }
    }
    return acc;
  }
  // Fold, software pipelined: the entries of batch b+1 are loaded right after the
  // value loads of batch b are issued, before batch b is folded, so a batch
  // waits on one memory round trip (its values) instead of two (entries,
  // then values): config 4 Reduce 164 -> 112 us.
  int32_t en[kB];
#pragma unroll
  for (int q = 0; q < kB; ++q) en[q] = lo + q < hi ? __ldg(s.csr_ent + lo + q) : 0;
  for (int32_t j = lo; j < hi; j += kB) {
    T c[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q)
      if (j + q < hi)
        c[q] = en[q] >= 0 ? leaf[static_cast<int64_t>(en[q]) * bl + k]
                          : stage[static_cast<int64_t>(-en[q] - 1) * bl + k];
    int32_t nx[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) nx[q] = j + kB + q < hi ? __ldg(s.csr_ent + j + kB + q) : 0;
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      if (j + q >= hi) break;
      acc = apply_op<T, OP>(acc, c[q]);
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) en[q] = nx[q];
  }
  return acc;
}

// Bounds of piece q of root r (see DSeg::csr_np).
__device__ __forceinline__ void csr_piece(const DSeg& s, int64_t r, int q, int32_t& lo, int32_t& hi) {
  const int32_t* pt = s.csr_ptab + r * s.csr_pt_stride;
  lo = q == 0 ? __ldg(s.csr_lo + r) : __ldg(pt + q * s.csr_pt_step - 1);
  hi = q == s.csr_np - 1 ? __ldg(s.csr_hi + r) : __ldg(pt + (q + 1) * s.csr_pt_step - 1);
}

// Group of a CSR entry under a free-order fetch shuffle (see FetchShuffle).
__device__ __forceinline__ int shuf_group(const FetchShuffle& f, int32_t e) {
  if (e >= 0) return 0;
  const int32_t pos = -e - 1;
  int k = 0;
  const int nrem = f.n - f.self;
  while (k + 1 < nrem && pos >= f.off[k + 1]) ++k;
  return f.self + k;
}

// First entry in [lo, hi) whose group is >= g (groups ascend along a root's
// entries).
__device__ __forceinline__ int32_t shuf_bound(const FetchShuffle& f, const int32_t* ent, int32_t lo,
                                              int32_t hi, int g) {
  while (lo < hi) {
    const int32_t mid = lo + (hi - lo) / 2;
    if (shuf_group(f, __ldg(ent + mid)) < g)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Root-sorted fold in the reference order (self leaves ascending, then remote
// groups ascending rank, each in ascending leaf order), one thread per root
// item: sequential per root, so floating-point results are bit-identical to
// the CPU reference, and a warp instruction advances 32 roots at once.
// With pieces (csr_np > 1) the grid walks L2-sized leaf windows piece-major
// (see run_csr_warp).
template <class T, int OP, int kB, bool FETCH, class PP>
__device__ __forceinline__ void run_csr_t(const DSeg& s, const PP& P, int64_t blk) {
  T* root = static_cast<T*>(P.bufs[s.dst_buf]);
  const T* leaf = static_cast<const T*>(P.bufs[s.src_buf]);
  T* stage = static_cast<T*>(P.bufs[s.stage_buf]);
  T* aux = static_cast<T*>(P.bufs[s.aux_buf]);
  const int64_t bl = P.bl;
  const int64_t total = s.n * bl;
  const ItemMap im{bl, total < (int64_t(1) << 31), P.bldiv};
  const int64_t t0 = blk * kThreads + threadIdx.x;
  if (s.csr_np <= 1) {
    if (t0 >= total) return;
    int64_t r, k;
    im.split(t0, r, k);
    // root id and entry range loaded together (one memory round trip)
    const int32_t rid = __ldg(s.csr_roots + r);
    const int32_t lo = __ldg(s.csr_lo + r);
    const int32_t hi = __ldg(s.csr_hi + r);
    if (skipped(s.skip_dst, rid)) return;
    if (lo >= hi) return;
    const int64_t ro = static_cast<int64_t>(rid) * bl + k;
    if (FETCH && P.shuf.n > 1) {
      T acc = root[ro];
      for (int q = 0; q < P.shuf.n; ++q) {
        const int g = P.shuf.perm[q];
        const int32_t a = shuf_bound(P.shuf, s.csr_ent, lo, hi, g);
        const int32_t b = shuf_bound(P.shuf, s.csr_ent, a, hi, g + 1);
        if (a < b) acc = csr_thread_range<T, OP, kB, FETCH>(s, leaf, stage, aux, bl, k, a, b, acc);
      }
      root[ro] = acc;
      return;
    }
    root[ro] = csr_thread_range<T, OP, kB, FETCH>(s, leaf, stage, aux, bl, k, lo, hi, root[ro]);
    return;
  }
  for (int q = 0; q < s.csr_np; ++q) {
    for (int64_t e = t0; e < total; e += s.csr_grid_threads) {
      int64_t r, k;
      im.split(e, r, k);
      if (skipped(s.skip_dst, __ldg(s.csr_roots + r))) continue;
      int32_t lo, hi;
      csr_piece(s, r, q, lo, hi);
      if (lo >= hi) continue;
      const int64_t ro = static_cast<int64_t>(__ldg(s.csr_roots + r)) * bl + k;
      root[ro] = csr_thread_range<T, OP, kB, FETCH>(s, leaf, stage, aux, bl, k, lo, hi, root[ro]);
    }
  }
}

template <class T, int OP, int kB = 8>
__device__ __forceinline__ void run_csr(const DSeg& s, const LaunchParams& P, int64_t blk, bool fetch) {
  if (fetch)
    run_csr_t<T, OP, kB, true, LaunchParams>(s, P, blk);
  else
    run_csr_t<T, OP, kB, false, LaunchParams>(s, P, blk);
}

// One warp folds contributions [lo, hi) of one root item into acc (held by
// every lane). The 32 lanes load 32 consecutive contributions (coalesced
// entry reads), 8 chunks in flight; with csr_seq the fold runs in exact entry
// order through shuffles (bit-identical to the sequential reference for
// floating point), otherwise as a warp tree (fold) or inclusive scan (fetch),
// exact for the associative integer ops.
template <class T, int OP>
__device__ __forceinline__ T csr_warp_range(const DSeg& s, const T* leaf, T* stage, T* aux,
                                            int64_t bl, int64_t k, int32_t lo, int32_t hi, T acc,
                                            bool fetch) {
  const int lane = threadIdx.x & 31;
  constexpr int kChunks = 8;  // 256 contributions in flight per warp
  for (int32_t sbase = lo; sbase < hi; sbase += 32 * kChunks) {
    int32_t ens[kChunks];
    T vs[kChunks];
#pragma unroll
    for (int c = 0; c < kChunks; ++c) {
      const int32_t j = sbase + 32 * c + lane;
      ens[c] = j < hi ? __ldg(s.csr_ent + j) : 0;
    }
#pragma unroll
    for (int c = 0; c < kChunks; ++c) {
      const int32_t j = sbase + 32 * c + lane;
      vs[c] = T(0);
      if (j < hi)
        vs[c] = ens[c] >= 0 ? leaf[static_cast<int64_t>(ens[c]) * bl + k]
                            : stage[static_cast<int64_t>(-ens[c] - 1) * bl + k];
    }
#pragma unroll
    for (int c = 0; c < kChunks; ++c) {
      const int32_t base = sbase + 32 * c;
      if (base >= hi) break;
      const int32_t j = base + lane;
      const int cnt = min(32, hi - base);
      const int32_t en = ens[c];
      const T v = vs[c];
      T mine = acc;
      if (s.csr_seq) {
        for (int q = 0; q < cnt; ++q) {
          const T vq = __shfl_sync(0xffffffffu, v, q);
          if (lane == q) mine = acc;
          acc = apply_op<T, OP>(acc, vq);
        }
      } else if (!fetch) {
        T x = v;
        for (int off = 16; off > 0; off >>= 1) {
          const T y = __shfl_down_sync(0xffffffffu, x, off);
          if (lane + off < cnt) x = apply_op<T, OP>(x, y);
        }
        acc = apply_op<T, OP>(acc, __shfl_sync(0xffffffffu, x, 0));
      } else {
        T x = v;  // inclusive scan over lanes < cnt
        for (int off = 1; off < 32; off <<= 1) {
          const T y = __shfl_up_sync(0xffffffffu, x, off);
          if (lane >= off && lane < cnt) x = apply_op<T, OP>(y, x);
        }
        const T excl = __shfl_up_sync(0xffffffffu, x, 1);
        mine = lane == 0 ? acc : apply_op<T, OP>(acc, excl);
        acc = apply_op<T, OP>(acc, __shfl_sync(0xffffffffu, x, cnt - 1));
      }
      if (fetch && j < hi) {
        if (en >= 0)
          aux[static_cast<int64_t>(en) * bl + k] = mine;
        else
          stage[static_cast<int64_t>(-en - 1) * bl + k] = mine;
      }
    }
  }
  return acc;
}

// Warp-per-root CSR fold / fetch for high-degree roots.
//
// L2-tiled ("pieces") when the gathered leaf array is larger than L2: the
// self contributions of every root are split at leaf-index boundaries
// (csr_ptab), and the grid — sized to be fully resident — walks the pieces
// in order, each warp folding piece q of all its roots before piece q+1, so
// at any time the CTAs gather from one L2-sized window of the leaf (and
// leafupdate) arrays and every 32-byte sector is fetched from DRAM once
// instead of once per contribution. Each root is owned by one warp, so the
// fold order per root is unchanged (pieces ascend in leaf index, exactly the
// reference order) and no grid barrier is needed for correctness.
template <class T, int OP>
__device__ __forceinline__ void run_csr_warp(const DSeg& s, const LaunchParams& P, int64_t blk,
                                             bool fetch) {
  T* root = static_cast<T*>(P.bufs[s.dst_buf]);
  const T* leaf = static_cast<const T*>(P.bufs[s.src_buf]);
  T* stage = static_cast<T*>(P.bufs[s.stage_buf]);
  T* aux = static_cast<T*>(P.bufs[s.aux_buf]);
  const int64_t bl = P.bl;
  const int lane = threadIdx.x & 31;
  const int64_t items = s.n * bl;
  const ItemMap im{bl, items < (int64_t(1) << 31), P.bldiv};
  const int64_t w0 = blk * (kThreads / 32) + (threadIdx.x >> 5);
  if (s.csr_np <= 1) {
    if (w0 >= items) return;
    int64_t r, k;
    im.split(w0, r, k);
    // root id and entry range loaded together (one memory round trip)
    const int32_t rid = __ldg(s.csr_roots + r);
    const int32_t lo = __ldg(s.csr_lo + r);
    const int32_t hi = __ldg(s.csr_hi + r);
    if (skipped(s.skip_dst, rid)) return;
    if (lo >= hi) return;
    const int64_t ro = static_cast<int64_t>(rid) * bl + k;
    if (fetch && P.shuf.n > 1) {
      // group boundaries in one coalesced pass over the root's entries:
      // bound[g] = lo + #entries of a group < g (entries ascend by group)
      int32_t bound[kMaxShuffle + 1];
#pragma unroll
      for (int g = 0; g <= kMaxShuffle; ++g) bound[g] = lo;
      for (int32_t c = lo; c < hi; c += 32) {
        const int32_t j = c + lane;
        const int gj = j < hi ? shuf_group(P.shuf, __ldg(s.csr_ent + j)) : kMaxShuffle;
#pragma unroll
        for (int g = 1; g <= kMaxShuffle; ++g)
          bound[g] += __popc(__ballot_sync(0xffffffffu, gj < g));
      }
      T acc = root[ro];
      for (int q = 0; q < P.shuf.n; ++q) {
        const int g = P.shuf.perm[q];
        const int32_t a = bound[g];
        const int32_t b = g + 1 < P.shuf.n ? bound[g + 1] : hi;
        if (a < b) acc = csr_warp_range<T, OP>(s, leaf, stage, aux, bl, k, a, b, acc, true);
      }
      if (lane == 0) root[ro] = acc;
      return;
    }
    const T acc = csr_warp_range<T, OP>(s, leaf, stage, aux, bl, k, lo, hi, root[ro], fetch);
    if (lane == 0) root[ro] = acc;
    return;
  }
  const int64_t nw = s.csr_grid_threads / 32;
  for (int q = 0; q < s.csr_np; ++q) {
    for (int64_t w = w0; w < items; w += nw) {
      int64_t r, k;
      im.split(w, r, k);
      if (skipped(s.skip_dst, __ldg(s.csr_roots + r))) continue;
      int32_t lo, hi;
      csr_piece(s, r, q, lo, hi);
      if (lo >= hi) continue;
      const int64_t ro = static_cast<int64_t>(__ldg(s.csr_roots + r)) * bl + k;
      const T acc = csr_warp_range<T, OP>(s, leaf, stage, aux, bl, k, lo, hi, root[ro], fetch);
      if (lane == 0) root[ro] = acc;
    }
  }
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// LL128 acknowledgements: the acknowledged LL lines were all read (their
// values consumed) before the last CTA arrived, and a peer only reuses that
// parity two messages later, so no system fence is needed (a MEMBAR.SYS at
// the end of every receiving launch would lengthen each exchange).
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread 0 acquires every selected flag (system scope: written by a peer GPU
// over NVLink), then the CTA proceeds. A peer that never signals (it died or
// broke the collective order) ends in a trap after 30 s, not a hang.
__device__ __forceinline__ void wait_flags(const LaunchParams& P, uint32_t mask) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = global_ns();
    for (uint32_t m = mask; m; m &= m - 1) {
      const FlagWait& w = P.waits[__ffs(m) - 1];
      const long long want = static_cast<long long>(*w.count) + w.delta;
      if (want <= 0) continue;
      const unsigned long long need = static_cast<unsigned long long>(want);
      while (ld_acquire_sys(w.flag) < need) {
        __nanosleep(32);
        if (global_ns() - t0 > 30000000000ull) {
          printf("sfgpu p2p: peer flag stuck at %llu < %llu\n", ld_acquire_sys(w.flag), need);
          __trap();
        }
      }
    }
  }
  __syncthreads();
}

// CTA arrival counter with acquire-release semantics at GPU scope: orders
// this CTA's prior loads and stores (peer stores over NVLink included) before
// the increment, and everything the last CTA observed before its own
// system-scope release. The PTX memory model makes causality transitive
// across scopes (CTA barrier -> GPU-scope atomic -> system-scope release ->
// the peer's system-scope acquire), so one MEMBAR.SYS by the last CTA
// replaces a fence.sc.sys per CTA — measured on B200 (scripts/p2p_microbench.cu,
// profiles/r1_p2p_microbench.md): 2 MB put + flag 13.0 us -> 6.5 us, 8 B
// put + flag 5.1 us -> 3.7 us.
__device__ __forceinline__ unsigned int cta_arrive(unsigned int* counter) {
  unsigned int prev;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counter) : "memory");
  return prev;
}

// Launch completion: the last CTA raises every done flag (after all CTAs'
// reads of the slot and stores).
__device__ __forceinline__ void signal_launch_done(const LaunchParams& P) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  // LL128 acknowledgements (done_relaxed): every CTA's reads of the lines
  // returned their values before it arrives, so a relaxed arrival suffices
  // (an acq_rel one waits for each CTA's stores to drain, ~1.5 us at the end
  // of every receiving launch, measured with SFG_TRACE_LAUNCHES).
  const unsigned prev = P.done_relaxed ? atomicAdd(P.done_count, 1u) : cta_arrive(P.done_count);
  if (prev + 1 == gridDim.x) {
    *P.done_count = 0u;
    for (int i = 0; i < P.ndone; ++i) {
      const unsigned long long v = *P.done_seq[i] + 1;
      *P.done_seq[i] = v;
      if (P.done_relaxed)
        st_relaxed_sys(P.done_flag[i], v);
      else
        st_release_sys(P.done_flag[i], v);
    }
  }
}

// Put completion: every CTA of the segment counts itself in after its stores
// (into the peer's slot over NVLink); the last one publishes the segment's
// flag with a system-scope release store, which the receiving GPU's unpack
// kernel acquires (wait_flags).
__device__ __forceinline__ void signal_segment_done(const DSeg& seg, int64_t nblk) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (static_cast<int64_t>(cta_arrive(seg.sig_count)) + 1 == nblk) {
    *seg.sig_count = 0u;  // ready for the next launch on this stream
    const unsigned long long v = *seg.sig_seq + 1;
    *seg.sig_seq = v;
    st_release_sys(seg.sig_flag, v);
  }
}

// Debug trace: word k of the launch's slot keeps max(value); start times are
// stored as ~t so that max() keeps the earliest.
__device__ __forceinline__ void trace_mark(unsigned long long* slot, int k, unsigned long long v) {
  if (slot != nullptr && threadIdx.x == 0) atomicMax(slot + k, v);
}

// ------------------------------------------------------------ LL128 (p2p)
__device__ __forceinline__ void st_v2_volatile(unsigned long long* p, unsigned long long a,
                                               unsigned long long b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_v2_volatile(const unsigned long long* p, unsigned long long& a,
                                               unsigned long long& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Message number of this CTA's segment: *counter + 1 (the counter advances
// only after every CTA of the segment / launch has arrived).
__device__ __forceinline__ unsigned long long ll_message(const unsigned long long* counter) {
  __shared__ unsigned long long m;
  __syncthreads();
  if (threadIdx.x == 0) m = *counter + 1;
  __syncthreads();
  return m;
}

// Put: word w of the message = word (w % wpv) of vertex src[pat(w / wpv)].
// A CTA covers kLLLines lines: warp q, iteration u, lane l writes words
// 2j, 2j+1 (j = l % 8) of line 4*(kLLIters*q + u) + l/8; lane 7 of each line
// carries the flag m in word 15. All source loads of a thread are issued
// before its stores.
__device__ __forceinline__ void run_put_ll(const DSeg& s, const LaunchParams& P, int64_t blk) {
  // One thread reads the channel counter once, waits (relaxed polls: the
  // lines carry their own validity) until the peer acknowledged message m-2,
  // and publishes m to the CTA: a single barrier before the first store.
  __shared__ unsigned long long msh;
  if (threadIdx.x == 0) {
    const unsigned long long seq = *s.sig_seq;
    if (s.ll_credit != nullptr && seq >= 1) {
      const unsigned long long t0 = global_ns();
      while (ld_volatile_u64(s.ll_credit) + 1 < seq) {
        __nanosleep(32);
        if (global_ns() - t0 > 30000000000ull) {
          printf("sfgpu p2p: LL128 credit stuck at %llu < %llu\n", ld_volatile_u64(s.ll_credit), seq - 1);
          __trap();
        }
      }
    }
    msh = seq + 1;
  }
  __syncthreads();
  const unsigned long long m = msh;
  // descriptor fields in registers (the shared-memory copy is re-read after
  // every volatile store otherwise)
  const DPat sp = s.src;
  const auto* src = static_cast<const unsigned long long*>(P.bufs[s.src_buf]);
  auto* dst = static_cast<unsigned long long*>(P.bufs[s.dst_buf]) + static_cast<int64_t>(m & 1) * s.ll_par +
              s.ll_line * 16;
  const int64_t wpv = P.wpv;
  const int64_t W = s.n * wpv;
  const int64_t lines = (W + 14) / 15;
  const int lane = threadIdx.x & 31;
  const int j = lane & 7;
  // One chunk of kLLLines lines starting at the warp's line L0.
  auto chunk = [&](const int64_t L0) {
    unsigned long long a[kLLIters], b[kLLIters];
#pragma unroll
    for (int u = 0; u < kLLIters; ++u) {
      const int64_t L = L0 + 4 * u;
      const int64_t w0 = L * 15 + 2 * j;
      a[u] = 0;
      b[u] = m;
      if (sp.kind == PAT_CONTIG) {  // the common case: one contiguous run of words
        const unsigned long long* base = src + sp.start * wpv;
        if (L < lines && w0 < W) a[u] = base[w0];
        if (L < lines && j != 7 && w0 + 1 < W) b[u] = base[w0 + 1];
        continue;
      }
      if (L < lines && w0 < W) {
        const int64_t i = wpv == 1 ? w0 : w0 / wpv;
        a[u] = src[pat_index(sp, i) * wpv + (w0 - i * wpv)];
      }
      if (L < lines && j != 7 && w0 + 1 < W) {
        const int64_t i = wpv == 1 ? w0 + 1 : (w0 + 1) / wpv;
        b[u] = src[pat_index(sp, i) * wpv + (w0 + 1 - i * wpv)];
      }
    }
#pragma unroll
    for (int u = 0; u < kLLIters; ++u) {
      const int64_t L = L0 + 4 * u;
      if (L < lines) st_v2_volatile(dst + L * 16 + 2 * j, a[u], b[u]);
    }
  };
  const int64_t off = (threadIdx.x >> 5) * (4 * kLLIters) + (lane >> 3);
  if (s.ll_loop <= 1) {
    chunk(blk * kLLLines + off);
    return;
  }
  for (int64_t c = blk * s.ll_loop; c < (blk + 1) * s.ll_loop; ++c) {
    const int64_t L0 = c * kLLLines + off;
    if (__all_sync(0xffffffffu, L0 >= lines)) break;
    chunk(L0);
  }
}

// Receive: poll this thread's lines until every flag is m, then apply each
// data word's elements to dst[pat(vertex)] (op; REPLACE copies).
template <class T, int OP, class PP = LaunchParams>
__device__ __forceinline__ void run_recv_ll(const DSeg& s, const PP& P, int64_t blk) {
  const unsigned long long m = ll_message(s.sig_seq);
  const DPat dp = s.dst;
  const auto* reg = static_cast<const unsigned long long*>(P.bufs[s.src_buf]) + static_cast<int64_t>(m & 1) * s.ll_par +
                    s.ll_line * 16;
  T* dst = static_cast<T*>(P.bufs[s.dst_buf]);
  constexpr int kEpw = 8 / static_cast<int>(sizeof(T));  // elements per word
  const int64_t wpv = P.wpv;
  const int64_t W = s.n * wpv;
  const int64_t lines = (W + 14) / 15;
  const int lane = threadIdx.x & 31;
  const int j = lane & 7;
  const int64_t L0 = blk * kLLLines + (threadIdx.x >> 5) * (4 * kLLIters) + (lane >> 3);
  if (__all_sync(0xffffffffu, L0 >= lines)) return;
  const int64_t bl = P.bl;
  // Destination of every element this lane may receive, computed before the
  // data arrives (2 words per line group, kEpw elements per word); for a
  // reduction the old values are loaded up front too, so applying a line
  // group that lands costs no further memory round trip.
  constexpr int kE = kLLIters * 2 * kEpw;
  T* dptr[kE];
  T old[kE];
#pragma unroll
  for (int u = 0; u < kLLIters; ++u) {
    const int64_t w0 = (L0 + 4 * u) * 15 + 2 * j;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t w = w0 + q;
      const bool valid = L0 + 4 * u < lines && !(q == 1 && j == 7) && w < W;
#pragma unroll
      for (int t = 0; t < kEpw; ++t) {
        const int x = (u * 2 + q) * kEpw + t;
        dptr[x] = nullptr;
        if (!valid) continue;
        const int64_t e = w * kEpw + t;  // element index in the message
        const int64_t i = bl == 1 ? e : e / bl;
        const int64_t k = e - i * bl;
        dptr[x] = dst + pat_index(dp, i) * bl + k;
        if constexpr (OP != OP_REPLACE) old[x] = *dptr[x];
      }
    }
  }
  auto apply = [&](int u, unsigned long long a, unsigned long long b) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const unsigned long long word = q == 0 ? a : b;
#pragma unroll
      for (int t = 0; t < kEpw; ++t) {
        const int x = (u * 2 + q) * kEpw + t;
        if (dptr[x] == nullptr) continue;
        T v;
        if constexpr (sizeof(T) == 8) {
          v = *reinterpret_cast<const T*>(&word);
        } else {
          const uint32_t part = static_cast<uint32_t>(word >> (32 * t));
          v = *reinterpret_cast<const T*>(&part);
        }
        if constexpr (OP == OP_REPLACE)
          *dptr[x] = v;
        else
          *dptr[x] = apply_op<T, OP>(old[x], v);
      }
    }
  };
  // Poll the warp's line groups; unpack each group as soon as all 4 of its
  // lines carry flag m (warp-uniform decisions), re-read only the others.
  unsigned pending = 0;
#pragma unroll
  for (int u = 0; u < kLLIters; ++u)
    if (__any_sync(0xffffffffu, L0 + 4 * u < lines)) pending |= 1u << u;
  const unsigned long long t0 = global_ns();
  unsigned long long a[kLLIters], b[kLLIters];
  while (pending) {
    // all pending loads in flight at once (one L2 round trip per poll) ...
#pragma unroll
    for (int u = 0; u < kLLIters; ++u) {
      const int64_t L = L0 + 4 * u;
      a[u] = 0;
      b[u] = m;
      if (((pending >> u) & 1u) && L < lines) ld_v2_volatile(reg + L * 16 + 2 * j, a[u], b[u]);
    }
    // ... then every group whose 4 lines all carry m is unpacked at once
#pragma unroll
    for (int u = 0; u < kLLIters; ++u) {
      if (!((pending >> u) & 1u)) continue;
      const unsigned long long f = __shfl_sync(0xffffffffu, b[u], (lane & ~7) | 7);  // every lane
      if (__all_sync(0xffffffffu, f == m)) {
        apply(u, a[u], b[u]);
        pending &= ~(1u << u);
      }
    }
    if (pending) {
      __nanosleep(P.ll_poll_ns);
      if (global_ns() - t0 > 30000000000ull) {
        if (lane == 0) printf("sfgpu p2p: LL128 line never arrived (message %llu)\n", m);
        __trap();
      }
    }
  }
  if constexpr (std::is_same_v<PP, LaunchParams>)
    if (P.trace && lane == 0) atomicMax(P.trace + 3, global_ns());
}

// LL128 put completion: no flag (every line carries its own); the last CTA
// of the segment advances the channel's message counter.
// The counter is only read by later launches (ordered by the kernel
// boundary), so the arrival is a relaxed atomic: an acq_rel one would make
// every put CTA wait for the acknowledgement of its NVLink stores.
__device__ __forceinline__ void count_put_ll(const DSeg& seg, int64_t nblk) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (static_cast<int64_t>(atomicAdd(seg.sig_count, 1u)) + 1 == nblk) {
    *seg.sig_count = 0u;
    *seg.sig_seq = *seg.sig_seq + 1;
  }
}

// Programmatic dependent launch: every library kernel is launched with
// programmatic stream serialization and starts by (1) allowing its own
// dependent launch to be scheduled (all of this grid's CTAs have then started,
// so the dependent's waiting CTAs never take a slot this grid still needs) and
// (2) waiting until the previous kernel on the stream has completed and its
// memory is visible — the same guarantee as a plain kernel boundary, with the
// launch latency of back-to-back exchanges overlapped.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// FULL = the launch contains root-sorted (CSR) or fetch segments. Pair-only
// launches (every pack, unpack and structured local scatter) get their own
// instantiation so the CSR paths do not raise their register allocation.
// MODE 0: pair segments only (4 CTAs/SM); 1 (FULL): CSR / fetch segments
// too (3 CTAs/SM); 2: pair + LL128 put/receive segments (2 CTAs/SM: the
// receive keeps 4 lines x 16 bytes per lane in flight without spilling);
// 3: the same for large exchanges at 3 CTAs/SM (80 registers, a 32-byte
// spill): more put and receive CTAs in flight beat the spill once a launch
// moves >= kLLWideLines lines (2048^3 halo Bcast at N=2 66.4 -> 57.8 us), not
// below (512^3: 9.2 -> 9.4 us).
template <class T, int OP, int MODE>
__global__ void __launch_bounds__(kThreads, MODE == 0 ? 4 : MODE == 1 ? 3 : MODE == 2 ? 2 : 3)
    segments_kernel(const __grid_constant__ LaunchParams P) {
  pdl_enter();
  constexpr bool FULL = MODE == 1;
  int64_t b = blockIdx.x;
  if (P.ilv_a > 0) {  // interleave group A (puts, local) with group B (receives)
    const int64_t na = P.ilv_a, nb = static_cast<int64_t>(gridDim.x) - na;
    const int64_t m = na < nb ? na : nb;
    if (b < 2 * m)
      b = (b & 1) ? na + (b >> 1) : (b >> 1);
    else
      b = na > nb ? b - m : b;  // the rest of the larger group, in order
  }
  const unsigned long long t_start = P.trace ? global_ns() : 0;
  int s = 0;
  while (s + 1 < P.nseg && b >= P.block_start[s + 1]) ++s;
  // The CTA's segment descriptor, copied once into shared memory: reading it
  // straight from the parameter block with a run-time segment index costs
  // indexed constant loads and register pressure (a 64-byte stack frame) in
  // every item loop — the single-segment form without it (pair_solo) ran
  // the config 1 gather 20 % faster.
  // (raw storage: a __shared__ DSeg would not run DSeg's member initialisers,
  // and must not)
  __shared__ alignas(8) unsigned long long sseg[sizeof(DSeg) / 8];
  static_assert(sizeof(DSeg) % 8 == 0, "DSeg copied as 8-byte words");
  if (threadIdx.x < sizeof(DSeg) / 8) sseg[threadIdx.x] = reinterpret_cast<const unsigned long long*>(&P.seg[s])[threadIdx.x];
  __syncthreads();
  const DSeg& seg = *reinterpret_cast<const DSeg*>(sseg);
  const int64_t blk = b - P.block_start[s];
  if (seg.wait_mask) wait_flags(P, seg.wait_mask);
  switch (seg.type) {
    case SEG_PAIR:
      if (seg.run > 0) {
        if (seg.replace)
          run_pair_rows<T, OP_REPLACE, LaunchParams>(seg, P, blk);
        else
          run_pair_rows<T, OP, LaunchParams>(seg, P, blk);
      } else {
        if (seg.replace)
          run_pair<T, OP_REPLACE, LaunchParams>(seg, P, blk);
        else
          run_pair<T, OP, LaunchParams>(seg, P, blk);
      }
      break;
    case SEG_PUT_LL:
      if constexpr (sizeof(T) >= 4 && MODE != 0) run_put_ll(seg, P, blk);
      break;
    case SEG_RECV_LL:
      if constexpr (sizeof(T) >= 4 && MODE != 0) {
        if (seg.replace)
          run_recv_ll<T, OP_REPLACE>(seg, P, blk);
        else
          run_recv_ll<T, OP>(seg, P, blk);
      }
      break;
    case SEG_CSR_FOLD:
      if constexpr (OP != OP_REPLACE && FULL) {
        if (seg.csr_warp)
          run_csr_warp<T, OP>(seg, P, blk, false);
        else
          run_csr<T, OP>(seg, P, blk, false);
      }
      break;
    case SEG_CSR_FETCH:
      if constexpr (OP != OP_REPLACE && FULL) {
        if (seg.csr_warp)
          run_csr_warp<T, OP>(seg, P, blk, true);
        else
          run_csr<T, OP>(seg, P, blk, true);
      }
      break;
    default:
      break;
  }
  if (P.trace) {
    const unsigned long long t_end = global_ns();
    const int k = seg.type == SEG_PUT_LL ? 0 : seg.type == SEG_RECV_LL ? 2 : 6;
    trace_mark(P.trace, k, ~t_start);
    if (k == 0) trace_mark(P.trace, 1, t_end);
    if (k == 2) trace_mark(P.trace, 4, t_end);
    trace_mark(P.trace, 7, ~t_start);
  }
  if (seg.type == SEG_PUT_LL)
    count_put_ll(seg, P.block_start[s + 1] - P.block_start[s]);
  else if (seg.sig_flag != nullptr)
    signal_segment_done(seg, P.block_start[s + 1] - P.block_start[s]);
  if (P.ndone > 0) signal_launch_done(P);
  if (P.trace) trace_mark(P.trace, 5, global_ns());
}

// A launch that is one thread-per-root CSR segment runs in its own kernel,
// specialised for fold or fetch, at <= 64 registers (4 CTAs/SM): many roots
// in flight per SM plus the software-pipelined entry loads hide the latency
// of the per-root chains.
template <class T, int OP, bool FETCH>
__global__ void __launch_bounds__(kThreads, 4) csr_kernel(const __grid_constant__ LaunchParams P) {
  pdl_enter();
  const DSeg& seg = P.seg[0];
  if (seg.wait_mask) wait_flags(P, seg.wait_mask);
  if constexpr (OP != OP_REPLACE) run_csr_t<T, OP, 8, FETCH, LaunchParams>(seg, P, blockIdx.x);
  if (P.ndone > 0) signal_launch_done(P);
}

// A launch that is ONE pair or CSR segment with no p2p waits or signals (a
// local scatter, a gather, a self-only fold) runs from a compact parameter
// block (~0.6 KB instead of LaunchParams' ~5 KB).
struct SoloParams {
  DSeg seg;
  void* bufs[BUF_COUNT];
  int64_t bl = 1;
  FastDiv bldiv;
  int64_t wpv = 1;
  FetchShuffle shuf;
};

template <class T, int OP>
__global__ void __launch_bounds__(kThreads, 4) pair_solo(const __grid_constant__ SoloParams P) {
  pdl_enter();
  if (P.seg.run > 0)
    run_pair_rows<T, OP, SoloParams>(P.seg, P, blockIdx.x);
  else
    run_pair<T, OP, SoloParams>(P.seg, P, blockIdx.x);
}

template <class T, int OP, bool FETCH>
__global__ void __launch_bounds__(kThreads, 4) csr_solo(const __grid_constant__ SoloParams P) {
  pdl_enter();
  if constexpr (OP != OP_REPLACE) run_csr_t<T, OP, 8, FETCH, SoloParams>(P.seg, P, blockIdx.x);
}

bool solo_ok(const LaunchParams& p) {
  if (p.nseg != 1 || p.ndone != 0) return false;
  const DSeg& g = p.seg[0];
  if (g.wait_mask || g.sig_flag || g.sig_count) return false;
  return g.type == SEG_PAIR || ((g.type == SEG_CSR_FOLD || g.type == SEG_CSR_FETCH) && !g.csr_warp);
}

SoloParams solo_of(const LaunchParams& p) {
  SoloParams q;
  q.seg = p.seg[0];
  for (int b = 0; b < BUF_COUNT; ++b) q.bufs[b] = p.bufs[b];
  q.bl = p.bl;
  q.bldiv = p.bldiv;
  q.wpv = p.wpv;
  q.shuf = p.shuf;
  return q;
}

// Launch, with programmatic stream serialization when `pdl` (see pdl_enter):
// the exchange launches (LL128 put/receive) and the signalling kernel, whose
// back-to-back launches are latency-bound; local bulk work launches plainly
// (PDL there measured -2 % on the N=2 headline step). SFG_NO_PDL=1 turns it
// off (ablation). Errors surface through cudaGetLastError like <<<>>>.
bool pdl_on() {
  static const bool on = std::getenv("SFG_NO_PDL") == nullptr;
  return on;
}
template <class... K, class... A>
void launch_k(void (*kernel)(K...), int64_t blocks, int threads, cudaStream_t st, bool pdl, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl && pdl_on() ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

template <class T, int OP>
void launch_t(const LaunchParams& p, int64_t blocks, cudaStream_t st) {
  bool full = false;  // CSR / fetch segments present
  for (int s = 0; s < p.nseg; ++s)
    full = full || p.seg[s].type == SEG_CSR_FOLD || p.seg[s].type == SEG_CSR_FETCH;
  static const bool no_solo = std::getenv("SFG_NO_SOLO") != nullptr;  // ablation
  if (!no_solo && solo_ok(p)) {
    const SoloParams q = solo_of(p);
    if (p.seg[0].type == SEG_PAIR) {
      if (p.seg[0].replace)
        launch_k(pair_solo<T, OP_REPLACE>, blocks, kThreads, st, false, q);
      else
        launch_k(pair_solo<T, OP>, blocks, kThreads, st, false, q);
      return;
    }
    if constexpr (OP != OP_REPLACE && (std::is_same_v<T, double> || std::is_same_v<T, int64_t> ||
                                       std::is_same_v<T, int32_t>)) {
      if (p.seg[0].type == SEG_CSR_FETCH)
        launch_k(csr_solo<T, OP, true>, blocks, kThreads, st, false, q);
      else
        launch_k(csr_solo<T, OP, false>, blocks, kThreads, st, false, q);
      return;
    }
  }
  bool ll = false;
  int64_t ll_lines = 0;
  for (int s = 0; s < p.nseg; ++s)
    if (p.seg[s].type == SEG_PUT_LL || p.seg[s].type == SEG_RECV_LL) {
      ll = true;
      ll_lines += (p.seg[s].n * p.wpv + 14) / 15;
    }
  static const int64_t wide_lines = [] {  // ablation / override
    const char* e = std::getenv("SFG_LL_WIDE_LINES");
    return e ? std::atoll(e) : kLLWideLines;
  }();
  if (ll && !full && ll_lines >= wide_lines) {
    launch_k(segments_kernel<T, OP, 3>, blocks, kThreads, st, true, p);
  } else if (ll && !full) {
    launch_k(segments_kernel<T, OP, 2>, blocks, kThreads, st, true, p);
  } else if constexpr (OP == OP_REPLACE) {
    launch_k(segments_kernel<T, OP, 0>, blocks, kThreads, st, false, p);
  } else if (p.nseg == 1 && (p.seg[0].type == SEG_CSR_FOLD || p.seg[0].type == SEG_CSR_FETCH) &&
             !p.seg[0].csr_warp && (std::is_same_v<T, double> || std::is_same_v<T, int64_t> ||
                                    std::is_same_v<T, int32_t>)) {
    if (p.seg[0].type == SEG_CSR_FETCH)
      launch_k(csr_kernel<T, OP, true>, blocks, kThreads, st, false, p);
    else
      launch_k(csr_kernel<T, OP, false>, blocks, kThreads, st, false, p);
  } else {
    if (full)
      launch_k(segments_kernel<T, OP, 1>, blocks, kThreads, st, false, p);
    else
      launch_k(segments_kernel<T, OP, 0>, blocks, kThreads, st, false, p);
  }
}

template <class T>
bool launch_int_ops(const LaunchParams& p, int op, int64_t blocks, cudaStream_t st) {
  switch (op) {
    case OP_REPLACE: launch_t<T, OP_REPLACE>(p, blocks, st); return true;
    case OP_SUM: launch_t<T, OP_SUM>(p, blocks, st); return true;
    case OP_PROD: launch_t<T, OP_PROD>(p, blocks, st); return true;
    case OP_MAX: launch_t<T, OP_MAX>(p, blocks, st); return true;
    case OP_MIN: launch_t<T, OP_MIN>(p, blocks, st); return true;
    case OP_LAND: launch_t<T, OP_LAND>(p, blocks, st); return true;
    case OP_LOR: launch_t<T, OP_LOR>(p, blocks, st); return true;
    case OP_BAND: launch_t<T, OP_BAND>(p, blocks, st); return true;
    case OP_BOR: launch_t<T, OP_BOR>(p, blocks, st); return true;
  }
  return false;
}

bool launch_f64_ops(const LaunchParams& p, int op, int64_t blocks, cudaStream_t st) {
  switch (op) {
    case OP_REPLACE: launch_t<double, OP_REPLACE>(p, blocks, st); return true;
    case OP_SUM: launch_t<double, OP_SUM>(p, blocks, st); return true;
    case OP_PROD: launch_t<double, OP_PROD>(p, blocks, st); return true;
    case OP_MAX: launch_t<double, OP_MAX>(p, blocks, st); return true;
    case OP_MIN: launch_t<double, OP_MIN>(p, blocks, st); return true;
  }
  return false;
}

__global__ void digest_kernel(const unsigned char* p, size_t bytes, unsigned long long* out) {
  const size_t nwords = bytes / 8;
  unsigned long long acc = 0;
  const auto* w = reinterpret_cast<const unsigned long long*>(p);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nwords;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    unsigned long long z = w[i] ^ (static_cast<unsigned long long>(i) * 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    acc += z ^ (z >> 31);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (size_t i = nwords * 8; i < bytes; ++i) acc += (static_cast<unsigned long long>(p[i]) + 1) * (i + 7);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

template <class T, int OP>
int64_t resident_full() {
  static const int64_t v = [] {
    int dev = 0, sms = 0, a = 0, b = 0;
    // the smaller residency of the two kernels a CSR segment may run in
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, segments_kernel<T, OP, 1>, kThreads, 0);
    int c = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, csr_kernel<T, OP, false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, csr_kernel<T, OP, true>, kThreads, 0);
    int d1 = 0, d2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d1, csr_solo<T, OP, false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d2, csr_solo<T, OP, true>, kThreads, 0);
    const int per_sm = std::min(std::min(a, std::min(b, c)), std::min(d1, d2));
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return static_cast<int64_t>(std::max(1, per_sm) * std::max(1, sms));
  }();
  return v;
}

template <class T>
int64_t resident_t(int op) {
  switch (op) {
    case OP_SUM: return resident_full<T, OP_SUM>();
    case OP_PROD: return resident_full<T, OP_PROD>();
    case OP_MAX: return resident_full<T, OP_MAX>();
    case OP_MIN: return resident_full<T, OP_MIN>();
    default: break;
  }
  if constexpr (std::is_integral_v<T>) {
    switch (op) {
      case OP_LAND: return resident_full<T, OP_LAND>();
      case OP_LOR: return resident_full<T, OP_LOR>();
      case OP_BAND: return resident_full<T, OP_BAND>();
      case OP_BOR: return resident_full<T, OP_BOR>();
      default: break;
    }
  }
  return 148;
}

// CTAs of the FULL (CSR-capable) instantiation that fit on the GPU at once.
int64_t resident_ctas(ElemType t, int op) {
  switch (t) {
    case ElemType::i32: return resident_t<int32_t>(op);
    case ElemType::i64: return resident_t<int64_t>(op);
    case ElemType::f64: return resident_t<double>(op);
    default: return 148;
  }
}

}  // namespace

int launch_segments(LaunchParams& p, ElemType t, int op, cudaStream_t stream) {
  int64_t blocks = 0;
  int n = 0;
  bool op_recv = false;  // an LL128 receive applies an op (not a copy)
  for (int s = 0; s < p.nseg; ++s) op_recv = op_recv || (p.seg[s].type == SEG_RECV_LL && !p.seg[s].replace);
  for (int s = 0; s < p.nseg; ++s) {
    const int64_t items = p.seg[s].n * p.bl;
    if (items <= 0) continue;
    p.seg[n] = p.seg[s];
    p.block_start[n] = blocks;
    const bool csr = p.seg[s].type == SEG_CSR_FOLD || p.seg[s].type == SEG_CSR_FETCH;
    const bool ll = p.seg[s].type == SEG_PUT_LL || p.seg[s].type == SEG_RECV_LL;
    const int64_t per_block = !csr ? kThreads * kItems : p.seg[n].csr_warp ? kThreads / 32 : kThreads;
    int64_t nb = (items + per_block - 1) / per_block;
    if (ll) {
      // Large puts in a launch whose receives apply an op (a halo Reduce
      // folding contributions as they land) write two chunks per CTA, which
      // leaves the receive CTAs more SM slots: 2048^3 halo Reduce at N=2
      // 79 -> 69 us. A Bcast's copying receives do not gain (66 -> 68 us).
      const int64_t lines = (p.seg[s].n * p.wpv + 14) / 15;
      int64_t loop = 1;
      static const int64_t put_loop = [] {  // ablation / override (any size)
        const char* e = std::getenv("SFG_LL_PUT_LOOP");
        return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(0);
      }();
      if (p.seg[s].type == SEG_PUT_LL)
        loop = put_loop > 0 ? put_loop : op_recv && lines >= 8192 ? 2 : 1;
      p.seg[n].ll_loop = loop;
      nb = (lines + kLLLines * loop - 1) / (kLLLines * loop);
    }
    if (csr && p.seg[n].csr_np > 1) {
      // Piece-major walk: every CTA of the segment must be resident at once.
      const int64_t res = resident_ctas(t, op);
      nb = std::min<int64_t>(nb, res);
      p.seg[n].csr_grid_threads = nb * kThreads;
    }
    blocks += nb;
    ++n;
  }
  p.nseg = n;
  p.block_start[n] = blocks;
  if (blocks == 0) return 0;
  if (p.ilv_a < 0) {
    // Only when the CTAs ahead of the receives are streaming work (no
    // indexed gather or scatter): receive CTAs that spin among put CTAs doing
    // random gathers take SM slots those gathers need (config 4 at N=4:
    // Reduce 143 -> 174 us with interleaving), while structured puts finish
    // at the rate the link drains them anyway.
    static const int mode = [] {
      const char* e = std::getenv("SFG_LL_INTERLEAVE");  // ablation: "all" | "none"
      return e == nullptr ? 0 : std::strcmp(e, "all") == 0 ? 1 : std::strcmp(e, "none") == 0 ? 2 : 0;
    }();
    p.ilv_a = 0;
    for (int s = 1; s < n && mode != 2; ++s)
      if (p.seg[s].type == SEG_RECV_LL) {
        bool ok = true;  // receives must be the trailing segments
        for (int t = s; t < n; ++t) ok = ok && p.seg[t].type == SEG_RECV_LL;
        for (int t = 0; t < s && mode == 0; ++t)
          ok = ok && (p.seg[t].type == SEG_PUT_LL || p.seg[t].type == SEG_PAIR) &&
               p.seg[t].src.kind != PAT_INDEXED && p.seg[t].dst.kind != PAT_INDEXED;
        if (ok) p.ilv_a = p.block_start[s];
        break;
      }
  }
  p.bldiv = make_fastdiv(static_cast<uint32_t>(p.bl > 0x7fffffff ? 1 : p.bl));
  bool ok = false;
  switch (t) {
    case ElemType::u8: ok = op == OP_REPLACE && (launch_t<uint8_t, OP_REPLACE>(p, blocks, stream), true); break;
    case ElemType::u16: ok = op == OP_REPLACE && (launch_t<uint16_t, OP_REPLACE>(p, blocks, stream), true); break;
    case ElemType::u32: ok = op == OP_REPLACE && (launch_t<uint32_t, OP_REPLACE>(p, blocks, stream), true); break;
    case ElemType::u64: ok = op == OP_REPLACE && (launch_t<uint64_t, OP_REPLACE>(p, blocks, stream), true); break;
    case ElemType::i32: ok = launch_int_ops<int32_t>(p, op, blocks, stream); break;
    case ElemType::i64: ok = launch_int_ops<int64_t>(p, op, blocks, stream); break;
    case ElemType::f64: ok = launch_f64_ops(p, op, blocks, stream); break;
  }
  if (!ok) return -1;
  return 1;
}

constexpr int kFlagBatch = 64;
struct FlagBatch {
  int n = 0;
  unsigned long long* flag[kFlagBatch];
  unsigned long long* seq[kFlagBatch];
};

__global__ void quiesce_kernel(const __grid_constant__ FlagBatch q, unsigned long long timeout_ns) {
  const int i = threadIdx.x;
  if (i >= q.n) return;
  const unsigned long long t0 = global_ns();
  const unsigned long long need = *q.seq[i];
  while (ld_acquire_sys(q.flag[i]) < need) {
    __nanosleep(256);
    if (global_ns() - t0 > timeout_ns) {
      printf("sfgpu p2p: teardown gave up waiting for a peer acknowledgement (%llu < %llu)\n",
             ld_acquire_sys(q.flag[i]), need);
      return;
    }
  }
}

__global__ void signal_kernel(const __grid_constant__ FlagBatch q) {
  pdl_enter();
  for (int i = 0; i < q.n; ++i) {
    const unsigned long long v = *q.seq[i] + 1;
    *q.seq[i] = v;
    st_release_sys(q.flag[i], v);
  }
}

template <class K>
void batched(unsigned long long* const* flag, unsigned long long* const* seq, int n, K&& k) {
  for (int b = 0; b < n; b += kFlagBatch) {
    FlagBatch q;
    q.n = std::min(kFlagBatch, n - b);
    for (int i = 0; i < q.n; ++i) {
      q.flag[i] = flag[b + i];
      q.seq[i] = seq[b + i];
    }
    k(q);
  }
}

namespace {
struct TraceBuf {
  unsigned long long* dev = nullptr;
  int cap = 0;
  std::atomic<int> next{0};  // thread ranks launch concurrently
  TraceBuf() {
    const char* e = std::getenv("SFG_TRACE_LAUNCHES");
    cap = e ? std::atoi(e) : 0;
    if (cap > 0 && cudaMalloc(&dev, static_cast<size_t>(cap) * 64) == cudaSuccess)
      cudaMemset(dev, 0, static_cast<size_t>(cap) * 64);
    else
      cap = 0;
  }
};
TraceBuf& tbuf() {
  static TraceBuf t;
  return t;
}
}  // namespace

void trace_init() { (void)tbuf(); }

unsigned long long* trace_slot() {
  TraceBuf& t = tbuf();
  if (t.cap == 0) return nullptr;
  const int k = t.next.fetch_add(1);
  return k < t.cap ? t.dev + 8 * static_cast<size_t>(k) : nullptr;
}

void trace_dump(const char* path) {
  TraceBuf& t = tbuf();
  if (t.cap == 0) return;
  const int used = std::min(t.next.load(), t.cap);
  std::vector<unsigned long long> h(static_cast<size_t>(used) * 8);
  cudaDeviceSynchronize();
  if (!h.empty()) cudaMemcpy(h.data(), t.dev, h.size() * 8, cudaMemcpyDeviceToHost);
  FILE* f = std::fopen(path, "w");
  if (!f) return;
  auto st = [](unsigned long long v) { return v ? ~v : 0ull; };
  for (int i = 0; i < used; ++i) {
    const unsigned long long* w = h.data() + 8 * static_cast<size_t>(i);
    std::fprintf(f, "{\"launch\":%d,\"first_start\":%llu,\"put_start\":%llu,\"put_end\":%llu,"
                 "\"recv_start\":%llu,\"recv_ready\":%llu,\"recv_end\":%llu,\"end\":%llu,\"other_start\":%llu}\n",
                 i, st(w[7]), st(w[0]), w[1], st(w[2]), w[3], w[4], w[5], st(w[6]));
  }
  std::fclose(f);
}

void launch_signal(unsigned long long* const* flag, unsigned long long* const* seq, int n, cudaStream_t s) {
  batched(flag, seq, n, [&](const FlagBatch& q) { launch_k(signal_kernel, 1, 1, s, true, q); });
}

void launch_quiesce(const unsigned long long* const* flag, const unsigned long long* const* count, int n,
                    double timeout_s, cudaStream_t s) {
  batched(const_cast<unsigned long long* const*>(flag), const_cast<unsigned long long* const*>(count), n,
          [&](const FlagBatch& q) {
            quiesce_kernel<<<1, kFlagBatch, 0, s>>>(q, static_cast<unsigned long long>(timeout_s * 1e9));
          });
}

void launch_digest(const void* p, size_t bytes, unsigned long long* out_dev, cudaStream_t s) {
  cudaMemsetAsync(out_dev, 0, sizeof(unsigned long long), s);
  if (bytes == 0) return;
  size_t words = bytes / 8;
  int blocks = static_cast<int>(words / (256 * 8) + 1);
  if (blocks > 148 * 8) blocks = 148 * 8;
  digest_kernel<<<blocks, 256, 0, s>>>(static_cast<const unsigned char*>(p), bytes, out_dev);
}

}  // namespace sfg
