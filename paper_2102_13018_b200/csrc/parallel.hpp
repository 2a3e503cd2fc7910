// Host-side data parallelism for SetUp-size loops (100M+ edges): [0, n) in
// contiguous chunks, one std::thread per chunk (up to 16, >= 1M items each).
// The bodies must not throw; validation loops return the first offending
// index per chunk and the caller reports it sequentially (same message as
// the reference's sequential check).
#pragma once

#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace sfg {

inline int host_threads() {
  static const int t = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  return t;
}

// f(chunk, begin, end) for nchunks() chunks; returns the chunk count used.
template <class F>
int parallel_chunks(int64_t n, F&& f, int64_t grain = int64_t(1) << 20) {
  const int nt = static_cast<int>(std::min<int64_t>(host_threads(), std::max<int64_t>(1, n / grain)));
  if (nt <= 1) {
    f(0, int64_t(0), n);
    return 1;
  }
  const int64_t step = (n + nt - 1) / nt;
  std::vector<std::thread> th;
  th.reserve(static_cast<size_t>(nt - 1));
  for (int c = 1; c < nt; ++c)
    th.emplace_back([&f, c, step, n] { f(c, std::min(n, c * step), std::min(n, (c + 1) * step)); });
  f(0, int64_t(0), std::min(n, step));
  for (auto& t : th) t.join();
  return nt;
}

// Chunk count parallel_chunks(n) will use (to size per-chunk scratch).
inline int chunk_count(int64_t n, int64_t grain = int64_t(1) << 20) {
  return static_cast<int>(std::min<int64_t>(host_threads(), std::max<int64_t>(1, n / grain)));
}

// First index in [0, n) where bad(i) holds, or n.
template <class Pred>
int64_t parallel_find_first(int64_t n, Pred&& bad) {
  std::vector<int64_t> first(static_cast<size_t>(chunk_count(n)), n);
  parallel_chunks(n, [&](int c, int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i)
      if (bad(i)) {
        first[static_cast<size_t>(c)] = i;
        return;
      }
  });
  return *std::min_element(first.begin(), first.end());
}

}  // namespace sfg
