// TEST/BASELINE INFRASTRUCTURE ONLY — C entry points onto the UNMODIFIED
// reference library (/root/reference/proj/src/*.cpp), compiled from where
// the sources lie by oracle/Makefile into oracle/_ref/libsfref.so.
//
// Used to (1) pin the C oracle restatement against the reference's own
// distributed CPU path on identical graphs and data, (2) generate golden
// fixtures (tests/golden/make_golden.py), and (3) time the reference CPU
// path for bench.py's reference arm / cpu_baseline. Never used by the
// product package.
//
// Everything here calls the reference's public API: sf::run_ranks
// (harness.hpp:58-72), StarForest::set_graph/setup (starforest.hpp:71-79)
// and the ops in ops.hpp:57-94.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "sf/bench.hpp"
#include "sf/harness.hpp"
#include "sf/rng.hpp"
#include "sf/ops.hpp"
#include "sf/spmv.hpp"
#include "sf/starforest.hpp"

namespace {
thread_local std::string g_err;

sf::GraphSpec make_spec(int r, const int64_t* nroots, const int64_t* nleaves,
                        const int64_t* const* local, const int32_t* const* rrank,
                        const int64_t* const* roff) {
  sf::GraphSpec s;
  s.nroots = nroots[r];
  s.nleaves = nleaves[r];
  if (local && local[r]) s.local = std::vector<int64_t>(local[r], local[r] + nleaves[r]);
  s.remote.resize(static_cast<size_t>(nleaves[r]));
  for (int64_t i = 0; i < nleaves[r]; ++i) s.remote[static_cast<size_t>(i)] = sf::RootRef{rrank[r][i], roff[r][i]};
  return s;
}
}  // namespace

extern "C" {

const char* sfref_last_error() { return g_err.c_str(); }

// opkind: 0 bcast(a=root in, b=leaf inout), 1 reduce(a=leaf in, b=root inout),
// 2 fetch_and_op(a=root inout, b=leaf in, c=leafupdate inout),
// 3 gather(a=leaf in, b=multiroot out), 4 scatter(a=multiroot in, b=leaf inout)
int sfref_run(int nranks, const int64_t* nroots, const int64_t* nleaves,
              const int64_t* const* local, const int32_t* const* rrank,
              const int64_t* const* roff, int opkind, int kind, int64_t blocklen, int op,
              int deterministic, int force_remote, uint64_t seed, void* const* a, void* const* b,
              void* const* c) {
  try {
    sf::RunConfig cfg;
    cfg.nranks = nranks;
    cfg.deterministic = deterministic != 0;
    cfg.force_remote = force_remote != 0;
    cfg.seed = seed;
    cfg.timeout_s = 60.0;
    const sf::Unit u{static_cast<sf::Kind>(kind), blocklen};
    const auto rop = static_cast<sf::ReduceOp>(op);
    sf::run_ranks(cfg, [&](sf::Comm& comm) {
      const int r = comm.rank();
      sf::StarForest f(comm);
      f.set_graph(make_spec(r, nroots, nleaves, local, rrank, roff));
      f.setup();
      switch (opkind) {
        case 0: sf::bcast(f, u, a[r], b[r], rop); break;
        case 1: sf::reduce(f, u, a[r], b[r], rop); break;
        case 2: sf::fetch_and_op(f, u, a[r], b[r], c[r], rop); break;
        case 3: sf::gather(f, u, a[r], b[r]); break;
        case 4: sf::scatter(f, u, a[r], b[r]); break;
        default: throw sf::Error("unknown opkind");
      }
    });
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Two-sided info of every rank (starforest.hpp:47-55) flattened as
// [ngroups, (rank, n, items...)...] for root groups then leaf groups.
int sfref_two_sided(int nranks, const int64_t* nroots, const int64_t* nleaves,
                    const int64_t* const* local, const int32_t* const* rrank,
                    const int64_t* const* roff, int64_t* const* out, const int64_t* out_cap) {
  try {
    sf::RunConfig cfg;
    cfg.nranks = nranks;
    sf::run_ranks(cfg, [&](sf::Comm& comm) {
      const int r = comm.rank();
      sf::StarForest f(comm);
      f.set_graph(make_spec(r, nroots, nleaves, local, rrank, roff));
      f.setup();
      std::vector<int64_t> v;
      const auto& ti = f.two_sided();
      for (const auto* gs : {&ti.root_ranks, &ti.leaf_ranks}) {
        v.push_back(static_cast<int64_t>(gs->size()));
        for (const auto& g : *gs) {
          v.push_back(g.rank);
          v.push_back(static_cast<int64_t>(g.items.size()));
          v.insert(v.end(), g.items.begin(), g.items.end());
        }
      }
      if (static_cast<int64_t>(v.size()) > out_cap[r]) throw sf::Error("two_sided: output too small");
      std::memcpy(out[r], v.data(), v.size() * sizeof(int64_t));
    });
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Time `steps` iterations of Bcast(REPLACE) + Reduce(SUM) on float64 data
// over the given graph with the reference's threads backend (one thread per
// rank, single-threaded per rank by design). Timing per rank with
// steady_clock between barriers; out[0] = max SetUp seconds, out[1] = max over
// ranks of mean microseconds per step, out[2] = mean bcast us, out[3] = mean
// reduce us (rank 0).
int sfref_time_bcast_reduce(int nranks, const int64_t* nroots, const int64_t* nleaves,
                            const int64_t* const* local, const int32_t* const* rrank,
                            const int64_t* const* roff, int steps, int warmup, double* out) {
  try {
    sf::RunConfig cfg;
    cfg.nranks = nranks;
    cfg.timeout_s = 3600.0;
    std::vector<double> setup_s(static_cast<size_t>(nranks)), step_us(static_cast<size_t>(nranks)),
        b_us(static_cast<size_t>(nranks)), r_us(static_cast<size_t>(nranks));
    sf::run_ranks(cfg, [&](sf::Comm& comm) {
      using clk = std::chrono::steady_clock;
      const int r = comm.rank();
      sf::StarForest f(comm);
      f.set_graph(make_spec(r, nroots, nleaves, local, rrank, roff));
      comm.barrier();
      const auto t0 = clk::now();
      f.setup();
      setup_s[static_cast<size_t>(r)] = std::chrono::duration<double>(clk::now() - t0).count();
      std::vector<double> root(static_cast<size_t>(nroots[r])), leaf(static_cast<size_t>(f.leaf_index_bound()));
      for (size_t i = 0; i < root.size(); ++i) root[i] = 1.0 + static_cast<double>(i % 97) * 1e-3;
      for (size_t i = 0; i < leaf.size(); ++i) leaf[i] = 0.0;
      const sf::Unit u = sf::unit_of<double>();
      for (int w = 0; w < warmup; ++w) {
        sf::bcast(f, u, root.data(), leaf.data(), sf::ReduceOp::replace);
        sf::reduce(f, u, leaf.data(), root.data(), sf::ReduceOp::sum);
      }
      double tb = 0, tr = 0;
      comm.barrier();
      const auto s0 = clk::now();
      for (int s = 0; s < steps; ++s) {
        const auto a0 = clk::now();
        sf::bcast(f, u, root.data(), leaf.data(), sf::ReduceOp::replace);
        const auto a1 = clk::now();
        sf::reduce(f, u, leaf.data(), root.data(), sf::ReduceOp::sum);
        const auto a2 = clk::now();
        tb += std::chrono::duration<double, std::micro>(a1 - a0).count();
        tr += std::chrono::duration<double, std::micro>(a2 - a1).count();
      }
      const auto s1 = clk::now();
      comm.barrier();
      step_us[static_cast<size_t>(r)] = std::chrono::duration<double, std::micro>(s1 - s0).count() / steps;
      b_us[static_cast<size_t>(r)] = tb / steps;
      r_us[static_cast<size_t>(r)] = tr / steps;
    });
    double ms = 0, mu = 0;
    for (int r = 0; r < nranks; ++r) {
      ms = std::max(ms, setup_s[static_cast<size_t>(r)]);
      mu = std::max(mu, step_us[static_cast<size_t>(r)]);
    }
    out[0] = ms;
    out[1] = mu;
    out[2] = b_us[0];
    out[3] = r_us[0];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Time `steps` calls of one operation (opkind as sfref_run: 1 reduce, 2
// fetch_and_op, 0 bcast) on the given kind with deterministic data. out[0] =
// max SetUp s, out[1] = max over ranks of mean us per call.
int sfref_time_op(int nranks, const int64_t* nroots, const int64_t* nleaves,
                  const int64_t* const* local, const int32_t* const* rrank,
                  const int64_t* const* roff, int opkind, int kind, int op, int steps, int warmup,
                  double* out) {
  try {
    sf::RunConfig cfg;
    cfg.nranks = nranks;
    cfg.timeout_s = 3600.0;
    std::vector<double> setup_s(static_cast<size_t>(nranks)), us(static_cast<size_t>(nranks));
    sf::run_ranks(cfg, [&](sf::Comm& comm) {
      using clk = std::chrono::steady_clock;
      const int r = comm.rank();
      sf::StarForest f(comm);
      f.set_graph(make_spec(r, nroots, nleaves, local, rrank, roff));
      const auto t0 = clk::now();
      f.setup();
      setup_s[static_cast<size_t>(r)] = std::chrono::duration<double>(clk::now() - t0).count();
      const sf::Unit u{static_cast<sf::Kind>(kind), 1};
      const size_t ub = u.bytes();
      std::vector<unsigned char> root(static_cast<size_t>(nroots[r]) * ub + 8),
          leaf(static_cast<size_t>(f.leaf_index_bound()) * ub + 8),
          upd(static_cast<size_t>(f.leaf_index_bound()) * ub + 8);
      for (size_t i = 0; i + ub <= root.size(); i += ub) {
        if (kind == 2) { double v = 1.0; std::memcpy(&root[i], &v, 8); }
        else root[i] = 1;
      }
      for (size_t i = 0; i + ub <= leaf.size(); i += ub) {
        if (kind == 2) { double v = 0.5; std::memcpy(&leaf[i], &v, 8); }
        else leaf[i] = 1;
      }
      const auto rop = static_cast<sf::ReduceOp>(op);
      auto call = [&] {
        switch (opkind) {
          case 0: sf::bcast(f, u, root.data(), leaf.data(), rop); break;
          case 1: sf::reduce(f, u, leaf.data(), root.data(), rop); break;
          case 2: sf::fetch_and_op(f, u, root.data(), leaf.data(), upd.data(), rop); break;
          default: throw sf::Error("unknown opkind");
        }
      };
      for (int w = 0; w < warmup; ++w) call();
      comm.barrier();
      const auto s0 = clk::now();
      for (int s = 0; s < steps; ++s) call();
      const auto s1 = clk::now();
      comm.barrier();
      us[static_cast<size_t>(r)] = std::chrono::duration<double, std::micro>(s1 - s0).count() / steps;
    });
    out[0] = *std::max_element(setup_s.begin(), setup_s.end());
    out[1] = *std::max_element(us.begin(), us.end());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference's own ping-pong benchmark (bench.cpp:24-100, sf::pingpong):
// sizes min_bytes, 4*min_bytes, ... <= max_bytes; per size out[3*k] = bytes,
// out[3*k+1] = median half round trip (us), out[3*k+2] = min (us). Returns the
// number of rows, -1 on error.
int sfref_pingpong(int64_t min_bytes, int64_t max_bytes, int iters, int warmup, double* out, int cap) {
  try {
    sf::PingPongConfig cfg;
    cfg.min_bytes = min_bytes;
    cfg.max_bytes = max_bytes;
    cfg.iters = iters;
    cfg.warmup = warmup;
    const auto rows = sf::pingpong(cfg);
    int k = 0;
    for (const auto& r : rows) {
      if (k >= cap) break;
      out[3 * k] = static_cast<double>(r.bytes);
      out[3 * k + 1] = r.median_us;
      out[3 * k + 2] = r.min_us;
      ++k;
    }
    return k;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The reference's splitmix64 stream and mix_seed (rng.hpp:14-51), to pin the
// Python port used by the generators.
int sfref_rng(uint64_t seed, int64_t n, uint64_t* out, uint64_t salt, uint64_t* mixed) {
  sf::Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.next();
  *mixed = sf::mix_seed(seed, salt);
  return 0;
}

// random_graph_specs (harness.cpp:148-193) flattened per rank as
// [nroots, nleaves, has_local, local[nleaves] if has_local, (rank, off)*nleaves].
int sfref_random_graph(uint64_t seed, int nranks, int64_t maxv, int64_t* out, int64_t cap) {
  try {
    auto specs = sf::random_graph_specs(seed, nranks, maxv);
    std::vector<int64_t> v;
    for (const auto& s : specs) {
      v.push_back(s.nroots);
      v.push_back(s.nleaves);
      v.push_back(s.local ? 1 : 0);
      if (s.local) v.insert(v.end(), s.local->begin(), s.local->end());
      for (const auto& r : s.remote) {
        v.push_back(r.rank);
        v.push_back(r.offset);
      }
    }
    if (static_cast<int64_t>(v.size()) > cap) throw sf::Error("random_graph: output too small");
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
    return static_cast<int>(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"

namespace {
// spmv_trial's distributed part (selfcheck.cpp:684-723): contiguous row and
// column layouts, split_matrix, build_ghost_sf, spmv / spmv_transpose per
// rank thread; y concatenated in rank order.
template <class T>
void spmv_run(int nranks, int64_t n, const int64_t* rowptr, const int64_t* colind, const T* vals,
              int transpose, const T* x, T* y) {
  sf::Csr<T> g;
  g.rows = n;
  g.cols = n;
  g.rowptr.assign(rowptr, rowptr + n + 1);
  g.colind.assign(colind, colind + rowptr[n]);
  g.vals.assign(vals, vals + rowptr[n]);
  const sf::Layout layout = sf::Layout::contiguous(n, nranks);
  sf::RunConfig cfg;
  cfg.nranks = nranks;
  cfg.timeout_s = 60.0;
  auto pieces = sf::run_ranks(cfg, [&](sf::Comm& comm) {
    const int me = comm.rank();
    auto m = sf::split_matrix(g, layout, layout, me);
    sf::StarForest forest = sf::build_ghost_sf(comm, m);
    sf::GhostVector<T> gx;
    gx.owned.assign(x + layout.begin(me), x + layout.end(me));
    gx.lvec.assign(m.garray.size(), T{});
    std::vector<T> yy(static_cast<size_t>(layout.local_size(me)), T{});
    if (!transpose)
      sf::spmv(m, forest, gx, yy);
    else
      sf::spmv_transpose(m, forest, gx, yy);
    return yy;
  });
  size_t k = 0;
  for (const auto& p : pieces)
    for (T v : p) y[k++] = v;
}
}  // namespace

extern "C" {
// kind: 1 int64, 2 float64 (sfg_kind numbering)
int sfref_spmv(int nranks, int64_t n, const int64_t* rowptr, const int64_t* colind, const void* vals,
               int kind, int transpose, const void* x, void* y) {
  try {
    if (kind == 2)
      spmv_run<double>(nranks, n, rowptr, colind, static_cast<const double*>(vals), transpose,
                       static_cast<const double*>(x), static_cast<double*>(y));
    else
      spmv_run<int64_t>(nranks, n, rowptr, colind, static_cast<const int64_t*>(vals), transpose,
                        static_cast<const int64_t*>(x), static_cast<int64_t*>(y));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
}  // extern "C"

