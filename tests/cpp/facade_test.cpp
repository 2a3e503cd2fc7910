// Drop-in check of the C++ facade (include/sfgpu/sf.hpp): the reference's
// own worked-example tests (tests/test_sfgraph.cpp, test_sfops.cpp) written
// against sf:: exactly as a reference user would, device buffers aside.
//   facade_test host   -> SetUp / degrees / multi-SF / errors, no GPU
//   facade_test gpu    -> operations on cuda:0 with 3 thread ranks
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sfgpu/sf.hpp"

using namespace sf;

static int failures = 0;
#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("CHECK failed: %s (line %d)\n", #c, __LINE__); \
      ++failures;                                                 \
    }                                                             \
  } while (0)

static std::vector<GraphSpec> fig2() {
  // "3 4 0:1.2 1:1.0 2:1.0 3:0.2 / 4 3 0:2.0 1:0.0 3:2.1 / 2 3 0:0.0 1:1.0 2:1.3"
  std::vector<GraphSpec> s(3);
  s[0] = {3, 4, std::vector<std::int64_t>{0, 1, 2, 3}, {{1, 2}, {1, 0}, {1, 0}, {0, 2}}};
  s[1] = {4, 3, std::vector<std::int64_t>{0, 1, 3}, {{2, 0}, {0, 0}, {2, 1}}};
  s[2] = {2, 3, std::vector<std::int64_t>{0, 1, 2}, {{0, 0}, {1, 0}, {1, 3}}};
  return s;
}

static void host_mode() {
  const auto specs = fig2();
  CommConfig cfg;
  cfg.nranks = 3;
  std::vector<std::vector<std::int64_t>> deg(3);
  std::vector<TwoSidedInfo> ti(3);
  std::vector<std::int64_t> multi(3);
  std::vector<std::int64_t> embedded(3), composed(3);
  run_ranks(cfg, [&](Comm& c) {
    StarForest f(c);
    f.set_graph(specs[static_cast<std::size_t>(c.rank())]);
    f.setup();
    ti[static_cast<std::size_t>(c.rank())] = f.two_sided();
    deg[static_cast<std::size_t>(c.rank())] = f.compute_degrees();
    multi[static_cast<std::size_t>(c.rank())] = f.multi_sf().nroots();
    // graph algebra (test_sfgraph.cpp:416-434, 266-284)
    std::vector<std::int64_t> sel;
    if (c.rank() == 1) sel.push_back(0);
    embedded[static_cast<std::size_t>(c.rank())] = embed_root(f, sel).nleaves();
    StarForest id = identity_sf(c, f.nroots());
    id.setup();
    composed[static_cast<std::size_t>(c.rank())] = compose(id, f).nleaves();
  }, {-1, -1, -1});
  CHECK((embedded == std::vector<std::int64_t>{2, 0, 1}));
  CHECK((composed == std::vector<std::int64_t>{4, 3, 3}));
  CHECK((deg[0] == std::vector<std::int64_t>{2, 0, 1}));
  CHECK((deg[1] == std::vector<std::int64_t>{3, 0, 1, 1}));
  CHECK((deg[2] == std::vector<std::int64_t>{1, 1}));
  CHECK(multi[0] == 3 && multi[1] == 5 && multi[2] == 2);
  CHECK(ti[0].self_first && ti[0].root_ranks.size() == 2 && ti[0].root_ranks[1].rank == 1);
  CHECK((ti[1].leaf_ranks[0].items == std::vector<std::int64_t>{2, 0, 0}));
  CHECK((ti[1].leaf_ranks[1].items == std::vector<std::int64_t>{0, 3}));
  // validation messages
  CommConfig one;
  run_ranks(one, [&](Comm& c) {
    StarForest f(c);
    bool threw = false;
    try {
      f.set_graph(1, 2, std::vector<std::int64_t>{0, 0}, {{0, 0}, {0, 0}});
    } catch (const Error& e) {
      threw = std::string(e.what()).find("forest property") != std::string::npos;
    }
    CHECK(threw);
  }, {-1});
}

template <class T>
static T* dev(const std::vector<T>& v) {
  T* p = nullptr;
  cudaMalloc(&p, sizeof(T) * (v.empty() ? 1 : v.size()));
  if (!v.empty()) cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
  return p;
}
template <class T>
static std::vector<T> host(const T* p, std::size_t n) {
  std::vector<T> v(n);
  if (n) cudaMemcpy(v.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost);
  return v;
}

static void gpu_mode() {
  const auto specs = fig2();
  const std::vector<std::vector<std::int64_t>> roots{{11, 12, 13}, {21, 22, 23, 24}, {31, 32}};
  const std::vector<std::vector<std::int64_t>> leaves{{110, 120, 130, 140}, {210, 220, 230, 240}, {310, 320, 330}};
  std::vector<std::vector<std::int64_t>> got_b(3), got_r(3), got_g(3);
  CommConfig cfg;
  cfg.nranks = 3;
  run_ranks(cfg, [&](Comm& c) {
    const auto r = static_cast<std::size_t>(c.rank());
    StarForest f(c);
    f.set_graph(specs[r]);
    f.setup();
    const Unit u = unit_of<std::int64_t>();
    auto* rd = dev(roots[r]);
    auto* ld = dev(leaves[r]);
    bcast(f, u, rd, ld, ReduceOp::replace);
    got_b[r] = host(ld, leaves[r].size());
    std::vector<std::int64_t> zero(roots[r].size(), 0);
    auto* zr = dev(zero);
    auto* l0 = dev(leaves[r]);
    reduce(f, u, l0, zr, ReduceOp::sum);
    got_r[r] = host(zr, roots[r].size());
    const auto d = f.compute_degrees();
    std::int64_t nm = 0;
    for (auto x : d) nm += x;
    std::vector<std::int64_t> m(static_cast<std::size_t>(nm), -1);
    auto* md = dev(m);
    gather(f, u, l0, md);
    got_g[r] = host(md, m.size());
    cudaFree(rd); cudaFree(ld); cudaFree(zr); cudaFree(l0); cudaFree(md);
  });
  CHECK((got_b[0] == std::vector<std::int64_t>{23, 21, 21, 13}));
  CHECK((got_b[1] == std::vector<std::int64_t>{31, 11, 230, 32}));
  CHECK((got_b[2] == std::vector<std::int64_t>{11, 21, 24}));
  CHECK((got_r[0] == std::vector<std::int64_t>{530, 0, 140}));
  CHECK((got_r[1] == std::vector<std::int64_t>{570, 0, 110, 330}));
  CHECK((got_g[1] == std::vector<std::int64_t>{120, 130, 320, 110, 330}));
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  try {
    if (mode == "host") host_mode();
    else gpu_mode();
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %d failures\n", mode.c_str(), failures);
  return failures ? 1 : 0;
}
