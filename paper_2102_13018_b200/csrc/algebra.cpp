// Graph algebra over star forests: compose, compose_inverse, embed_root,
// embed_leaf, identity (reference /root/reference/proj/src/starforest.cpp
// :270-465, declared in starforest.hpp:150-171). Setup-time host work, like
// the reference's; the difference is the algorithm. The reference gathers
// both edge lists on rank 0 and joins them there (compose_common); here every
// join is a distributed request/response over the control plane — a rank asks
// the owner of each vertex it needs and gets the answer back — so no rank
// ever holds more than its own edges.
#include <algorithm>
#include <array>
#include <cstring>

#include "sfg.hpp"

namespace sfg {
namespace {

using Bytes = std::vector<uint8_t>;

template <class T>
Bytes pack_vec(const std::vector<T>& v) {
  Bytes b(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
  return b;
}

template <class T>
std::vector<T> unpack_vec(const Bytes& b) {
  SFG_REQUIRE(b.size() % sizeof(T) == 0, "graph algebra: malformed exchange payload");
  std::vector<T> v(b.size() / sizeof(T));
  if (!v.empty()) std::memcpy(v.data(), b.data(), b.size());
  return v;
}

void same_comm(StarForest& a, StarForest& b, const char* what) {
  SFG_REQUIRE(&a.comm() == &b.comm(), std::string(what) + ": operands must live on the same communicator");
}

// Per rank: leaf index -> (root rank, root offset) of forest f, for indices
// in [0, bound); rank -1 where f has no leaf.
struct LeafMap {
  std::vector<int32_t> rank;
  std::vector<int64_t> off;
  explicit LeafMap(StarForest& f) {
    const int64_t bound = f.leaf_index_bound();
    rank.assign(static_cast<size_t>(bound), -1);
    off.assign(static_cast<size_t>(bound), -1);
    for (int64_t o = 0; o < f.nleaves(); ++o) {
      const int64_t idx = f.leaf_index(o);
      rank[static_cast<size_t>(idx)] = f.remote_rank_of(o);
      off[static_cast<size_t>(idx)] = f.remote_off_of(o);
    }
  }
  bool has(int64_t idx) const {
    return idx >= 0 && idx < static_cast<int64_t>(rank.size()) && rank[static_cast<size_t>(idx)] >= 0;
  }
};

std::unique_ptr<StarForest> build(Comm& c, int64_t nroots, std::vector<std::array<int64_t, 3>>& edges) {
  std::sort(edges.begin(), edges.end());  // ascending leaf index (compose_common's std::sort)
  std::vector<int64_t> local, off;
  std::vector<int32_t> rk;
  for (const auto& e : edges) {
    local.push_back(e[0]);
    rk.push_back(static_cast<int32_t>(e[1]));
    off.push_back(e[2]);
  }
  auto f = std::make_unique<StarForest>(&c);
  f->set_graph(nroots, static_cast<int64_t>(local.size()), local.empty() ? nullptr : local.data(), rk.data(),
               off.data());
  f->setup();
  return f;
}

}  // namespace

// starforest.hpp:150-154: roots of AB are A's roots, leaves are B's leaves; an
// edge where an A leaf and a B root coincide on (rank, index).
std::unique_ptr<StarForest> compose(StarForest& A, StarForest& B) {
  A.require_state(SfState::set_up, "compose");
  A.host_graph();
  B.require_state(SfState::set_up, "compose");
  B.host_graph();
  same_comm(A, B, "compose");
  Comm& c = A.comm();
  const int P = c.size();
  // 1. ask the owner of every B root (q, m) for A's root of its leaf m
  std::vector<std::vector<int64_t>> ask(static_cast<size_t>(P));
  std::vector<std::vector<int64_t>> who(static_cast<size_t>(P));  // B leaf ordinals per request
  for (int64_t o = 0; o < B.nleaves(); ++o) {
    const int q = B.remote_rank_of(o);
    ask[static_cast<size_t>(q)].push_back(B.remote_off_of(o));
    who[static_cast<size_t>(q)].push_back(o);
  }
  std::vector<Bytes> send(static_cast<size_t>(P));
  for (int q = 0; q < P; ++q) send[static_cast<size_t>(q)] = pack_vec(ask[static_cast<size_t>(q)]);
  auto req = c.ctrl().alltoallv(std::move(send));
  // 2. answer: (rank, offset) of my A leaf at each requested index, rank -1 if none
  const LeafMap am(A);
  std::vector<Bytes> ans(static_cast<size_t>(P));
  for (int p = 0; p < P; ++p) {
    const auto idx = unpack_vec<int64_t>(req[static_cast<size_t>(p)]);
    std::vector<int64_t> a(idx.size() * 2);
    for (size_t i = 0; i < idx.size(); ++i) {
      const bool h = am.has(idx[i]);
      a[2 * i] = h ? am.rank[static_cast<size_t>(idx[i])] : -1;
      a[2 * i + 1] = h ? am.off[static_cast<size_t>(idx[i])] : -1;
    }
    ans[static_cast<size_t>(p)] = pack_vec(a);
  }
  auto got = c.ctrl().alltoallv(std::move(ans));
  // 3. AB edges: B leaf -> A root, where the join hit
  std::vector<std::array<int64_t, 3>> edges;
  for (int q = 0; q < P; ++q) {
    const auto a = unpack_vec<int64_t>(got[static_cast<size_t>(q)]);
    const auto& w = who[static_cast<size_t>(q)];
    SFG_REQUIRE(a.size() == 2 * w.size(), "compose: malformed reply");
    for (size_t i = 0; i < w.size(); ++i)
      if (a[2 * i] >= 0) edges.push_back({B.leaf_index(w[i]), a[2 * i], a[2 * i + 1]});
  }
  return build(c, A.nroots(), edges);
}

// starforest.hpp:156-159: roots of AB are A's roots, leaves are B's roots.
std::unique_ptr<StarForest> compose_inverse(StarForest& A, StarForest& B) {
  A.require_state(SfState::set_up, "compose_inverse");
  A.host_graph();
  B.require_state(SfState::set_up, "compose_inverse");
  B.host_graph();
  same_comm(A, B, "compose_inverse");
  Comm& c = A.comm();
  const int P = c.size();
  // Preconditions, agreed globally so every rank fails together:
  // every B root has degree <= 1; every A leaf is also a B leaf (same rank).
  int64_t verdict[2] = {0, 0};
  for (int64_t d : B.compute_degrees()) verdict[0] = std::max(verdict[0], d);
  const LeafMap bm(B);
  for (int64_t o = 0; o < A.nleaves(); ++o)
    if (!bm.has(A.leaf_index(o))) verdict[1] = 1;
  std::vector<int64_t> all(2 * static_cast<size_t>(P));
  c.ctrl().allgather(verdict, sizeof(verdict), all.data());
  int64_t maxdeg = 0, uncovered = 0;
  for (int r = 0; r < P; ++r) {
    maxdeg = std::max(maxdeg, all[2 * static_cast<size_t>(r)]);
    uncovered |= all[2 * static_cast<size_t>(r) + 1];
  }
  SFG_REQUIRE(maxdeg <= 1, "compose_inverse: a B root has degree > 1");
  SFG_REQUIRE(uncovered == 0, "compose_inverse: A's leaves are not completely overlapped by B's leaves");
  // Each B leaf b with root (r, off) that is also an A leaf sends
  // (off, A's root of b) to r: on r the B root `off` becomes an AB leaf.
  const LeafMap am(A);
  std::vector<std::vector<int64_t>> out(static_cast<size_t>(P));
  for (int64_t o = 0; o < B.nleaves(); ++o) {
    const int64_t b = B.leaf_index(o);
    if (!am.has(b)) continue;
    auto& v = out[static_cast<size_t>(B.remote_rank_of(o))];
    v.push_back(B.remote_off_of(o));
    v.push_back(am.rank[static_cast<size_t>(b)]);
    v.push_back(am.off[static_cast<size_t>(b)]);
  }
  std::vector<Bytes> send(static_cast<size_t>(P));
  for (int r = 0; r < P; ++r) send[static_cast<size_t>(r)] = pack_vec(out[static_cast<size_t>(r)]);
  auto got = c.ctrl().alltoallv(std::move(send));
  std::vector<std::array<int64_t, 3>> edges;
  for (int s = 0; s < P; ++s) {
    const auto v = unpack_vec<int64_t>(got[static_cast<size_t>(s)]);
    for (size_t i = 0; i + 2 < v.size(); i += 3) edges.push_back({v[i], v[i + 1], v[i + 2]});
  }
  return build(c, A.nroots(), edges);
}

// starforest.hpp:161-167: keep the edges whose root is selected.
std::unique_ptr<StarForest> embed_root(StarForest& f, const int64_t* sel, int64_t nsel) {
  f.require_state(SfState::set_up, "embed_root");
  f.host_graph();
  Comm& c = f.comm();
  const int P = c.size();
  std::vector<uint8_t> flag(static_cast<size_t>(f.nroots()), 0);
  for (int64_t i = 0; i < nsel; ++i) {
    SFG_REQUIRE(sel[i] >= 0 && sel[i] < f.nroots(), "embed_root: selected root out of range");
    flag[static_cast<size_t>(sel[i])] = 1;  // duplicates collapse silently
  }
  // every leaf learns its root's verdict from the root's owner
  std::vector<std::vector<int64_t>> ask(static_cast<size_t>(P));
  std::vector<std::vector<int64_t>> who(static_cast<size_t>(P));
  for (int64_t o = 0; o < f.nleaves(); ++o) {
    ask[static_cast<size_t>(f.remote_rank_of(o))].push_back(f.remote_off_of(o));
    who[static_cast<size_t>(f.remote_rank_of(o))].push_back(o);
  }
  std::vector<Bytes> send(static_cast<size_t>(P));
  for (int q = 0; q < P; ++q) send[static_cast<size_t>(q)] = pack_vec(ask[static_cast<size_t>(q)]);
  auto req = c.ctrl().alltoallv(std::move(send));
  std::vector<Bytes> ans(static_cast<size_t>(P));
  for (int p = 0; p < P; ++p) {
    const auto idx = unpack_vec<int64_t>(req[static_cast<size_t>(p)]);
    Bytes a(idx.size());
    for (size_t i = 0; i < idx.size(); ++i) a[i] = flag[static_cast<size_t>(idx[i])];
    ans[static_cast<size_t>(p)] = std::move(a);
  }
  auto got = c.ctrl().alltoallv(std::move(ans));
  std::vector<std::array<int64_t, 3>> edges;
  for (int q = 0; q < P; ++q) {
    const auto& w = who[static_cast<size_t>(q)];
    const auto& a = got[static_cast<size_t>(q)];
    SFG_REQUIRE(a.size() == w.size(), "embed_root: malformed reply");
    for (size_t i = 0; i < w.size(); ++i)
      if (a[i]) edges.push_back({f.leaf_index(w[i]), f.remote_rank_of(w[i]), f.remote_off_of(w[i])});
  }
  return build(c, f.nroots(), edges);
}

// starforest.hpp:161-167: keep the edges whose leaf index is selected.
std::unique_ptr<StarForest> embed_leaf(StarForest& f, const int64_t* sel, int64_t nsel) {
  f.require_state(SfState::set_up, "embed_leaf");
  f.host_graph();
  std::vector<int64_t> s(sel, sel + nsel);
  for (int64_t l : s) SFG_REQUIRE(l >= 0, "embed_leaf: selected leaf index is negative");
  std::sort(s.begin(), s.end());
  s.erase(std::unique(s.begin(), s.end()), s.end());
  std::vector<std::array<int64_t, 3>> edges;
  for (int64_t o = 0; o < f.nleaves(); ++o) {
    const int64_t idx = f.leaf_index(o);
    if (std::binary_search(s.begin(), s.end(), idx))
      edges.push_back({idx, f.remote_rank_of(o), f.remote_off_of(o)});
  }
  return build(f.comm(), f.nroots(), edges);
}

// starforest.hpp:169-171: leaf i -> root i on the same rank (graph set, not set up).
std::unique_ptr<StarForest> identity_sf(Comm& c, int64_t n) {
  SFG_REQUIRE(n >= 0, "identity_sf: negative size");
  std::vector<int32_t> rk(static_cast<size_t>(n), c.rank());
  std::vector<int64_t> off(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) off[static_cast<size_t>(i)] = i;
  auto f = std::make_unique<StarForest>(&c);
  f->set_graph(n, n, nullptr, rk.data(), off.data());
  return f;
}

}  // namespace sfg
