// sfgpu/sf.hpp — header-only C++ façade over the C ABI (include/sfgpu.h)
// with the reference's `sf::` API surface, so a user of
// /root/reference/proj/include/sf/{unit,errors,starforest,ops,harness}.hpp can
// switch by changing the include path and linking _sfgpu.so.
//
// Differences a caller must know:
//  * data buffers are CUDA device pointers on the rank's GPU;
//  * *_end() is stream-ordered; the one-shot forms (sf::bcast, ...) and
//    wait() synchronise the stream, like the reference's End;
//  * Comm is created per rank: thread ranks share an sf::World
//    (sf::run_ranks below mirrors harness.hpp:58-72), process ranks pass an
//    NCCL unique id.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../sfgpu.h"

namespace sf {

// ------------------------------------------------------------ vocabulary
enum class Kind : std::uint8_t { int32 = SFG_INT32, int64 = SFG_INT64, float64 = SFG_FLOAT64, bytes = SFG_BYTES };
enum class ReduceOp : std::uint8_t { replace = 0, sum, prod, max, min, land, lor, band, bor };
enum class SfState { created = 0, graph_set = 1, set_up = 2 };
enum class SetupAlg { automatic = 0, dense = 1, consensus = 2 };
enum class OpKind : std::uint8_t { bcast = 0, reduce, fetch_and_op, gather, scatter };

struct Unit {
  Kind kind = Kind::int64;
  std::int64_t blocklen = 1;
  std::size_t elem_size() const { return kind == Kind::int32 ? 4 : kind == Kind::bytes ? 1 : 8; }
  std::size_t bytes() const { return elem_size() * static_cast<std::size_t>(blocklen); }
};
template <class T> constexpr Kind kind_of();
template <> constexpr Kind kind_of<std::int32_t>() { return Kind::int32; }
template <> constexpr Kind kind_of<std::int64_t>() { return Kind::int64; }
template <> constexpr Kind kind_of<double>() { return Kind::float64; }
template <class T> constexpr Unit unit_of(std::int64_t blocklen = 1) { return Unit{kind_of<T>(), blocklen}; }

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class TimeoutError : public Error {
 public:
  using Error::Error;
};

namespace detail {
inline void check(int rc) {
  if (rc == SFG_OK) return;
  const std::string msg = sfg_last_error();
  if (rc == SFG_ERR_TIMEOUT) throw TimeoutError(msg);
  throw Error(msg);
}
// The one-shot forms block like the reference's (ops.cpp: Begin + End).
inline void sync(cudaStream_t s) {
  if (cudaStreamSynchronize(s) != cudaSuccess) throw Error("stream synchronisation failed");
}
}  // namespace detail

struct RootRef {
  int rank = -1;
  std::int64_t offset = -1;
  bool operator==(const RootRef&) const = default;
};

struct GraphSpec {
  std::int64_t nroots = 0;
  std::int64_t nleaves = 0;
  std::optional<std::vector<std::int64_t>> local;
  std::vector<RootRef> remote;
};

struct TwoSidedInfo {
  struct Group {
    int rank = -1;
    std::vector<std::int64_t> items;
  };
  std::vector<Group> root_ranks;
  std::vector<Group> leaf_ranks;
  bool self_first = false;
};

struct CommConfig {
  int nranks = 1;
  std::string backend = "threads";  // threads | nccl | p2p
  bool deterministic = true;
  bool debug_checksum = false;
  bool force_remote = false;
  int dense_discovery_threshold = 64;
  std::uint64_t seed = 1;
  double timeout_s = 30.0;
  sfg_config c() const {
    sfg_config x;
    sfg_config_default(&x);
    x.deterministic = deterministic;
    x.debug_checksum = debug_checksum;
    x.force_remote = force_remote;
    x.dense_discovery_threshold = dense_discovery_threshold;
    x.seed = seed;
    x.timeout_s = timeout_s;
    return x;
  }
};

// ------------------------------------------------------------ world / comm
class World {
 public:
  World(int nranks, double timeout_s) { detail::check(sfg_world_create(nranks, timeout_s, &w_)); }
  ~World() { sfg_world_destroy(w_); }
  World(const World&) = delete;
  World& operator=(const World&) = delete;
  void abort() { sfg_world_abort(w_); }
  sfg_world handle() const { return w_; }

 private:
  sfg_world w_ = nullptr;
};

class Comm {
 public:
  // Thread rank of an in-process world (device < 0: host-only).
  Comm(World& world, const CommConfig& cfg, int rank, int device, const void* nccl_id = nullptr) {
    const sfg_config c = cfg.c();
    detail::check(sfg_comm_create(world.handle(), cfg.nranks, rank, device, cfg.backend.c_str(),
                                  nccl_id, &c, &h_));
    rank_ = rank;
    size_ = cfg.nranks;
  }
  // One rank per process over NCCL (nccl_id shared by the caller).
  Comm(const CommConfig& cfg, int rank, int device, const void* nccl_id) {
    const sfg_config c = cfg.c();
    detail::check(sfg_comm_create(nullptr, cfg.nranks, rank, device, "nccl", nccl_id, &c, &h_));
    rank_ = rank;
    size_ = cfg.nranks;
  }
  ~Comm() {
    if (h_) sfg_comm_destroy(h_);
  }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  int rank() const { return rank_; }
  int size() const { return size_; }
  sfg_comm handle() const { return h_; }

 private:
  sfg_comm h_ = nullptr;
  int rank_ = 0, size_ = 1;
};

// ------------------------------------------------------------ star forest
class StarForest {
 public:
  explicit StarForest(Comm& comm) { detail::check(sfg_sf_create(comm.handle(), &h_)); }
  ~StarForest() {
    if (owned_ && h_) sfg_sf_destroy(h_);
  }
  StarForest(StarForest&& o) noexcept : h_(o.h_), owned_(o.owned_) { o.h_ = nullptr; }
  StarForest(const StarForest&) = delete;

  void set_graph(std::int64_t nroots, std::int64_t nleaves,
                 std::optional<std::vector<std::int64_t>> leaf_local, std::vector<RootRef> leaf_remote) {
    if (leaf_local && static_cast<std::int64_t>(leaf_local->size()) != nleaves)
      throw Error("set_graph: leaf_local length does not match nleaves");
    if (static_cast<std::int64_t>(leaf_remote.size()) != nleaves)
      throw Error("set_graph: leaf_remote length does not match nleaves");
    std::vector<std::int32_t> rr(leaf_remote.size());
    std::vector<std::int64_t> ro(leaf_remote.size());
    for (std::size_t i = 0; i < leaf_remote.size(); ++i) {
      rr[i] = leaf_remote[i].rank;
      ro[i] = leaf_remote[i].offset;
    }
    static const std::int64_t none = 0;
    detail::check(sfg_sf_set_graph(h_, nroots, nleaves,
                                   leaf_local ? (leaf_local->empty() ? &none : leaf_local->data()) : nullptr,
                                   rr.data(), ro.data()));
  }
  void set_graph(const GraphSpec& s) { set_graph(s.nroots, s.nleaves, s.local, s.remote); }
  // The graph already in the communicator's device memory:
  // leaf_local may be nullptr; setup() then plans on the GPU.
  void set_graph_device(std::int64_t nroots, std::int64_t nleaves, const std::int64_t* leaf_local,
                        const std::int32_t* remote_rank, const std::int64_t* remote_off) {
    detail::check(sfg_sf_set_graph_device(h_, nroots, nleaves, leaf_local, remote_rank, remote_off));
  }
  void setup(SetupAlg alg = SetupAlg::automatic) { detail::check(sfg_sf_setup(h_, static_cast<int>(alg))); }
  // Device plans and a staging slot for `unit` before a CUDA-graph capture
  // (SetUp already did this for 8-byte units). Collective on p2p.
  void prepare(const Unit& unit) {
    detail::check(sfg_sf_prepare(h_, static_cast<int>(unit.kind), unit.blocklen));
  }

  SfState state() const { return static_cast<SfState>(info().state); }
  std::int64_t nroots() const { return info().nroots; }
  std::int64_t nleaves() const { return info().nleaves; }
  std::int64_t leaf_index_bound() const { return info().leaf_index_bound; }
  bool contiguous_leaves() const { return info().contiguous_leaves != 0; }
  bool has_self_edges() const { return info().self_first != 0; }

  TwoSidedInfo two_sided() const {
    const sfg_sf_info i = info();
    if (i.state != 2) detail::check(sfg_sf_group(h_, 0, 0, nullptr, nullptr, nullptr));
    TwoSidedInfo t;
    t.self_first = i.self_first != 0;
    for (int which = 0; which < 2; ++which) {
      const int n = which == 0 ? i.n_root_groups : i.n_leaf_groups;
      for (int g = 0; g < n; ++g) {
        TwoSidedInfo::Group grp;
        std::int64_t cnt = 0;
        detail::check(sfg_sf_group(h_, which, g, &grp.rank, &cnt, nullptr));
        grp.items.resize(static_cast<std::size_t>(cnt));
        detail::check(sfg_sf_group_items(h_, which, g, grp.items.data()));
        (which == 0 ? t.root_ranks : t.leaf_ranks).push_back(std::move(grp));
      }
    }
    return t;
  }

  std::vector<std::int64_t> compute_degrees() const {
    std::vector<std::int64_t> d(static_cast<std::size_t>(nroots()));
    detail::check(sfg_sf_compute_degrees(h_, d.data()));
    return d;
  }

  StarForest& multi_sf() {
    if (!multi_) {
      sfg_sf m = nullptr;
      detail::check(sfg_sf_multi_sf(h_, &m));
      multi_.reset(new StarForest(m));
    }
    return *multi_;
  }

  sfg_sf handle() const { return h_; }
  // Takes ownership of a forest the library created (graph algebra).
  static StarForest adopt(sfg_sf owned) {
    StarForest f(owned);
    f.owned_ = true;
    return f;
  }

 private:
  explicit StarForest(sfg_sf borrowed) : h_(borrowed), owned_(false) {}
  sfg_sf_info info() const {
    sfg_sf_info i;
    detail::check(sfg_sf_get_info(h_, &i));
    return i;
  }
  sfg_sf h_ = nullptr;
  bool owned_ = true;
  std::unique_ptr<StarForest> multi_;
};

// --------------------------------------------------------- graph algebra
// starforest.hpp:150-171
inline StarForest compose(StarForest& a, StarForest& b) {
  sfg_sf h = nullptr;
  detail::check(sfg_sf_compose(a.handle(), b.handle(), 0, &h));
  return StarForest::adopt(h);
}
inline StarForest compose_inverse(StarForest& a, StarForest& b) {
  sfg_sf h = nullptr;
  detail::check(sfg_sf_compose(a.handle(), b.handle(), 1, &h));
  return StarForest::adopt(h);
}
inline StarForest embed_root(StarForest& f, const std::vector<std::int64_t>& selected) {
  sfg_sf h = nullptr;
  detail::check(sfg_sf_embed(f.handle(), 0, selected.data(), static_cast<std::int64_t>(selected.size()), &h));
  return StarForest::adopt(h);
}
inline StarForest embed_leaf(StarForest& f, const std::vector<std::int64_t>& selected) {
  sfg_sf h = nullptr;
  detail::check(sfg_sf_embed(f.handle(), 1, selected.data(), static_cast<std::int64_t>(selected.size()), &h));
  return StarForest::adopt(h);
}
inline StarForest identity_sf(Comm& c, std::int64_t n) {
  sfg_sf h = nullptr;
  detail::check(sfg_sf_identity(c.handle(), n, &h));
  return StarForest::adopt(h);
}

// ------------------------------------------------------------ operations
class OpHandle {
 public:
  OpHandle() = default;
  OpHandle(sfg_handle h, cudaStream_t s) : h_(h), s_(s) {}
  OpHandle(OpHandle&& o) noexcept : h_(o.h_), s_(o.s_) { o.h_ = nullptr; }
  OpHandle& operator=(OpHandle&& o) noexcept {
    std::swap(h_, o.h_);
    std::swap(s_, o.s_);
    return *this;
  }
  ~OpHandle() {
    if (h_) sfg_handle_free(h_);
  }
  OpKind kind() const { return static_cast<OpKind>(q(0)); }
  ReduceOp op() const { return static_cast<ReduceOp>(q(1)); }
  bool ended() const { return q(2) != 0; }
  sfg_handle handle() const { return h_; }
  // Block until everything enqueued for this operation has completed.
  void wait() const {
    if (cudaStreamSynchronize(s_) != cudaSuccess) throw Error("stream synchronisation failed");
  }

 private:
  int q(int which) const {
    int k = 0, o = 0, e = 0;
    detail::check(sfg_handle_info(h_, &k, &o, &e));
    return which == 0 ? k : which == 1 ? o : e;
  }
  sfg_handle h_ = nullptr;
  cudaStream_t s_ = nullptr;
};

inline OpHandle bcast_begin(StarForest& sf, const Unit& u, const void* rootdata, void* leafdata,
                            ReduceOp op, cudaStream_t s = nullptr) {
  sfg_handle h = nullptr;
  detail::check(sfg_bcast_begin(sf.handle(), static_cast<int>(u.kind), u.blocklen, rootdata,
                                leafdata, static_cast<int>(op), s, &h));
  return OpHandle(h, s);
}
inline void bcast_end(OpHandle& h) { detail::check(sfg_bcast_end(h.handle())); }
inline void bcast(StarForest& sf, const Unit& u, const void* rootdata, void* leafdata, ReduceOp op,
                  cudaStream_t s = nullptr) {
  detail::check(sfg_bcast(sf.handle(), static_cast<int>(u.kind), u.blocklen, rootdata, leafdata,
                          static_cast<int>(op), s));
  detail::sync(s);
}

inline OpHandle reduce_begin(StarForest& sf, const Unit& u, const void* leafdata, void* rootdata,
                             ReduceOp op, cudaStream_t s = nullptr) {
  sfg_handle h = nullptr;
  detail::check(sfg_reduce_begin(sf.handle(), static_cast<int>(u.kind), u.blocklen, leafdata,
                                 rootdata, static_cast<int>(op), s, &h));
  return OpHandle(h, s);
}
inline void reduce_end(OpHandle& h) { detail::check(sfg_reduce_end(h.handle())); }
inline void reduce(StarForest& sf, const Unit& u, const void* leafdata, void* rootdata, ReduceOp op,
                   cudaStream_t s = nullptr) {
  detail::check(sfg_reduce(sf.handle(), static_cast<int>(u.kind), u.blocklen, leafdata, rootdata,
                           static_cast<int>(op), s));
  detail::sync(s);
}

inline OpHandle fetch_and_op_begin(StarForest& sf, const Unit& u, void* rootdata,
                                   const void* leafdata, void* leafupdate, ReduceOp op,
                                   cudaStream_t s = nullptr) {
  sfg_handle h = nullptr;
  detail::check(sfg_fetch_and_op_begin(sf.handle(), static_cast<int>(u.kind), u.blocklen, rootdata,
                                       leafdata, leafupdate, static_cast<int>(op), s, &h));
  return OpHandle(h, s);
}
inline void fetch_and_op_end(OpHandle& h) { detail::check(sfg_fetch_and_op_end(h.handle())); }
inline void fetch_and_op(StarForest& sf, const Unit& u, void* rootdata, const void* leafdata,
                         void* leafupdate, ReduceOp op, cudaStream_t s = nullptr) {
  detail::check(sfg_fetch_and_op(sf.handle(), static_cast<int>(u.kind), u.blocklen, rootdata, leafdata,
                                 leafupdate, static_cast<int>(op), s));
  detail::sync(s);
}

inline OpHandle gather_begin(StarForest& sf, const Unit& u, const void* leafdata,
                             void* multirootdata, cudaStream_t s = nullptr) {
  sfg_handle h = nullptr;
  detail::check(sfg_gather_begin(sf.handle(), static_cast<int>(u.kind), u.blocklen, leafdata,
                                 multirootdata, s, &h));
  return OpHandle(h, s);
}
inline void gather_end(OpHandle& h) { detail::check(sfg_gather_end(h.handle())); }
inline void gather(StarForest& sf, const Unit& u, const void* leafdata, void* multirootdata,
                   cudaStream_t s = nullptr) {
  detail::check(sfg_gather(sf.handle(), static_cast<int>(u.kind), u.blocklen, leafdata, multirootdata, s));
  detail::sync(s);
}

inline OpHandle scatter_begin(StarForest& sf, const Unit& u, const void* multirootdata,
                              void* leafdata, cudaStream_t s = nullptr) {
  sfg_handle h = nullptr;
  detail::check(sfg_scatter_begin(sf.handle(), static_cast<int>(u.kind), u.blocklen,
                                  multirootdata, leafdata, s, &h));
  return OpHandle(h, s);
}
inline void scatter_end(OpHandle& h) { detail::check(sfg_scatter_end(h.handle())); }
inline void scatter(StarForest& sf, const Unit& u, const void* multirootdata, void* leafdata,
                    cudaStream_t s = nullptr) {
  detail::check(sfg_scatter(sf.handle(), static_cast<int>(u.kind), u.blocklen, multirootdata, leafdata, s));
  detail::sync(s);
}

// ------------------------------------------------------------ harness
// run_ranks (harness.hpp:58-72): one thread per rank; devices[r] is the CUDA
// device of rank r (-1: host-only). A failing rank aborts the others; the
// first failure is rethrown after every rank has joined.
inline void run_ranks(const CommConfig& cfg, const std::function<void(Comm&)>& body,
                      std::vector<int> devices = {}) {
  if (devices.empty()) devices.assign(static_cast<std::size_t>(cfg.nranks), 0);
  World world(cfg.nranks, cfg.timeout_s);
  std::vector<std::exception_ptr> errors(static_cast<std::size_t>(cfg.nranks));
  std::vector<unsigned char> id(128, 0);
  if (cfg.backend == "nccl") detail::check(sfg_nccl_unique_id(id.data(), id.size()));
  std::vector<std::thread> ts;
  for (int r = 0; r < cfg.nranks; ++r) {
    ts.emplace_back([&, r] {
      try {
        if (devices[static_cast<std::size_t>(r)] >= 0) cudaSetDevice(devices[static_cast<std::size_t>(r)]);
        Comm c(world, cfg, r, devices[static_cast<std::size_t>(r)],
               cfg.backend == "nccl" ? id.data() : nullptr);
        body(c);
      } catch (...) {
        errors[static_cast<std::size_t>(r)] = std::current_exception();
        world.abort();
      }
    });
  }
  for (auto& t : ts) t.join();
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
}

}  // namespace sf
