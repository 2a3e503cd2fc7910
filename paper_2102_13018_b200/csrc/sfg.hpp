// Internal C++ core of the B200 star-forest layer.
//
// Mirrors the reference's layering (/root/reference/proj/include/sf/*.hpp):
//   vocabulary (Unit/Kind/ReduceOp/Error)   <- unit.hpp, errors.hpp
//   Comm = control plane + data-plane transport   <- comm.hpp, exchange.hpp
//   StarForest (set_graph/setup/degrees/multi_sf) <- starforest.hpp
//   split-phase operations                        <- ops.hpp
// but the data plane is device-resident: per-peer plans live in HBM, packs
// and unpacks are sm_100a kernels (kernels.cu), remote exchange is one-sided
// NVLink puts with in-kernel flags (p2p.cpp), grouped NCCL send/recv, or
// stream-ordered peer copies for in-process ranks, and nothing synchronises
// the host between Begin and End.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.hpp"

namespace sfg {

// Host arrays of SetUp size (10^8 edges) are filled right after allocation
// by parallel loops: an allocator that default-initialises (no zero pass)
// lets the filling threads take the first-touch page faults in parallel.
template <class T>
struct DefaultInit : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInit<U>;
  };
  DefaultInit() = default;
  template <class U>
  DefaultInit(const DefaultInit<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using HostVec = std::vector<T, DefaultInit<T>>;

// ---------------------------------------------------------------- vocabulary
// /root/reference/proj/include/sf/unit.hpp:14-82
enum class Kind : uint8_t { int32 = 0, int64 = 1, float64 = 2, bytes = 3 };
enum class ReduceOp : uint8_t { replace = 0, sum, prod, max, min, land, lor, band, bor };

const char* kind_name(Kind k);
const char* op_name(ReduceOp op);

struct Unit {
  Kind kind = Kind::int64;
  int64_t blocklen = 1;
  size_t elem_size() const;
  size_t bytes() const { return elem_size() * static_cast<size_t>(blocklen); }
};

// /root/reference/proj/include/sf/errors.hpp:11-32
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class TimeoutError : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

[[noreturn]] void fail(const std::string& msg);
#define SFG_REQUIRE(cond, msg)   \
  do {                           \
    if (!(cond)) ::sfg::fail(msg); \
  } while (0)
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void nccl_check(ncclResult_t r, const char* what, const char* file, int line);
#define SFG_CUDA(x) ::sfg::cuda_check((x), #x, __FILE__, __LINE__)
#define SFG_NCCL(x) ::sfg::nccl_check((x), #x, __FILE__, __LINE__)

void check_unit_op(const Unit& u, ReduceOp op);

// ------------------------------------------------------------------- config
// /root/reference/proj/include/sf/comm.hpp:54-66
struct CommConfig {
  std::string backend = "threads";  // threads (in-process ranks) | nccl | p2p
  bool deterministic = true;        // reference fold order, bit-exact
  bool debug_checksum = false;      // verify source buffers between begin/end
  bool force_remote = false;        // route self edges through the transport
  int dense_discovery_threshold = 64;
  uint64_t seed = 1;
  double timeout_s = 30.0;
};

// Copy instrumentation, the analogue of PackCounters
// (/root/reference/proj/include/sf/pack.hpp:20-32).
struct Counters {
  std::atomic<uint64_t> pack_copies{0};      // remote groups packed into staging
  std::atomic<uint64_t> pack_elided{0};      // zero-copy sends (contiguous)
  std::atomic<uint64_t> unpack_copies{0};    // remote groups unpacked from staging
  std::atomic<uint64_t> unpack_elided{0};    // zero-copy receives
  std::atomic<uint64_t> replace_dup_collisions{0};
  std::atomic<uint64_t> kernel_launches{0};
  std::atomic<uint64_t> bytes_sent{0};
  std::atomic<uint64_t> bytes_recv{0};
  std::atomic<uint64_t> transport_calls{0};
  void reset();
};
Counters& counters();

// Per-launch device timing (CUDA events recorded on the launching stream
// around each kernel) and algorithmic bytes, for the bench's roofline.
struct TimingRec {
  std::string tag;
  uint64_t launches = 0;
  double total_ms = 0.0;
  double bytes = 0.0;
  double link_bytes = 0.0;  // stored into peer GPUs (p2p puts)
};
void timing_enable(bool on);
bool timing_enabled();
void timing_record(const char* tag, cudaEvent_t a, cudaEvent_t b, double bytes,
                   double link_bytes = 0.0);
std::vector<TimingRec> timing_collect();  // synchronises the events
cudaEvent_t timing_event();

// --------------------------------------------------------------- pattern
// Classification of an index list (/root/reference/proj/include/sf/pattern.hpp:28-102).
// Unlike the reference (which only recognises strided subdomains when handed
// GridExtents, pattern.cpp:50-64), the planner infers Affine3D blocks from the
// indices themselves and verifies them, as PetscSF does.
struct Pattern {
  enum Kind : uint8_t { contiguous = 0, affine = 1, indexed = 2 };
  Kind kind = contiguous;
  int64_t count = 0;
  int64_t start = 0;
  int64_t dx = 0, dy = 0, dz = 0, s1 = 0, s2 = 0;  // affine
  HostVec<int64_t> idx;                             // indexed
  const int64_t* didx = nullptr;  // indexed, device SetUp: the list in HBM (DevGraph-owned)
  bool has_duplicates = false;
  int64_t distinct = 0;  // number of distinct indices
  int64_t bound = 0;  // largest index + 1 (0 when empty)

  // extents_x / extents_xy > 0: reference-style detection with known extents.
  static Pattern analyze(const int64_t* idx, int64_t n, bool infer_affine = true,
                         int64_t extents_x = 0, int64_t extents_xy = 0);
  static Pattern contiguous_range(int64_t start, int64_t n);
  int64_t index(int64_t i) const;
  bool is_contiguous() const { return kind == contiguous; }
};

// -------------------------------------------------------- control plane
// Host-side collectives used only by SetUp / multi-SF construction
// (the reference's allreduce + sparse exchange, comm.cpp:196-214,
// exchange.cpp:32-102).
class ControlPlane {
 public:
  virtual ~ControlPlane() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // out receives size()*bytes: rank r's contribution at r*bytes.
  virtual void allgather(const void* in, size_t bytes, void* out) = 0;
  // send[r] goes to rank r; returns what each rank sent to me.
  virtual std::vector<std::vector<uint8_t>> alltoallv(std::vector<std::vector<uint8_t>> send) = 0;
  // Same exchange between DEVICE buffers of the calling rank's GPU (the
  // device SetUp's discovery payload): send + soff[r] holds sbytes[r] for
  // rank r, rank r's payload lands at recv + roff[r] (rbytes[r], agreed
  // beforehand). Entries for the own rank are ignored. Synchronous. Returns
  // false when this control plane cannot move device memory (the caller then
  // stages through the host).
  virtual bool alltoallv_device(const uint8_t* send, const std::vector<int64_t>& soff,
                                const std::vector<int64_t>& sbytes, uint8_t* recv,
                                const std::vector<int64_t>& roff, const std::vector<int64_t>& rbytes) {
    return false;
  }
  virtual void barrier() = 0;
};

// One posted buffer of the in-process transport's put protocol.
struct Post {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaEvent_t ev = nullptr;
  int device = -1;
};

// In-process world: ranks are threads of one process (the reference's
// harness model, /root/reference/proj/src/harness.cpp:51-101). Hosts the
// threads control plane and the rendezvous table of the threads transport.
class World {
 public:
  World(int n, double timeout_s);
  int size() const { return n_; }
  double timeout_s() const { return timeout_s_; }
  void abort() { aborted_.store(true); cv_.notify_all(); }
  bool aborted() const { return aborted_.load(); }

  void barrier(const char* what);
  void put_slot(int rank, std::vector<uint8_t> data);
  const std::vector<uint8_t>& slot(int rank) const { return slots_[rank]; }
  void put_mail(int src, int dst, std::vector<uint8_t> data);
  std::vector<uint8_t> take_mail(int src, int dst);

  // key: (tag, src, dst, kind)
  struct Key {
    uint64_t tag;
    int src, dst, kind;
    bool operator<(const Key& o) const {
      if (tag != o.tag) return tag < o.tag;
      if (src != o.src) return src < o.src;
      if (dst != o.dst) return dst < o.dst;
      return kind < o.kind;
    }
  };
  void post(const Key& k, const Post& p);
  Post take(const Key& k, const char* what);

 private:
  int n_;
  double timeout_s_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<bool> aborted_{false};
  int arrived_ = 0;
  uint64_t generation_ = 0;
  std::vector<std::vector<uint8_t>> slots_;
  std::vector<std::vector<std::vector<uint8_t>>> mail_;
  std::map<Key, Post> posts_;
};

struct XferOp {
  int peer = -1;
  void* ptr = nullptr;
  size_t bytes = 0;
};

// Data-plane transport. start() enqueues one exchange phase on `stream`
// (sends of data produced earlier on `stream`); finish() makes `stream`
// wait until the receives of that phase have landed. Neither blocks the host
// on the GPU.
class Transport {
 public:
  virtual ~Transport() = default;
  virtual void start(uint64_t tag, const std::vector<XferOp>& sends,
                     const std::vector<XferOp>& recvs, cudaStream_t stream) = 0;
  virtual void finish(uint64_t tag, const std::vector<XferOp>& recvs, cudaStream_t stream) = 0;
  virtual const char* name() const = 0;
};

class Comm {
 public:
  Comm(int nranks, int rank, int device, CommConfig cfg);
  ~Comm();
  int rank() const { return rank_; }
  int size() const { return size_; }
  int device() const { return device_; }
  bool has_device() const { return device_ >= 0; }
  const CommConfig& config() const { return cfg_; }
  CommConfig& config_mut() { return cfg_; }
  ControlPlane& ctrl() { return *ctrl_; }
  Transport& transport();
  // Operation ids 0, 1, 2, ... per communicator, as the reference's
  // Comm::next_op_seq (comm.cpp:184-186: fetch_add from 0); they seed the
  // free-order fetch shuffle, so the same sequence of calls serializes
  // exactly as the reference does.
  uint64_t next_op_seq() { return op_seq_++; }
  void bind_device() const;
  // One-sided put/signal data plane over NVLink peer mappings (backend "p2p").
  bool p2p() const { return cfg_.backend == "p2p"; }

  // Every transport call of this communicator runs on one internal stream
  // (NCCL requires a single issue order per communicator); fork/join order it
  // against the caller's stream so exchanges overlap the local scatter.
  cudaStream_t comm_stream();
  void fork(cudaStream_t user);  // comm stream waits for work queued on `user`
  void join(cudaStream_t user);  // `user` waits for work queued on the comm stream

  // wiring (abi.cpp)
  std::unique_ptr<ControlPlane> ctrl_;
  std::unique_ptr<Transport> transport_;
  ncclComm_t nccl_ = nullptr;
  World* world_ = nullptr;

 private:
  int size_, rank_, device_;
  CommConfig cfg_;
  uint64_t op_seq_ = 0;
  cudaStream_t cstream_ = nullptr;
  cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
};

std::unique_ptr<ControlPlane> make_threads_ctrl(World* w, int rank);
std::unique_ptr<ControlPlane> make_single_ctrl();
std::unique_ptr<ControlPlane> make_nccl_ctrl(ncclComm_t comm, int rank, int size, int device);
std::unique_ptr<Transport> make_threads_transport(World* w, int rank, int device, double timeout_s);
std::unique_ptr<Transport> make_nccl_transport(ncclComm_t comm, int rank, int device);

// ------------------------------------------------------------ star forest
enum class SfState { created = 0, graph_set = 1, set_up = 2 };
enum class SetupAlg { automatic = 0, dense = 1, consensus = 2 };

// One neighbor group, aligned across the pair (starforest.hpp:47-55,110-121).
struct Group {
  int rank = -1;
  HostVec<int64_t> items;  // root groups: leaf ordinals; leaf groups: root offsets
  Pattern pat;                 // root groups: leaf-index pattern; leaf groups: root pattern
  const int64_t* ditems = nullptr;  // device SetUp: items in HBM (host copy made on demand)
  int64_t count() const { return pat.count; }
};

// Graph and SetUp products of a forest whose graph was given in device
// memory (set_graph_device). SetUp then runs on the GPU
// (dsetup.cu); host copies of the groups are only made when a host-side
// consumer (degrees, multi-SF, algebra, CSR build, group export) asks.
struct DevGraph {
  int device = -1;
  int64_t* local = nullptr;  // leaf indices, nullptr = identity
  int32_t* rank = nullptr;
  int64_t* off = nullptr;
  bool ascending = true;     // leaf indices strictly increasing
  int64_t* ords = nullptr;   // root groups' items (leaf ordinals), groups back to back
  int64_t* ridx = nullptr;   // their leaf indices (== ords when local is nullptr)
  int64_t* loffs = nullptr;  // leaf groups' items (root offsets), groups back to back
  bool host_ready = false;   // host copies made
  ~DevGraph();
};

// Device-resident plan (built once per forest, on first use).
struct DevPlan {
  bool built = false;
  void* blob = nullptr;  // all device index arrays
  bool has_self = false;
  int64_t n_self = 0;
  DPat self_root, self_leaf;
  struct Seg {
    int rank;
    int64_t n;
    int64_t stage_off;  // vertices
    DPat pat;
    bool contiguous;
    int64_t contig_start;
    int64_t distinct;  // distinct indices of `pat`
  };
  int64_t self_root_distinct = 0;
  std::vector<Seg> rg;  // remote root groups (I own the leaves)
  std::vector<Seg> lg;  // remote leaf groups (I own the roots)
  int64_t n_leafside = 0;  // total remote edges, leaf side
  int64_t n_rootside = 0;  // total remote edges, root side
  bool self_root_dups = false;
  bool remote_root_dups = false;
  // root-sorted CSR (lazy)
  bool csr_built = false;
  void* csr_blob = nullptr;
  int64_t csr_n = 0;
  int32_t* csr_roots = nullptr;
  int32_t* csr_off = nullptr;    // [csr_n + 1]
  int32_t* csr_split = nullptr;  // [csr_n]: end of self entries
  int32_t* csr_ent = nullptr;
  int64_t csr_self_entries = 0;
  int64_t csr_remote_entries = 0;
  // L2 tiling of the self contributions: boundaries at multiples of
  // csr_piece_leaves leaf indices, csr_np_max - 1 per root (row-major).
  int32_t csr_np_max = 1;
  int64_t csr_piece_leaves = 0;
  int32_t* csr_ptab = nullptr;
  // remote-only CSR: just the roots that receive remote contributions
  int64_t rcsr_n = 0;
  int32_t* rcsr_roots = nullptr;
  int32_t* rcsr_off = nullptr;  // [rcsr_n + 1]
  int32_t* rcsr_ent = nullptr;
  // "coupled" roots (self AND remote contributions): their whole fold (self
  // entries then remote, the reference order) runs in End from the full CSR
  // (ccsr_lo/hi index csr_ent, aligned with rcsr_roots); Begin's local
  // reduction skips them (coupled_bits, one bit per root), so it can run
  // concurrently with the exchange and the End fold.
  int32_t* ccsr_lo = nullptr;
  int32_t* ccsr_hi = nullptr;
  uint32_t* coupled_bits = nullptr;
  int64_t ccsr_entries = 0;
  ~DevPlan();
};

// Where this rank writes inside peer r's staging slot (p2p backend). The
// slot is one allocation [leaf_stage | root_stage | leaf_reply | flags],
// mapped into every neighbor (CUDA IPC across processes, a plain peer pointer
// between threads of one process).
struct PeerSlot {
  char* base = nullptr;   // peer's slot allocation as mapped here
  bool ipc = false;       // opened with cudaIpcOpenMemHandle
  size_t root_at = 0, reply_at = 0, flags_at = 0;  // byte offsets inside the slot
  int64_t leaf_off = -1;  // peer's leaf-stage vertex offset of my group (its rg)
  int64_t root_off = -1;  // peer's root-stage vertex offset of my group (its lg)
  // LL128 slots: my group's first line in the peer's leaf / root (and reply)
  // regions, and the peer's words per parity buffer of each region
  int64_t leaf_line = -1, root_line = -1;
  int64_t par[3] = {0, 0, 0};
};

struct Staging {
  size_t unit_bytes = 0;
  void* leaf_stage = nullptr;   // n_leafside * ub
  void* root_stage = nullptr;   // n_rootside * ub
  void* leaf_reply = nullptr;   // n_leafside * ub (fetch-and-op)
  unsigned long long* digest = nullptr;
  cudaEvent_t released = nullptr;
  bool released_recorded = false;
  unsigned long long released_capture = 0;  // capture id the release was recorded in (0: none)
  bool in_use = false;
  bool retired = false;  // freed handle never ended (p2p): never reused
  size_t leaf_bytes = 0, root_bytes = 0;
  // p2p: one allocation holding the three stages (regions: 0 leaf stage,
  // 1 root stage, 2 leaf reply) and the flags
  //   arrive[3][P], free[3][P]  (uint64, written by peers)
  //   sent[3][P], recvd[3][P]   (uint64 local message counters)
  //   seg_counts[3][P], done_count (uint32 CTA arrival counters: one per
  //   put channel, one for the launches that acknowledge)
  // Per directed pair and region: the n-th put from me into region g of
  // peer d waits for free[g][d] >= n-1 (d consumed my previous message
  // there) and raises d.arrive[g][me] = n; the n-th message from s into my
  // region g is consumed after arrive[g][s] >= n and acknowledged with
  // s.free[g][me] = n. (One channel per region keeps fetch-and-op's reply
  // puts independent of the acknowledgement of the request they answer.)
  // The kernels advance the counters themselves — no host bookkeeping — so
  // operations can be captured into a CUDA graph and replayed.
  void* slot_mem = nullptr;
  // LL128 protocol (unit bytes a multiple of 8): the three regions receive
  // LL128 lines, two messages per channel; incoming root-side messages are
  // copied into the plain root_stage (its own allocation) for the folds.
  bool ll = false;
  void* ll_region[3] = {nullptr, nullptr, nullptr};
  int64_t ll_par[3] = {0, 0, 0};        // words per parity buffer of each region
  std::vector<int64_t> rg_line, lg_line;  // first line of each of my groups (rg: regions 0/2, lg: region 1)
  void* plain_root = nullptr;
  unsigned long long* flags = nullptr;
  unsigned int* seg_counts = nullptr;
  unsigned int* done_count = nullptr;
  int nranks = 0;
  unsigned long long* sent(int g, int r) const { return flags + (6 + g) * nranks + r; }
  unsigned long long* recvd(int g, int r) const { return flags + (9 + g) * nranks + r; }
  unsigned int* seg_count(int g, int r) const { return seg_counts + g * nranks + r; }
  std::vector<PeerSlot> peers;  // by rank
  const unsigned long long* arrive_flag(int g, int src) const { return flags + g * nranks + src; }
  const unsigned long long* free_flag(int g, int dst) const { return flags + (3 + g) * nranks + dst; }
  unsigned long long* peer_arrive_flag(int g, int peer, int me) const {
    const PeerSlot& p = peers[static_cast<size_t>(peer)];
    return reinterpret_cast<unsigned long long*>(p.base + p.flags_at) + g * nranks + me;
  }
  unsigned long long* peer_free_flag(int g, int peer, int me) const {
    const PeerSlot& p = peers[static_cast<size_t>(peer)];
    return reinterpret_cast<unsigned long long*>(p.base + p.flags_at) + (3 + g) * nranks + me;
  }
  ~Staging();
};

class StarForest {
 public:
  explicit StarForest(Comm* comm);
  ~StarForest();

  void set_graph(int64_t nroots, int64_t nleaves, const int64_t* leaf_local,
                 const int32_t* remote_rank, const int64_t* remote_off);
  // Same contract, arrays in the communicator's device memory (dsetup.cu).
  void set_graph_device(int64_t nroots, int64_t nleaves, const int64_t* leaf_local,
                        const int32_t* remote_rank, const int64_t* remote_off);
  void setup(SetupAlg alg = SetupAlg::automatic);
  bool device_graph() const { return dg_ != nullptr; }
  // Host copies of a device-set graph and its groups (no-op otherwise).
  void host_graph() const;
  void setup_device();  // setup() of a device-set graph (dsetup.cu)

  Comm& comm() { return *comm_; }
  SfState state() const { return state_; }
  int64_t nroots() const { return nroots_; }
  int64_t nleaves() const { return nleaves_; }
  int64_t leaf_index_bound() const { return leaf_bound_; }
  bool contiguous_leaves() const { return contiguous_leaves_; }
  int64_t leaf_index(int64_t ordinal) const {
    return leaf_local_.empty() ? ordinal : leaf_local_[static_cast<size_t>(ordinal)];
  }
  const std::vector<Group>& root_groups() const;
  const std::vector<Group>& leaf_groups() const;
  bool has_self_edges() const;
  std::vector<int64_t> compute_degrees() const;
  StarForest& multi_sf();
  void require_state(SfState s, const char* what) const;

  // device side
  DevPlan& dev();
  void ensure_csr();
  void ensure_csr_host();
  // Everything the first operation of unit size `ub` would otherwise build
  // inside Begin/End (host syncs, cudaMalloc, the p2p slot's collective
  // attachment): the device plan, the root-sorted CSR when some root has
  // several leaves, and a free staging slot of that unit size. Collective
  // (p2p). SetUp calls it for 8-byte units on a device communicator; after
  // it, such operations can be captured into a CUDA graph from the start.
  void prepare(size_t ub);
  void prepare_default();
  bool prepared() const;  // device plan (+ CSR where needed) built
  Staging* acquire_staging(size_t ub, cudaStream_t stream);
  void release_staging(Staging* s, cudaStream_t stream);
  void p2p_attach(Staging& s);  // collective: allocate the slot, map it into the neighbors

  int32_t remote_rank_of(int64_t o) const { return remote_rank_[static_cast<size_t>(o)]; }
  int64_t remote_off_of(int64_t o) const { return remote_off_[static_cast<size_t>(o)]; }
  bool has_local() const { return has_local_; }

 private:
  Comm* comm_;
  SfState state_ = SfState::created;
  int64_t nroots_ = 0, nleaves_ = 0, leaf_bound_ = 0;
  bool contiguous_leaves_ = true;
  bool has_local_ = false;
  // mutable: host_graph() fills them lazily for device-set graphs
  mutable HostVec<int64_t> leaf_local_;
  mutable HostVec<int32_t> remote_rank_;
  mutable HostVec<int64_t> remote_off_;
  mutable std::vector<Group> root_groups_, leaf_groups_;
  bool self_first_ = false;
  std::unique_ptr<DevGraph> dg_;
  std::unique_ptr<StarForest> multi_;
  std::unique_ptr<DevPlan> dev_;
  std::vector<std::unique_ptr<Staging>> staging_;
  // Message order of the remote groups (build_wire_order): the group itself
  // when its items already travel in root order, else a re-sorted copy.
  std::vector<const Group*> wire_rg_, wire_lg_;
  std::vector<std::unique_ptr<Group>> wire_store_;
  void build_wire_order(bool self);
};

bool stream_capturing(cudaStream_t s);

// ------------------------------------------------------------ operations
// /root/reference/proj/include/sf/ops.hpp:14-94
enum class OpKind : uint8_t { bcast = 0, reduce, fetch_and_op, gather, scatter };

struct OpHandle {
  StarForest* sf = nullptr;  // forest the transfer runs over (multi-SF for gather/scatter)
  OpKind kind = OpKind::bcast;
  Unit unit;
  ReduceOp op = ReduceOp::replace;
  const void* src = nullptr;
  void* dst = nullptr;
  void* leafupdate = nullptr;
  uint64_t opid = 0;
  bool ended = false;
  bool xfer = false;  // this op has transport work
  cudaStream_t stream = nullptr;
  Staging* stg = nullptr;
  std::vector<XferOp> recvs;        // phase-1 receives
  std::vector<XferOp> reply_recvs;  // fetch-and-op replies
  bool forked = false;              // p2p: the puts ran on the comm stream
  bool fused_unpack = false;        // p2p Bcast: the unpack ran in the put launch
  bool ll_direct = false;           // p2p Reduce: remote contributions applied in the put launch
  bool immediate = false;           // one-shot form: End follows Begin with nothing in between
  bool coupled_split = false;       // reduce: coupled roots folded in End (DevPlan::coupled_bits)
  std::vector<uint8_t> zero_copy_recv;
  std::vector<int32_t> fetch_order;  // free-order fetch: group order used (empty: stored order)
  // debug checksum
  const void* ck_ptr = nullptr;
  size_t ck_bytes = 0;
  unsigned long long ck_value = 0;
  // host-memory staging (reference-style host pointers)
  bool host_mode = false;
};

std::unique_ptr<OpHandle> bcast_begin(StarForest& sf, const Unit& u, const void* rootdata,
                                      void* leafdata, ReduceOp op, cudaStream_t s);
void bcast_end(OpHandle& h);
std::unique_ptr<OpHandle> reduce_begin(StarForest& sf, const Unit& u, const void* leafdata,
                                       void* rootdata, ReduceOp op, cudaStream_t s);
void reduce_end(OpHandle& h);
std::unique_ptr<OpHandle> fetch_and_op_begin(StarForest& sf, const Unit& u, void* rootdata,
                                             const void* leafdata, void* leafupdate, ReduceOp op,
                                             cudaStream_t s);
void fetch_and_op_end(OpHandle& h);
std::unique_ptr<OpHandle> gather_begin(StarForest& sf, const Unit& u, const void* leafdata,
                                       void* multirootdata, cudaStream_t s);
void gather_end(OpHandle& h);
std::unique_ptr<OpHandle> scatter_begin(StarForest& sf, const Unit& u, const void* multirootdata,
                                        void* leafdata, cudaStream_t s);
void scatter_end(OpHandle& h);
// One-shot forms (ops.hpp:60-94), stream-ordered: Begin and End back to back.
void bcast(StarForest& sf, const Unit& u, const void* rootdata, void* leafdata, ReduceOp op, cudaStream_t s);
void reduce(StarForest& sf, const Unit& u, const void* leafdata, void* rootdata, ReduceOp op, cudaStream_t s);
void fetch_and_op(StarForest& sf, const Unit& u, void* rootdata, const void* leafdata, void* leafupdate,
                  ReduceOp op, cudaStream_t s);
void gather(StarForest& sf, const Unit& u, const void* leafdata, void* multirootdata, cudaStream_t s);
void scatter(StarForest& sf, const Unit& u, const void* multirootdata, void* leafdata, cudaStream_t s);

DPat to_dpat(const Pattern& p, const int32_t* dev_idx);

// Device SetUp helpers (dsetup.cu), on the current device, synchronous.
// Planner scratch from the stream-ordered pool (ordered on cudaStreamPerThread).
void* dev_pool_alloc(size_t bytes);
void dev_pool_free(void* p);
// dst[i] = src[i] as int32; throws when a value exceeds the int32 range.
void dev_narrow_index(const int64_t* src, int64_t n, int32_t* dst);
// CSR build (StarForest::ensure_csr): keys/vals to int32 pairs (vals ==
// nullptr: remote entries -(base+i)-1), then the root-sorted CSR into d.
void dev_csr_fill(const int64_t* keys, const int64_t* vals, int64_t n, int64_t base, int32_t* kout,
                  int32_t* vout);
struct DevPlan;
void dev_build_csr(DevPlan& d, int32_t* key, int32_t* val, int64_t total, int64_t n_self, int64_t nroots,
                   int64_t leaf_bound, bool self);
// Whether keys never decrease: items[i] (src == nullptr) or src[items[i]].
bool dev_keys_sorted(const int64_t* items, const int64_t* src, int64_t n);
// Whether any value in [0, bound) occurs twice across the lists.
bool dev_any_repeat(const std::vector<std::pair<const int64_t*, int64_t>>& lists, int64_t bound);

// ------------------------------------------------------- graph algebra
// starforest.hpp:150-171 (algebra.cpp). Collective; results are set up
// (identity_sf: graph set).
std::unique_ptr<StarForest> compose(StarForest& A, StarForest& B);
std::unique_ptr<StarForest> compose_inverse(StarForest& A, StarForest& B);
std::unique_ptr<StarForest> embed_root(StarForest& f, const int64_t* sel, int64_t nsel);
std::unique_ptr<StarForest> embed_leaf(StarForest& f, const int64_t* sel, int64_t nsel);
std::unique_ptr<StarForest> identity_sf(Comm& c, int64_t n);

// ------------------------------------------------------- SpMV consumer
// Device matrix block for the distributed SpMV (spmv.cu; reference
// Csr<T> / SplitMatrix<T>, spmv.hpp:31-127): SELL-32 images of the block
// and of its transpose.
struct DevMatrix {
  struct Sell {
    int64_t rows = 0, cols = 0, nnz = 0, slots = 0;
    int64_t* slice_off = nullptr;
    int32_t* row_len = nullptr;
    int32_t* col = nullptr;
    void* val = nullptr;
    int64_t n_nz_rows = 0;        // rows with at least one entry
    int32_t* nz_rows = nullptr;   // their indices, ascending
  };
  int device = -1;
  Kind kind = Kind::float64;
  int64_t rows = 0, cols = 0, nnz = 0;
  Sell fwd, bwd;  // the block and its transpose
  std::vector<void*> allocs;
  ~DevMatrix();
};
std::unique_ptr<DevMatrix> matrix_upload(Comm& comm, int64_t rows, int64_t cols, const int64_t* rowptr,
                                         const int64_t* colind, const void* vals, Kind kind);
void spmv(StarForest& sf, const DevMatrix& diag, const DevMatrix& off, const void* x_owned, void* lvec,
          void* y, cudaStream_t s);
void spmv_transpose(StarForest& sf, const DevMatrix& diag, const DevMatrix& off, const void* x_owned,
                    void* lvec, void* y, cudaStream_t s);

}  // namespace sfg
