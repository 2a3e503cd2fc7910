// Split-phase operations: Bcast, Reduce, FetchAndOp, Gather, Scatter.
//
// Reference engines: /root/reference/proj/src/ops.cpp
//   root->leaf two-sided  :276-324   (bcast, scatter)
//   leaf->root two-sided  :326-376   (reduce, gather)
//   one-sided engines     :160-246, 381-476, 572-658 (the p2p backend here)
//   fetch-and-op          :481-570
//   public begin/end      :697-876
// Per Begin: the exchange is forked onto the communicator's stream — ONE
// launch packs every remote group (p2p: straight into the peers' slots over
// NVLink; nccl: into staging, then ONE grouped send/recv; contiguous groups
// are zero-copy sends) — while the local (self-edge) scatter runs on the
// caller's stream (or joins the pack launch when small). Per End: ONE unpack
// launch (on the comm stream when it cannot conflict with the local scatter:
// Reduce's fold of the "coupled" roots), then the caller's stream joins; a
// p2p Bcast's unpack is already part of the put launch, so its End only
// joins. Nothing synchronises the host with the GPU (§V
// "stream-aware, sync-free").
//
// Fold order. Where a reduction can hit the same root more than once, the
// fold runs through a root-sorted CSR in exactly the reference order —
// initial value, self edges by ascending leaf index, then remote ranks
// ascending, each in ascending leaf index (ops.cpp:364,372-376;
// oracle.cpp:84-90) — so floating-point results are bit-identical to the CPU
// reference. Free-order fetch-and-op applies the contribution groups in the
// reference's shuffled order (ops.cpp:531-544).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "sfg.hpp"

namespace sfg {
namespace {

constexpr int kOpReplace = 0;

// The reference's splitmix64 generator and seed mixing
// (/root/reference/proj/include/sf/rng.hpp:14-51).
struct SplitMix {
  uint64_t state;
  explicit SplitMix(uint64_t seed) : state(seed + 0x9e3779b97f4a7c15ull) {}
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  template <class T>
  void shuffle(std::vector<T>& v) {
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[next() % i]);
  }
};

uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  SplitMix r(seed ^ (salt * 0xd1342543de82ef95ull + 0x2545f4914f6cdd1dull));
  return r.next();
}

DPat contig(int64_t start) {
  DPat p;
  p.kind = PAT_CONTIG;
  p.start = start;
  return p;
}

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Length of the runs that are contiguous on both sides of a pair, or 0.
int64_t common_run(const DPat& a, const DPat& b, int64_t n) {
  if (a.kind == PAT_INDEXED || b.kind == PAT_INDEXED || n <= 0) return 0;
  const int64_t ra = a.kind == PAT_CONTIG ? n : static_cast<int64_t>(a.dx.d);
  const int64_t rb = b.kind == PAT_CONTIG ? n : static_cast<int64_t>(b.dx.d);
  const int64_t g = gcd64(ra, rb);
  return g >= 16 && g < (int64_t(1) << 31) ? g : 0;
}

DSeg pair_seg(const DPat& src, int sbuf, const DPat& dst, int dbuf, int64_t n, bool replace) {
  DSeg s;
  s.src = src;
  s.dst = dst;
  s.src_buf = sbuf;
  s.dst_buf = dbuf;
  s.n = n;
  s.replace = replace ? 1 : 0;
  s.type = SEG_PAIR;
  s.run = common_run(src, dst, n);
  if (s.run) s.rundiv = make_fastdiv(static_cast<uint32_t>(s.run));
  return s;
}

enum class CsrRange { self_only, remote_only, all };

// seq: keep the exact sequential fold order inside a warp (float data in
// deterministic mode). High-degree roots get a warp each.
DSeg csr_seg(const DevPlan& d, CsrRange range, int32_t type, bool seq, size_t ub) {
  DSeg s;
  s.type = type;
  const int64_t entries = range == CsrRange::self_only ? d.csr_self_entries
                          : range == CsrRange::remote_only ? d.csr_remote_entries
                                                           : d.csr_self_entries + d.csr_remote_entries;
  s.csr_warp = d.csr_n > 0 && entries >= 8 * d.csr_n ? 1 : 0;
  s.csr_seq = seq ? 1 : 0;
  s.n = d.csr_n;
  s.src_buf = BUF_SRC_RO;
  s.dst_buf = BUF_ROOT;
  s.aux_buf = BUF_LEAFUPDATE;
  s.stage_buf = BUF_ROOT_STAGE;
  s.csr_roots = d.csr_roots;
  s.csr_ent = d.csr_ent;
  switch (range) {
    case CsrRange::self_only:
      s.csr_lo = d.csr_off;
      s.csr_hi = d.csr_split;
      break;
    case CsrRange::remote_only:
      s.n = d.rcsr_n;
      s.csr_roots = d.rcsr_roots;
      s.csr_ent = d.rcsr_ent;
      s.csr_lo = d.rcsr_off;
      s.csr_hi = d.rcsr_off + 1;
      s.csr_warp = d.rcsr_n > 0 && entries >= 8 * d.rcsr_n ? 1 : 0;
      break;
    case CsrRange::all:
      s.csr_lo = d.csr_off;
      s.csr_hi = d.csr_off + 1;
      break;
  }
  // L2 tiling: pieces of the leaf (and, for fetch, leafupdate) arrays that
  // together fit a ~40 MB window of the 126 MB L2.
  static const bool no_pieces = std::getenv("SFG_NO_L2_PIECES") != nullptr;
  if (range != CsrRange::remote_only && d.csr_ptab && d.csr_np_max > 1 && !no_pieces) {
    const double window = 40e6;
    const double per_piece = static_cast<double>(ub) * static_cast<double>(d.csr_piece_leaves) *
                             (type == SEG_CSR_FETCH ? 2.0 : 1.0);
    const int step = std::max(1, static_cast<int>(window / per_piece));
    const int np = (d.csr_np_max + step - 1) / step;
    if (np > 1) {
      s.csr_np = np;
      s.csr_pt_stride = d.csr_np_max - 1;
      s.csr_pt_step = step;
      s.csr_ptab = d.csr_ptab;
    }
  }
  // Thread per root (sequential fold, no shuffles: one warp instruction
  // advances 32 roots) whenever there are enough roots to spread over the
  // GPU; a warp per root only for few, very high-degree roots.
  // Order-free fetch-and-op (integer ops, free-order mode) keeps a warp per
  // root (warp scan, exact for them) below 65,536 roots: the fetch's thread
  // chains are the slower ones, and with that few roots they leave the GPU
  // mostly idle (config 4 at N=4: fetch End 170 -> 100 us; the same rule for
  // Begin's local fold made it 8 -> 58 us, so that fold stays thread per root).
  static const int64_t warp_limit = [] {
    const char* e = std::getenv("SFG_CSR_WARP_LIMIT");
    return e ? std::atoll(e) : int64_t(32768);
  }();
  // Deterministic float fetches too, keeping the exact sequential order
  // through shuffles: config 4 at N=4 (16,384 roots per rank) FetchAndOp f64
  // 309 -> 256 us (profiles/r2_cfg4_n4*.log); SFG_CSR_NO_WARP_SEQ restores
  // thread per root for them.
  // The fetch's limit is twice the fold's: at 32,768 roots (config 4 at N=2)
  // the warp form still wins for the fetch (End 425 -> 398 us f64, 428 ->
  // 345 us i64) but loses for the fold (Reduce i64 170 -> 197 us); at 65,536
  // (N=1) thread per root wins for both (fetch 223 vs 460 us).
  static const bool no_warp_seq = std::getenv("SFG_CSR_NO_WARP_SEQ") != nullptr;
  const bool warp_fetch = type == SEG_CSR_FETCH && (!seq || !no_warp_seq) && s.n < 2 * warp_limit;
  // End's order-free folds (integers, free-order floats) over the roots that
  // receive remote contributions (every root of a rank in config 4 at N>1,
  // ~256 contributions each) likewise: config 4 Reduce at N=4 143 -> 125 us.
  // The exact-order float fold stays thread per root there (warp: 149 us).
  static const bool no_warp_end = std::getenv("SFG_CSR_NO_WARP_END") != nullptr;  // ablation
  const bool warp_end =
      type == SEG_CSR_FOLD && range == CsrRange::remote_only && !no_warp_end && !seq && s.n < warp_limit;
  if (s.n >= 8192 && !warp_fetch && !warp_end) s.csr_warp = 0;
  return s;
}

// Accumulates the segments of one operation phase, picks the element type
// and issues them. A phase is normally ONE kernel launch; when it holds more
// segments, flag waits or peer buffers than one launch's parameter block
// (kMaxSegs / kMaxPeers), it is split IN ORDER into several launches on the
// same stream — puts stay ahead of the receives that wait on peers, and the
// completion flags (acknowledgements) are raised by the last launch, after
// every earlier one finished — so any number of neighbour groups works.
struct Launch {
  struct Item {
    DSeg seg;
    std::vector<int> waits;  // indices into `waits`
    void* peer = nullptr;    // p2p put: the peer's mapped slot base
    bool remote_put = false;
    int64_t entries = 0, distinct_src = 0, distinct_dst = 0;
  };
  struct Done {
    unsigned long long* flag;
    unsigned long long* seq;
  };
  std::vector<Item> items;
  std::vector<FlagWait> waits;
  std::vector<Done> dones;
  unsigned int* done_count = nullptr;
  void* bufs[BUF_PEER0] = {};
  FetchShuffle shuffle;
  bool done_relaxed = false;  // LL128 acknowledgements (kernels.cu st_relaxed_sys)
  bool interleave = false;    // LL128: dispatch receive CTAs among the put CTAs
  bool any_op = false;
  const char* tag = "kernel";

  int nseg() const { return static_cast<int>(items.size()); }

  // entries: CSR contributions; src_distinct / dst_distinct: distinct
  // indices of the two patterns (-1 = all distinct), for algorithmic bytes.
  void add(const DSeg& s, int64_t entries = 0, int64_t src_distinct = -1, int64_t dst_distinct = -1,
           std::vector<int> w = {}) {
    if (s.n <= 0) return;
    Item it;
    it.seg = s;
    it.seg.wait_mask = 0;
    it.waits = std::move(w);
    it.entries = entries;
    it.distinct_src = src_distinct < 0 ? s.n : src_distinct;
    it.distinct_dst = dst_distinct < 0 ? s.n : dst_distinct;
    if (!s.replace) any_op = true;
    items.push_back(std::move(it));
  }

  // Append another phase's segments (its own buffers are the same slots).
  void absorb(const Launch& o) {
    for (const auto& it : o.items) {
      Item c = it;
      for (int& w : c.waits) w += static_cast<int>(waits.size());
      items.push_back(std::move(c));
      if (!it.seg.replace) any_op = true;
    }
    waits.insert(waits.end(), o.waits.begin(), o.waits.end());
  }

  // p2p: wait until *flag >= *count + delta; returns the wait's index.
  int add_wait(const unsigned long long* flag, const unsigned long long* count, uint64_t delta) {
    waits.push_back(FlagWait{flag, count, delta});
    return static_cast<int>(waits.size()) - 1;
  }

  // p2p: once every CTA of the phase is done, ++*seq and publish it in flag.
  void add_done(unsigned long long* flag, unsigned long long* seq, unsigned int* counter) {
    dones.push_back(Done{flag, seq});
    done_count = counter;
  }

  // One-sided put into a peer's slot (p2p) at vertex offset `peer_off`; it
  // waits for `wait`, and its completion advances *seq and publishes it in
  // `flag` (sig_count: the segment's CTA arrival counter).
  void add_put(const DPat& src, int sbuf, void* base, int64_t peer_off, int64_t n, int wait,
               unsigned int* sig_count, unsigned long long* flag, unsigned long long* seq, bool remote,
               int64_t src_distinct = -1) {
    DSeg s = pair_seg(src, sbuf, contig(peer_off), BUF_PEER0, n, true);
    s.sig_count = sig_count;
    s.sig_flag = flag;
    s.sig_seq = seq;
    add(s, 0, src_distinct, -1, {wait});
    items.back().peer = base;
    items.back().remote_put = remote;
  }

  // LL128 put into a peer's region (see kernels.hpp): credit wait `wait`,
  // the channel's message counter `seq` (sent), its CTA counter `sig_count`.
  void add_put_ll(const DPat& src, int sbuf, void* region, int64_t line, int64_t par, int64_t n,
                  const unsigned long long* credit, unsigned int* sig_count, unsigned long long* seq, bool remote,
                  int64_t src_distinct = -1) {
    DSeg s = pair_seg(src, sbuf, contig(0), BUF_PEER0, n, true);
    s.type = SEG_PUT_LL;
    s.run = 0;
    s.ll_line = line;
    s.ll_par = par;
    s.ll_credit = credit;
    s.sig_count = sig_count;
    s.sig_seq = seq;
    add(s, 0, src_distinct, -1);
    items.back().peer = region;
    items.back().remote_put = remote;
  }

  void run(const Unit& u, ReduceOp op, cudaStream_t st) {
    if (items.empty()) return;
    ElemType t;
    int kop = static_cast<int>(op);
    int64_t bl = 1;
    if (!any_op) {
      // Verbatim move: widest word that divides the vertex size and the
      // alignment of every buffer involved.
      uintptr_t align = u.bytes();
      for (int b = 0; b < BUF_PEER0; ++b)
        if (bufs[b]) align |= reinterpret_cast<uintptr_t>(bufs[b]);
      for (const auto& it : items)
        if (it.peer) align |= reinterpret_cast<uintptr_t>(it.peer);
      const size_t ub = u.bytes();
      if ((align & 7) == 0) {
        t = ElemType::u64;
        bl = static_cast<int64_t>(ub / 8);
      } else if ((align & 3) == 0) {
        t = ElemType::u32;
        bl = static_cast<int64_t>(ub / 4);
      } else if ((align & 1) == 0) {
        t = ElemType::u16;
        bl = static_cast<int64_t>(ub / 2);
      } else {
        t = ElemType::u8;
        bl = static_cast<int64_t>(ub);
      }
      kop = kOpReplace;
    } else {
      switch (u.kind) {
        case Kind::int32: t = ElemType::i32; break;
        case Kind::int64: t = ElemType::i64; break;
        case Kind::float64: t = ElemType::f64; break;
        default: fail("reduction requires a non-opaque unit kind");
      }
      bl = u.blocklen;
    }
    const bool timed = timing_enabled();
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
      e0 = timing_event();
      e1 = timing_event();
      SFG_CUDA(cudaEventRecord(e0, st));
    }
    // Greedy in-order split into launches that fit the parameter block.
    size_t i = 0;
    int launched = 0;
    while (i < items.size()) {
      LaunchParams p{};
      std::copy(bufs, bufs + BUF_PEER0, p.bufs);
      p.trace = trace_slot();
      p.ilv_a = interleave ? -1 : 0;
      static const int poll_ns = [] {
        const char* e = std::getenv("SFG_LL_POLL_NS");
        return e ? std::atoi(e) : 20;
      }();
      p.ll_poll_ns = poll_ns;
      p.bl = bl;
      p.wpv = static_cast<int64_t>(u.bytes() / 8);
      p.shuf = shuffle;
      std::vector<int> wmap(waits.size(), -1);
      int nw = 0, npeer = 0;
      while (i < items.size() && p.nseg < kMaxSegs) {
        const Item& it = items[i];
        int need = 0;
        for (int w : it.waits)
          if (wmap[static_cast<size_t>(w)] < 0) ++need;
        if (p.nseg > 0 && (nw + need > kMaxPeers || (it.peer && npeer + 1 > kMaxPeers))) break;
        SFG_REQUIRE(need <= kMaxPeers, "one segment waits on more than kMaxPeers flags");
        DSeg s = it.seg;
        for (int w : it.waits) {
          int& m = wmap[static_cast<size_t>(w)];
          if (m < 0) {
            m = nw++;
            p.waits[m] = waits[static_cast<size_t>(w)];
          }
          s.wait_mask |= 1u << m;
        }
        if (it.peer) {
          s.dst_buf = BUF_PEER0 + npeer;
          p.bufs[BUF_PEER0 + npeer] = it.peer;
          ++npeer;
        }
        p.seg[p.nseg++] = s;
        ++i;
      }
      const bool last = i == items.size();
      if (last && static_cast<int>(dones.size()) <= kMaxPeers) {
        for (const auto& d : dones) {
          p.done_flag[p.ndone] = d.flag;
          p.done_seq[p.ndone] = d.seq;
          ++p.ndone;
        }
        p.done_count = done_count;
        p.done_relaxed = done_relaxed ? 1 : 0;
      }
      const int r = launch_segments(p, t, kop, st);
      SFG_REQUIRE(r >= 0, "no kernel instantiation for this unit/op combination");
      SFG_CUDA(cudaGetLastError());
      launched += r;
      if (last && static_cast<int>(dones.size()) > kMaxPeers) {
        // more acknowledgements than one parameter block holds: raise them
        // from a signalling kernel behind the data launches
        std::vector<unsigned long long*> f, q;
        for (const auto& d : dones) {
          f.push_back(d.flag);
          q.push_back(d.seq);
        }
        launch_signal(f.data(), q.data(), static_cast<int>(f.size()), st);
        SFG_CUDA(cudaGetLastError());
        ++launched;
      }
    }
    counters().kernel_launches += static_cast<uint64_t>(launched);
    if (timed) {
      SFG_CUDA(cudaEventRecord(e1, st));
      double link = 0;
      for (const auto& it : items) link += it.remote_put ? static_cast<double>(it.seg.n) * u.bytes() : 0.0;
      timing_record(tag, e0, e1, algorithmic_bytes(u), link);
    }
  }

  // Compulsory bytes of this phase: every element read once and written
  // once, destination reads for reductions, int32 indices of Indexed
  // patterns; affine/contiguous patterns cost no index traffic.
  double algorithmic_bytes(const Unit& u) const {
    const double ub = static_cast<double>(u.bytes());
    double b = 0;
    for (const auto& it : items) {
      const DSeg& g = it.seg;
      const double n = static_cast<double>(g.n);
      const double idx = 4.0 * n * ((g.src.kind == PAT_INDEXED) + (g.dst.kind == PAT_INDEXED));
      const double ds = static_cast<double>(it.distinct_src);
      const double dd = static_cast<double>(it.distinct_dst);
      switch (g.type) {
        case SEG_PAIR:
        case SEG_RECV_LL: b += ds * ub + dd * ub * (g.replace ? 1.0 : 2.0) + idx; break;
        case SEG_PUT_LL: b += ds * ub + n * ub * 128.0 / 120.0 + idx; break;
        case SEG_CSR_FOLD:
        case SEG_CSR_FETCH: {
          const double e = static_cast<double>(it.entries);
          b += n * ub * 2.0 + e * ub * (g.type == SEG_CSR_FETCH ? 2.0 : 1.0) + 4.0 * e + 12.0 * n;
          break;
        }
      }
    }
    return b;
  }
};

void set_bufs(Launch& L, const OpHandle& h, void* root, void* leaf, const void* src_ro) {
  L.bufs[BUF_ROOT] = root;
  L.bufs[BUF_LEAF] = leaf;
  L.bufs[BUF_SRC_RO] = const_cast<void*>(src_ro);
  if (h.stg) {
    L.bufs[BUF_LEAF_STAGE] = h.stg->leaf_stage;
    L.bufs[BUF_ROOT_STAGE] = h.stg->root_stage;
    L.bufs[BUF_LEAF_REPLY] = h.stg->leaf_reply;
  }
  L.bufs[BUF_LEAFUPDATE] = h.leafupdate;
  if (h.stg && h.stg->ll)
    for (int r = 0; r < 3; ++r) L.bufs[BUF_LL0 + r] = h.stg->ll_region[r];
}

uint64_t data_tag(uint64_t opid) { return opid * 2; }
uint64_t reply_tag(uint64_t opid) { return opid * 2 + 1; }

void* at(void* base, int64_t vertex, size_t ub) {
  return static_cast<char*>(base) + static_cast<size_t>(vertex) * ub;
}
const void* at(const void* base, int64_t vertex, size_t ub) {
  return static_cast<const char*>(base) + static_cast<size_t>(vertex) * ub;
}

unsigned long long digest(OpHandle& h, const void* p, size_t bytes) {
  launch_digest(p, bytes, h.stg->digest, h.stream);
  unsigned long long v = 0;
  SFG_CUDA(cudaMemcpyAsync(&v, h.stg->digest, sizeof(v), cudaMemcpyDeviceToHost, h.stream));
  SFG_CUDA(cudaStreamSynchronize(h.stream));
  return v;
}

void begin_common(OpHandle& h, const void* ck_ptr, size_t ck_bytes) {
  StarForest& sf = *h.sf;
  sf.comm().bind_device();
  h.opid = sf.comm().next_op_seq();
  SFG_REQUIRE(sf.prepared() || !stream_capturing(h.stream),
              "first operation on a forest inside a CUDA graph capture: call prepare(unit) on the "
              "set-up forest before capturing");
  (void)sf.dev();
  h.stg = sf.acquire_staging(h.unit.bytes(), h.stream);
  if (sf.comm().config().debug_checksum && ck_ptr != nullptr && ck_bytes > 0) {
    h.ck_ptr = ck_ptr;
    h.ck_bytes = ck_bytes;
    h.ck_value = digest(h, ck_ptr, ck_bytes);
  }
}

void end_common(OpHandle& h) {
  if (h.ck_ptr != nullptr) {
    const unsigned long long v = digest(h, h.ck_ptr, h.ck_bytes);
    if (v != h.ck_value) {
      h.sf->release_staging(h.stg, h.stream);
      h.stg = nullptr;
      fail("buffer mutated between begin and end of a split-phase operation");
    }
  }
  if (h.stg) h.sf->release_staging(h.stg, h.stream);
  h.stg = nullptr;
}

// Root-sorted CSR execution for every reduction with duplicate roots, in
// both modes: the thread-per-root fold beats native atomics at every degree
// measured (config 1, degree 4: 44.5 us vs 54.8 us; config 4, degree 256:
// 164 us vs contended atomics, profiles/r1_configs.md) and is bit-exact, so
// the free-order atomics variant was removed in round 2.
void use_csr(StarForest& sf) { sf.ensure_csr(); }

// Reduce with self edges and remote contributions: Begin's local reduction
// skips the "coupled" roots (those that also receive remote contributions)
// and End folds them completely — self entries then remote ranks, the
// reference order — from the full CSR. The local reduction and the End fold
// then touch disjoint roots, so the End fold runs on the comm stream right
// behind the exchange while the local reduction is still running.
bool split_coupled(StarForest& sf, const OpHandle& h) {
  const DevPlan& d = sf.dev();
  if (h.op == ReduceOp::replace || !d.has_self || d.lg.empty()) return false;
  static const bool off = std::getenv("SFG_NO_COUPLED_SPLIT") != nullptr;
  if (off) return false;
  sf.ensure_csr();
  return d.coupled_bits != nullptr && d.ccsr_lo != nullptr && d.rcsr_n > 0;
}

// Exact sequential order is only needed for floating point; integer ops are
// associative under wrap-around, so tree/scan orders give identical bits.
bool exact_seq(const OpHandle& h, bool det) { return det && h.unit.kind == Kind::float64; }

// ------------------------------------------------------------ exchange phases
//
// Begin: the comm stream forks from the caller's stream, packs every remote
// group that is not zero-copy and posts the grouped transport call; the local
// (self-edge) scatter runs concurrently on the caller's stream. When the local
// segment is small it is fused into the pack launch instead (one launch, no
// overlap to win). End: the comm stream finishes the receives, the caller's
// stream joins it and unpacks.
constexpr double kFuseLocalBytes = 8.0 * (1 << 20);

const char* tag_of(const OpHandle& h, int phase) {  // 0 begin 1 end 2 pack 3 local
  static const char* names[5][4] = {
      {"bcast_begin", "bcast_end", "bcast_pack", "bcast_local"},
      {"reduce_begin", "reduce_end", "reduce_pack", "reduce_local"},
      {"fetch_begin", "fetch_end", "fetch_pack", "fetch_local"},
      {"gather_begin", "gather_end", "gather_pack", "gather_local"},
      {"scatter_begin", "scatter_end", "scatter_pack", "scatter_local"}};
  return names[static_cast<int>(h.kind)][phase];
}

void begin_phase(OpHandle& h, Launch& pack, Launch& local, const std::vector<XferOp>& sends,
                 const std::vector<XferOp>& recvs, uint64_t tag) {
  Comm& c = h.sf->comm();
  h.xfer = !sends.empty() || !recvs.empty();
  if (!h.xfer) {
    local.tag = tag_of(h, 0);
    local.run(h.unit, h.op, h.stream);
    return;
  }
  cudaStream_t cs = c.comm_stream();
  c.fork(h.stream);
  const bool fuse = local.algorithmic_bytes(h.unit) < kFuseLocalBytes;
  if (fuse) {
    pack.absorb(local);
    pack.tag = tag_of(h, 0);
  } else {
    pack.tag = tag_of(h, 2);
    local.tag = tag_of(h, 3);
  }
  pack.run(h.unit, h.op, cs);
  const bool timed = timing_enabled();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    e0 = timing_event();
    e1 = timing_event();
    SFG_CUDA(cudaEventRecord(e0, cs));
  }
  c.transport().start(tag, sends, recvs, cs);
  if (timed) {
    // Exchange interval on the comm stream (includes the rendezvous with the
    // peers); link bytes = what this rank sends to other ranks.
    SFG_CUDA(cudaEventRecord(e1, cs));
    double link = 0;
    for (const auto& s : sends)
      if (s.peer != c.rank()) link += static_cast<double>(s.bytes);
    static const char* xt[5] = {"bcast_xfer", "reduce_xfer", "fetch_xfer", "gather_xfer", "scatter_xfer"};
    timing_record(xt[static_cast<int>(h.kind)], e0, e1, 0.0, link);
  }
  counters().transport_calls++;
  if (!fuse) local.run(h.unit, h.op, h.stream);
}

void end_wait(OpHandle& h, uint64_t tag, const std::vector<XferOp>& recvs) {
  if (!h.xfer) return;
  Comm& c = h.sf->comm();
  c.transport().finish(tag, recvs, c.comm_stream());
  c.join(h.stream);
}

// ------------------------------------------------- one-sided (p2p) phases
//
// Message counts per directed pair and stage region (Staging) replace the
// reference's SendSig/RecvSig clearing (ops.cpp:160-246): the n-th put from
// me into region g of d's slot waits in-kernel for free[g][d] >= n-1 and
// raises d.arrive[g][me] = n; the unpack of the n-th message from s waits
// for arrive[g][s] >= n and its launch raises s.free[g][me] = n when done.
// The counters live on the device (advanced by the kernels). Per operation:
// one put launch on the comm stream (with the local scatter fused in when it
// is small, otherwise the local scatter runs concurrently on the caller's
// stream) and one unpack launch.
bool use_p2p(const OpHandle& h) { return h.sf->comm().p2p() && h.stg && h.stg->flags; }

// The puts always run on the comm stream, so whatever the caller enqueues on
// its stream between Begin and End (the local scatter, or its own work, e.g.
// the diagonal SpMV product) overlaps the exchange; a small local scatter
// joins the puts' launch instead.
void p2p_begin(OpHandle& h, Launch& pack, Launch& local,
               const std::function<void(Launch&)>& append_last = nullptr) {
  Comm& c = h.sf->comm();
  h.xfer = pack.nseg() > 0;
  h.forked = false;
  if (!h.xfer) {
    local.tag = tag_of(h, 0);
    local.run(h.unit, h.op, h.stream);
    return;
  }
  static const bool no_fork = std::getenv("SFG_P2P_NO_FORK") != nullptr;  // ablation
  const bool fuse_local = local.algorithmic_bytes(h.unit) < kFuseLocalBytes;
  // A one-shot operation (End right behind Begin) has no caller work to
  // overlap: its launch goes on the caller's stream, saving the fork / join
  // (2 MB halo Bcast at N=2: 10.3 -> 9.1 us).
  if ((no_fork || h.immediate) && fuse_local) {
    pack.absorb(local);
    pack.tag = tag_of(h, 0);
    if (append_last) append_last(pack);
    pack.run(h.unit, h.op, h.stream);
    counters().transport_calls++;
    return;
  }
  cudaStream_t cs = c.comm_stream();
  c.fork(h.stream);
  h.forked = true;
  if (fuse_local) {
    pack.absorb(local);
    pack.tag = tag_of(h, 0);
    if (append_last) append_last(pack);
    pack.run(h.unit, h.op, cs);
  } else {
    pack.tag = tag_of(h, 2);
    local.tag = tag_of(h, 3);
    if (append_last) append_last(pack);
    pack.run(h.unit, h.op, cs);
    local.run(h.unit, h.op, h.stream);
  }
  counters().transport_calls++;
}

// Before the unpack: order the caller's stream after this rank's own puts
// (they read the caller's buffers, and a spinning unpack must never starve
// them of SMs).
void p2p_join(OpHandle& h) {
  if (h.forked) h.sf->comm().join(h.stream);
  h.forked = false;
}

// Puts of `groups` from buffer `sbuf` (each group's own pattern, or its
// staging range when !use_pat) into each peer's stage `region` (0 leaf,
// 1 root, 2 reply).
void add_puts(OpHandle& h, Launch& L, const std::vector<DevPlan::Seg>& groups, bool use_pat,
              int sbuf, int region) {
  Staging& s = *h.stg;
  const int me = h.sf->comm().rank();
  const size_t ub = h.unit.bytes();
  for (size_t k = 0; k < groups.size(); ++k) {
    const auto& g = groups[k];
    const PeerSlot& ps = s.peers[static_cast<size_t>(g.rank)];
    char* base = ps.base + (region == 0 ? 0 : region == 1 ? ps.root_at : ps.reply_at);
    const int64_t off = region == 1 ? ps.root_off : ps.leaf_off;
    SFG_REQUIRE(off >= 0, "p2p: peer slot has no group for this rank");
    // my previous messages into this region of g.rank consumed
    const int w = L.add_wait(s.free_flag(region, g.rank), s.sent(region, g.rank), 0);
    L.add_put(use_pat ? g.pat : contig(g.stage_off), sbuf, base, off, g.n, w, s.seg_count(region, g.rank),
              s.peer_arrive_flag(region, g.rank, me), s.sent(region, g.rank), g.rank != me,
              use_pat ? g.distinct : -1);
    if (g.rank != me) counters().bytes_sent += static_cast<uint64_t>(g.n) * ub;
    counters().pack_copies++;
  }
}

// The next message from each group's rank: returns the wait index per group
// (in group order) and, when `ack` is set, makes the launch acknowledge the
// messages (sender's free flag) once it is done.
std::vector<int> add_receives(OpHandle& h, Launch& L, const std::vector<DevPlan::Seg>& groups,
                              int region, bool ack) {
  Staging& s = *h.stg;
  const int me = h.sf->comm().rank();
  std::vector<int> bits;
  for (const auto& g : groups) {
    // the next message from g.rank arrived: arrive >= recvd + 1
    bits.push_back(L.add_wait(s.arrive_flag(region, g.rank), s.recvd(region, g.rank), 1));
    if (ack) L.add_done(s.peer_free_flag(region, g.rank, me), s.recvd(region, g.rank), s.done_count);
    counters().bytes_recv += static_cast<uint64_t>(g.n) * h.unit.bytes();
  }
  return bits;
}

// Acknowledge the latest message from each group's rank in launch L.
void add_acks(OpHandle& h, Launch& L, const std::vector<DevPlan::Seg>& groups, int region) {
  Staging& s = *h.stg;
  const int me = h.sf->comm().rank();
  for (const auto& g : groups)
    L.add_done(s.peer_free_flag(region, g.rank, me), s.recvd(region, g.rank), s.done_count);
}

// ----------------------------------------------------- LL128 (p2p) phases
// Slots whose unit is whole 8-byte words use the LL128 protocol (kernels.hpp):
// puts carry a flag in every 128-byte line, receives poll the lines and
// unpack as they land, two messages per channel in flight.
bool use_ll(const OpHandle& h) { return use_p2p(h) && h.stg->ll; }

// LL128 puts of `groups` (each group's pattern over sbuf, or its contiguous
// range of the plain root stage when !use_pat) into the peers' `region`.
void add_puts_ll(OpHandle& h, Launch& L, const std::vector<DevPlan::Seg>& groups, bool use_pat, int sbuf,
                 int region) {
  Staging& s = *h.stg;
  const int me = h.sf->comm().rank();
  const size_t ub = h.unit.bytes();
  for (const auto& g : groups) {
    const PeerSlot& ps = s.peers[static_cast<size_t>(g.rank)];
    char* base = ps.base + (region == 0 ? 0 : region == 1 ? ps.root_at : ps.reply_at);
    const int64_t line = region == 1 ? ps.root_line : ps.leaf_line;
    SFG_REQUIRE(line >= 0, "p2p: peer slot has no group for this rank");
    // message m goes to parity m & 1: the put kernel waits in-line until the
    // peer consumed message m-2 there (its acknowledgement count)
    L.add_put_ll(use_pat ? g.pat : contig(g.stage_off), sbuf, base, line, ps.par[region], g.n,
                 s.free_flag(region, g.rank), s.seg_count(region, g.rank), s.sent(region, g.rank),
                 g.rank != me, use_pat ? g.distinct : -1);
    if (g.rank != me) counters().bytes_sent += static_cast<uint64_t>(g.n) * ub;
    counters().pack_elided++;  // the put gathers straight from the caller's buffer
  }
}

// LL128 receives of the next message of each group from my `region` into
// dpat(group) of dbuf (op, or REPLACE when `replace`); the launch
// acknowledges the messages once all its CTAs are done.
void add_recvs_ll(OpHandle& h, Launch& L, const std::vector<DevPlan::Seg>& groups, int region,
                  const std::function<DPat(const DevPlan::Seg&)>& dpat, int dbuf, bool replace) {
  Staging& s = *h.stg;
  const int me = h.sf->comm().rank();
  const auto& lines = region == 1 ? s.lg_line : s.rg_line;
  for (size_t k = 0; k < groups.size(); ++k) {
    const auto& g = groups[k];
    DSeg sg = pair_seg(contig(0), BUF_LL0 + region, dpat(g), dbuf, g.n, replace);
    sg.type = SEG_RECV_LL;
    sg.run = 0;
    sg.ll_line = lines[k];
    sg.ll_par = s.ll_par[region];
    sg.sig_seq = s.recvd(region, g.rank);
    L.add(sg, 0, -1, g.distinct);
    L.add_done(s.peer_free_flag(region, g.rank, me), s.recvd(region, g.rank), s.done_count);
    L.done_relaxed = true;
    L.interleave = true;
    counters().bytes_recv += static_cast<uint64_t>(g.n) * h.unit.bytes();
    counters().unpack_copies++;
  }
}

bool has_self_group(const OpHandle& h, const std::vector<DevPlan::Seg>& groups) {
  const int me = h.sf->comm().rank();
  return std::any_of(groups.begin(), groups.end(), [me](const DevPlan::Seg& g) { return g.rank == me; });
}

// ---------------------------------------------------------- root -> leaf
void begin_root_to_leaf(OpHandle& h) {
  StarForest& sf = *h.sf;
  DevPlan& d = sf.dev();
  const size_t ub = h.unit.bytes();
  const bool replace = h.op == ReduceOp::replace;
  Launch pack, local;
  set_bufs(pack, h, const_cast<void*>(h.src), h.dst, h.src);
  set_bufs(local, h, const_cast<void*>(h.src), h.dst, h.src);
  if (use_ll(h)) {
    add_puts_ll(h, pack, d.lg, true, BUF_ROOT, 0);
    if (d.has_self)
      local.add(pair_seg(d.self_root, BUF_ROOT, d.self_leaf, BUF_LEAF, d.n_self, replace), 0,
                d.self_root_distinct);
    // The receives join the put launch behind the puts and the local part
    // (leafdata belongs to the operation between Begin and End); a self
    // group (force_remote) receives in End instead.
    h.fused_unpack = false;
    const bool self_group = has_self_group(h, d.rg);
    static const bool no_fuse_ll = std::getenv("SFG_P2P_NO_FUSED_UNPACK") != nullptr;  // ablation
    auto fuse = [&](Launch& L) {
      if (self_group || no_fuse_ll) return;
      add_recvs_ll(h, L, d.rg, 0, [](const DevPlan::Seg& g) { return g.pat; }, BUF_LEAF, replace);
      h.fused_unpack = true;
    };
    p2p_begin(h, pack, local, fuse);
    return;
  }
  if (use_p2p(h)) {
    add_puts(h, pack, d.lg, true, BUF_ROOT, 0);
    if (d.has_self)
      local.add(pair_seg(d.self_root, BUF_ROOT, d.self_leaf, BUF_LEAF, d.n_self, replace), 0,
                d.self_root_distinct);
    // The unpack of the incoming messages joins the put launch, after the
    // puts and the local scatter (their CTAs dispatch first, so spinning
    // unpack CTAs never hold back work they wait on): one launch per
    // exchange. Leafdata belongs to the operation between Begin and End.
    static const bool no_fuse = std::getenv("SFG_P2P_NO_FUSED_UNPACK") != nullptr;
    h.fused_unpack = false;
    // Not when a group is my own rank (force_remote): its unpack CTAs would
    // wait on put CTAs of the same grid.
    const int me = sf.comm().rank();
    const bool self_group =
        std::any_of(d.rg.begin(), d.rg.end(), [me](const DevPlan::Seg& g) { return g.rank == me; });
    auto fuse = [&](Launch& L) {
      const size_t ng = d.rg.size();
      if (no_fuse || ng == 0 || self_group) return;
      const auto bits = add_receives(h, L, d.rg, 0, true);
      for (size_t k = 0; k < ng; ++k) {
        const auto& g = d.rg[k];
        DSeg sg = pair_seg(contig(g.stage_off), BUF_LEAF_STAGE, g.pat, BUF_LEAF, g.n, replace);
        L.add(sg, 0, -1, -1, {bits[k]});
        counters().unpack_copies++;
      }
      h.fused_unpack = true;
    };
    p2p_begin(h, pack, local, fuse);
    return;
  }

  std::vector<XferOp> sends;
  for (const auto& g : d.lg) {
    if (g.contiguous) {
      sends.push_back({g.rank, const_cast<void*>(at(h.src, g.contig_start, ub)), static_cast<size_t>(g.n) * ub});
      counters().pack_elided++;
    } else {
      pack.add(pair_seg(g.pat, BUF_ROOT, contig(g.stage_off), BUF_ROOT_STAGE, g.n, true), 0, g.distinct);
      sends.push_back({g.rank, at(h.stg->root_stage, g.stage_off, ub), static_cast<size_t>(g.n) * ub});
      counters().pack_copies++;
    }
  }
  if (d.has_self)
    local.add(pair_seg(d.self_root, BUF_ROOT, d.self_leaf, BUF_LEAF, d.n_self, replace), 0,
              d.self_root_distinct);

  h.recvs.clear();
  h.zero_copy_recv.clear();
  for (const auto& g : d.rg) {
    const bool zc = g.contiguous && replace;
    h.zero_copy_recv.push_back(zc ? 1 : 0);
    void* ptr = zc ? at(h.dst, g.contig_start, ub) : at(h.stg->leaf_stage, g.stage_off, ub);
    h.recvs.push_back({g.rank, ptr, static_cast<size_t>(g.n) * ub});
    if (zc) counters().unpack_elided++;
  }
  begin_phase(h, pack, local, sends, h.recvs, data_tag(h.opid));
}

void end_root_to_leaf(OpHandle& h) {
  StarForest& sf = *h.sf;
  DevPlan& d = sf.dev();
  const bool replace = h.op == ReduceOp::replace;
  Launch L;
  L.tag = tag_of(h, 1);
  set_bufs(L, h, const_cast<void*>(h.src), h.dst, h.src);
  // Remote leaves are disjoint from the self-edge leaves (each leaf has one
  // root), so the unpack runs on the comm stream right behind the exchange,
  // concurrently with a local scatter still running on the caller's stream;
  // the caller's stream then joins.
  Comm& c = sf.comm();
  if (use_p2p(h) && h.fused_unpack) {
    p2p_join(h);
    return;
  }
  if (use_ll(h)) {
    add_recvs_ll(h, L, d.rg, 0, [](const DevPlan::Seg& g) { return g.pat; }, BUF_LEAF, replace);
    L.run(h.unit, h.op, h.forked ? c.comm_stream() : h.stream);
    p2p_join(h);
    return;
  }
  if (use_p2p(h)) {
    const auto bits = add_receives(h, L, d.rg, 0, true);
    for (size_t k = 0; k < d.rg.size(); ++k) {
      const auto& g = d.rg[k];
      DSeg s = pair_seg(contig(g.stage_off), BUF_LEAF_STAGE, g.pat, BUF_LEAF, g.n, replace);
      L.add(s, 0, -1, -1, {bits[k]});
      counters().unpack_copies++;
    }
    L.run(h.unit, h.op, h.forked ? c.comm_stream() : h.stream);
    p2p_join(h);
    return;
  }
  for (size_t k = 0; k < d.rg.size(); ++k) {
    if (h.zero_copy_recv[k]) continue;
    const auto& g = d.rg[k];
    L.add(pair_seg(contig(g.stage_off), BUF_LEAF_STAGE, g.pat, BUF_LEAF, g.n, replace));
    counters().unpack_copies++;
  }
  if (h.xfer) {
    c.transport().finish(data_tag(h.opid), h.recvs, c.comm_stream());
    L.run(h.unit, h.op, c.comm_stream());
    c.join(h.stream);
  } else {
    L.run(h.unit, h.op, h.stream);
  }
}

// ---------------------------------------------------------- leaf -> root
void begin_leaf_to_root(OpHandle& h) {
  StarForest& sf = *h.sf;
  DevPlan& d = sf.dev();
  const size_t ub = h.unit.bytes();
  const bool replace = h.op == ReduceOp::replace;
  const bool det = sf.comm().config().deterministic;
  Launch pack, local;
  set_bufs(pack, h, h.dst, const_cast<void*>(h.src), h.src);
  set_bufs(local, h, h.dst, const_cast<void*>(h.src), h.src);
  const bool p2p = use_p2p(h);

  std::vector<XferOp> sends;
  const bool ll = use_ll(h);
  if (ll) {
    add_puts_ll(h, pack, d.rg, true, BUF_LEAF, 1);
  } else if (p2p) {
    add_puts(h, pack, d.rg, true, BUF_LEAF, 1);
  } else {
    for (const auto& g : d.rg) {
      if (g.contiguous) {
        sends.push_back({g.rank, const_cast<void*>(at(h.src, g.contig_start, ub)), static_cast<size_t>(g.n) * ub});
        counters().pack_elided++;
      } else {
        pack.add(pair_seg(g.pat, BUF_LEAF, contig(g.stage_off), BUF_LEAF_STAGE, g.n, true));
        sends.push_back({g.rank, at(h.stg->leaf_stage, g.stage_off, ub), static_cast<size_t>(g.n) * ub});
        counters().pack_copies++;
      }
    }
  }
  if (d.has_self) {
    if (replace && d.self_root_dups) counters().replace_dup_collisions++;
    if (replace || !d.self_root_dups) {
      local.add(pair_seg(d.self_leaf, BUF_LEAF, d.self_root, BUF_ROOT, d.n_self, replace), 0, -1,
                d.self_root_distinct);
    } else {
      use_csr(sf);
      local.add(csr_seg(d, CsrRange::self_only, SEG_CSR_FOLD, exact_seq(h, det), h.unit.bytes()), d.csr_self_entries);
    }
  }
  h.coupled_split = split_coupled(sf, h);
  if (h.coupled_split)
    for (auto& it : local.items) it.seg.skip_dst = d.coupled_bits;
  if (ll) {
    // Incoming contributions are copied out of the LL lines into the plain
    // root stage in the put launch (acknowledged there); End folds them.
    // Without self edges and with at most one remote contribution per root
    // (a halo), the order of application is immaterial: the put launch
    // applies them straight to rootdata and End only joins.
    const bool self_group = has_self_group(h, d.lg);
    h.fused_unpack = false;
    h.ll_direct = false;
    const bool direct = !d.has_self && !d.remote_root_dups && !self_group;
    auto fuse = [&](Launch& L) {
      if (self_group) return;
      if (direct)
        add_recvs_ll(h, L, d.lg, 1, [](const DevPlan::Seg& g) { return g.pat; }, BUF_ROOT, replace);
      else
        add_recvs_ll(h, L, d.lg, 1, [](const DevPlan::Seg& g) { return contig(g.stage_off); },
                     BUF_ROOT_STAGE, true);
      h.fused_unpack = true;
      h.ll_direct = direct;
    };
    p2p_begin(h, pack, local, fuse);
    return;
  }
  if (p2p) {
    p2p_begin(h, pack, local);
    return;
  }

  h.recvs.clear();
  h.zero_copy_recv.clear();
  for (const auto& g : d.lg) {
    const bool zc = g.contiguous && replace;
    h.zero_copy_recv.push_back(zc ? 1 : 0);
    void* ptr = zc ? at(h.dst, g.contig_start, ub) : at(h.stg->root_stage, g.stage_off, ub);
    h.recvs.push_back({g.rank, ptr, static_cast<size_t>(g.n) * ub});
    if (zc) counters().unpack_elided++;
  }
  begin_phase(h, pack, local, sends, h.recvs, data_tag(h.opid));
}

void end_leaf_to_root(OpHandle& h) {
  StarForest& sf = *h.sf;
  DevPlan& d = sf.dev();
  const bool replace = h.op == ReduceOp::replace;
  const bool det = sf.comm().config().deterministic;
  Launch L;
  L.tag = tag_of(h, 1);
  set_bufs(L, h, h.dst, const_cast<void*>(h.src), h.src);
  std::vector<int> bits;
  auto wait_k = [&bits](size_t k) { return bits.empty() ? std::vector<int>{} : std::vector<int>{bits[k]}; };
  Comm& c = sf.comm();
  const bool ll = use_ll(h);
  if (ll && h.ll_direct) {  // applied in the put launch
    p2p_join(h);
    return;
  }
  if (ll && !h.fused_unpack) {
    // self group (force_remote): copy the LL messages out here, behind Begin
    Launch R;
    R.tag = tag_of(h, 1);
    set_bufs(R, h, h.dst, const_cast<void*>(h.src), h.src);
    add_recvs_ll(h, R, d.lg, 1, [](const DevPlan::Seg& g) { return contig(g.stage_off); }, BUF_ROOT_STAGE,
                 true);
    R.run(h.unit, ReduceOp::replace, h.forked ? c.comm_stream() : h.stream);
  }
  if (h.coupled_split) {
    // Whole fold of the coupled roots, concurrent with Begin's local part.
    const bool p2p = use_p2p(h);
    if (p2p && !ll) bits = add_receives(h, L, d.lg, 1, true);
    DSeg s = csr_seg(d, CsrRange::remote_only, SEG_CSR_FOLD, exact_seq(h, det), h.unit.bytes());
    s.csr_lo = d.ccsr_lo;
    s.csr_hi = d.ccsr_hi;
    s.csr_ent = d.csr_ent;
    L.add(s, d.ccsr_entries, -1, -1, bits);
    counters().unpack_copies += d.lg.size();
    if (p2p) {
      L.run(h.unit, h.op, h.forked ? c.comm_stream() : h.stream);
      p2p_join(h);
    } else if (h.xfer) {
      c.transport().finish(data_tag(h.opid), h.recvs, c.comm_stream());
      L.run(h.unit, h.op, c.comm_stream());
      c.join(h.stream);
    } else {
      L.run(h.unit, h.op, h.stream);
    }
    return;
  }
  if (use_p2p(h)) {
    p2p_join(h);
    if (!ll) bits = add_receives(h, L, d.lg, 1, true);
  } else {
    end_wait(h, data_tag(h.opid), h.recvs);
  }
  if (!d.lg.empty()) {
    if (replace || !d.remote_root_dups) {
      if (replace && d.remote_root_dups) counters().replace_dup_collisions++;
      for (size_t k = 0; k < d.lg.size(); ++k) {
        if (!h.zero_copy_recv.empty() && h.zero_copy_recv[k]) continue;
        const auto& g = d.lg[k];
        DSeg s = pair_seg(contig(g.stage_off), BUF_ROOT_STAGE, g.pat, BUF_ROOT, g.n, replace);
        L.add(s, 0, -1, g.distinct, wait_k(k));
        counters().unpack_copies++;
      }
    } else {
      // Ascending-rank fold of every remote contribution (ops.cpp:372-376).
      use_csr(sf);
      DSeg s = csr_seg(d, CsrRange::remote_only, SEG_CSR_FOLD, exact_seq(h, det), h.unit.bytes());
      L.add(s, d.csr_remote_entries, -1, -1, bits);
      counters().unpack_copies += d.lg.size();
    }
  }
  L.run(h.unit, h.op, h.stream);
}

// ---------------------------------------------------------- fetch-and-op
void begin_fetch(OpHandle& h) {
  StarForest& sf = *h.sf;
  DevPlan& d = sf.dev();
  const size_t ub = h.unit.bytes();
  Launch pack, local;
  set_bufs(pack, h, h.dst, const_cast<void*>(h.src), h.src);
  if (use_ll(h)) {
    // requests: LL puts + the copy of the incoming ones into the plain root
    // stage (where End fetches in place and the replies start from)
    add_puts_ll(h, pack, d.rg, true, BUF_LEAF, 1);
    h.fused_unpack = false;
    const bool self_group = has_self_group(h, d.lg);
    auto fuse = [&](Launch& L) {
      if (self_group) return;
      add_recvs_ll(h, L, d.lg, 1, [](const DevPlan::Seg& g) { return contig(g.stage_off); },
                   BUF_ROOT_STAGE, true);
      h.fused_unpack = true;
    };
    p2p_begin(h, pack, local, fuse);
    return;
  }
  if (use_p2p(h)) {
    add_puts(h, pack, d.rg, true, BUF_LEAF, 1);
    p2p_begin(h, pack, local);
    return;
  }
  std::vector<XferOp> sends;
  for (const auto& g : d.rg) {
    if (g.contiguous) {
      sends.push_back({g.rank, const_cast<void*>(at(h.src, g.contig_start, ub)), static_cast<size_t>(g.n) * ub});
      counters().pack_elided++;
    } else {
      pack.add(pair_seg(g.pat, BUF_LEAF, contig(g.stage_off), BUF_LEAF_STAGE, g.n, true));
      sends.push_back({g.rank, at(h.stg->leaf_stage, g.stage_off, ub), static_cast<size_t>(g.n) * ub});
      counters().pack_copies++;
    }
  }
  h.recvs.clear();
  for (const auto& g : d.lg)
    h.recvs.push_back({g.rank, at(h.stg->root_stage, g.stage_off, ub), static_cast<size_t>(g.n) * ub});
  begin_phase(h, pack, local, sends, h.recvs, data_tag(h.opid));
}

void end_fetch(OpHandle& h) {
  StarForest& sf = *h.sf;
  DevPlan& d = sf.dev();
  Comm& c = sf.comm();
  const size_t ub = h.unit.bytes();
  const bool det = c.config().deterministic;
  const bool p2p = use_p2p(h);
  Launch L;
  L.tag = "fetch_end";
  set_bufs(L, h, h.dst, const_cast<void*>(h.src), h.src);
  std::vector<int> bits;
  const bool ll = use_ll(h);
  if (ll) {
    if (!h.fused_unpack) {
      Launch R;
      R.tag = "fetch_end";
      set_bufs(R, h, h.dst, const_cast<void*>(h.src), h.src);
      add_recvs_ll(h, R, d.lg, 1, [](const DevPlan::Seg& g) { return contig(g.stage_off); }, BUF_ROOT_STAGE,
                   true);
      R.run(h.unit, ReduceOp::replace, h.forked ? c.comm_stream() : h.stream);
    }
    p2p_join(h);
  } else if (p2p) {
    p2p_join(h);
    // Consumed (acknowledged) only after the replies have been read out of
    // the root stage below.
    bits = add_receives(h, L, d.lg, 1, false);
  } else {
    end_wait(h, data_tag(h.opid), h.recvs);
  }

  // Root side: serialize every contribution per root. Deterministic mode:
  // the reference order (self, then ascending rank). Free-order mode: the
  // groups in the reference's shuffled order (ops.cpp:531-544), a genuinely
  // different serialization per operation.
  use_csr(sf);
  DSeg s = csr_seg(d, CsrRange::all, SEG_CSR_FETCH, exact_seq(h, det), h.unit.bytes());
  L.add(s, d.csr_self_entries + d.csr_remote_entries, -1, -1, bits);
  const int ngroups = (d.has_self ? 1 : 0) + static_cast<int>(d.lg.size());
  if (!det && ngroups > 1 && ngroups <= kMaxShuffle) {
    FetchShuffle& f = L.shuffle;
    f.n = ngroups;
    f.self = d.has_self ? 1 : 0;
    for (size_t k = 0; k < d.lg.size(); ++k) f.off[k] = static_cast<int32_t>(d.lg[k].stage_off);
    f.off[d.lg.size()] = static_cast<int32_t>(d.n_rootside);
    std::vector<int32_t> order(static_cast<size_t>(ngroups));
    for (int g = 0; g < ngroups; ++g) order[static_cast<size_t>(g)] = g;
    SplitMix rng(mix_seed(c.config().seed ^ h.opid, static_cast<uint64_t>(c.rank())));
    rng.shuffle(order);
    for (int g = 0; g < ngroups; ++g) f.perm[g] = order[static_cast<size_t>(g)];
    h.fetch_order.assign(order.begin(), order.end());
  }
  L.run(h.unit, h.op, h.stream);

  // Replies travel back in place (ops.cpp:559-561), then land in leafupdate.
  if (ll) {
    // reply puts from the plain root stage and the receives of my replies
    // into leafupdate, one launch (a self group receives in a second one)
    Launch R;
    R.tag = "fetch_replies";
    set_bufs(R, h, h.dst, const_cast<void*>(h.src), h.src);
    add_puts_ll(h, R, d.lg, false, BUF_ROOT_STAGE, 2);
    auto upd = [](const DevPlan::Seg& g) { return g.pat; };
    const bool self_group = has_self_group(h, d.rg);
    if (!self_group) add_recvs_ll(h, R, d.rg, 2, upd, BUF_LEAFUPDATE, true);
    R.run(h.unit, ReduceOp::replace, h.stream);
    if (self_group) {
      Launch U;
      U.tag = "fetch_end_replies";
      set_bufs(U, h, h.dst, const_cast<void*>(h.src), h.src);
      add_recvs_ll(h, U, d.rg, 2, upd, BUF_LEAFUPDATE, true);
      U.run(h.unit, ReduceOp::replace, h.stream);
    }
    return;
  }
  if (p2p) {
    Launch R;
    R.tag = "fetch_replies";
    set_bufs(R, h, h.dst, const_cast<void*>(h.src), h.src);
    add_puts(h, R, d.lg, false, BUF_ROOT_STAGE, 2);
    add_acks(h, R, d.lg, 1);
    R.run(h.unit, ReduceOp::replace, h.stream);
    Launch U;
    U.tag = "fetch_end_replies";
    set_bufs(U, h, h.dst, const_cast<void*>(h.src), h.src);
    const auto rbits = add_receives(h, U, d.rg, 2, true);
    for (size_t k = 0; k < d.rg.size(); ++k) {
      const auto& g = d.rg[k];
      DSeg s = pair_seg(contig(g.stage_off), BUF_LEAF_REPLY, g.pat, BUF_LEAFUPDATE, g.n, true);
      U.add(s, 0, -1, -1, {rbits[k]});
      counters().unpack_copies++;
    }
    U.run(h.unit, ReduceOp::replace, h.stream);
    return;
  }
  std::vector<XferOp> sends;
  for (const auto& g : d.lg)
    sends.push_back({g.rank, at(h.stg->root_stage, g.stage_off, ub), static_cast<size_t>(g.n) * ub});
  h.reply_recvs.clear();
  h.zero_copy_recv.clear();
  for (const auto& g : d.rg) {
    const bool zc = g.contiguous;
    h.zero_copy_recv.push_back(zc ? 1 : 0);
    void* ptr = zc ? at(h.leafupdate, g.contig_start, ub) : at(h.stg->leaf_reply, g.stage_off, ub);
    h.reply_recvs.push_back({g.rank, ptr, static_cast<size_t>(g.n) * ub});
  }
  if (!sends.empty() || !h.reply_recvs.empty()) {
    cudaStream_t cs = c.comm_stream();
    c.fork(h.stream);
    c.transport().start(reply_tag(h.opid), sends, h.reply_recvs, cs);
    counters().transport_calls++;
    c.transport().finish(reply_tag(h.opid), h.reply_recvs, cs);
    c.join(h.stream);
  }
  Launch U;
  U.tag = "fetch_end_replies";
  set_bufs(U, h, h.dst, const_cast<void*>(h.src), h.src);
  for (size_t k = 0; k < d.rg.size(); ++k) {
    if (h.zero_copy_recv[k]) continue;
    const auto& g = d.rg[k];
    U.add(pair_seg(contig(g.stage_off), BUF_LEAF_REPLY, g.pat, BUF_LEAFUPDATE, g.n, true));
    counters().unpack_copies++;
  }
  U.run(h.unit, ReduceOp::replace, h.stream);
}

void require_ready(StarForest& sf, const Unit& unit, ReduceOp op, const char* what) {
  SFG_REQUIRE(sf.state() == SfState::set_up, std::string(what) + " requires a set-up star forest");
  check_unit_op(unit, op);
}

void require_end(OpHandle& h, OpKind kind, const char* what) {
  SFG_REQUIRE(h.sf != nullptr, std::string(what) + ": handle was never begun");
  SFG_REQUIRE(!h.ended, std::string(what) + ": handle already ended");
  SFG_REQUIRE(h.kind == kind, std::string(what) + ": handle belongs to a different operation");
  h.ended = true;
  h.sf->comm().bind_device();
}

std::unique_ptr<OpHandle> make_handle(StarForest& sf, OpKind kind, const Unit& u, ReduceOp op,
                                      const void* src, void* dst, cudaStream_t s) {
  auto h = std::make_unique<OpHandle>();
  h->sf = &sf;
  h->kind = kind;
  h->unit = u;
  h->op = op;
  h->src = src;
  h->dst = dst;
  h->stream = s;
  return h;
}

}  // namespace

std::unique_ptr<OpHandle> bcast_begin(StarForest& sf, const Unit& u, const void* rootdata,
                                      void* leafdata, ReduceOp op, cudaStream_t s) {
  require_ready(sf, u, op, "bcast");
  auto h = make_handle(sf, OpKind::bcast, u, op, rootdata, leafdata, s);
  begin_common(*h, rootdata, static_cast<size_t>(sf.nroots()) * u.bytes());
  begin_root_to_leaf(*h);
  return h;
}

void bcast_end(OpHandle& h) {
  require_end(h, OpKind::bcast, "bcast_end");
  end_root_to_leaf(h);
  end_common(h);
}

std::unique_ptr<OpHandle> reduce_begin(StarForest& sf, const Unit& u, const void* leafdata,
                                       void* rootdata, ReduceOp op, cudaStream_t s) {
  require_ready(sf, u, op, "reduce");
  auto h = make_handle(sf, OpKind::reduce, u, op, leafdata, rootdata, s);
  begin_common(*h, leafdata, static_cast<size_t>(sf.leaf_index_bound()) * u.bytes());
  begin_leaf_to_root(*h);
  return h;
}

void reduce_end(OpHandle& h) {
  require_end(h, OpKind::reduce, "reduce_end");
  end_leaf_to_root(h);
  end_common(h);
}

std::unique_ptr<OpHandle> fetch_and_op_begin(StarForest& sf, const Unit& u, void* rootdata,
                                             const void* leafdata, void* leafupdate, ReduceOp op,
                                             cudaStream_t s) {
  SFG_REQUIRE(op != ReduceOp::replace, "fetch-and-op with replace has no fetch semantics");
  require_ready(sf, u, op, "fetch_and_op");
  auto h = make_handle(sf, OpKind::fetch_and_op, u, op, leafdata, rootdata, s);
  h->leafupdate = leafupdate;
  begin_common(*h, leafdata, static_cast<size_t>(sf.leaf_index_bound()) * u.bytes());
  begin_fetch(*h);
  return h;
}

void fetch_and_op_end(OpHandle& h) {
  require_end(h, OpKind::fetch_and_op, "fetch_and_op_end");
  end_fetch(h);
  end_common(h);
}

std::unique_ptr<OpHandle> gather_begin(StarForest& sf, const Unit& u, const void* leafdata,
                                       void* multirootdata, cudaStream_t s) {
  require_ready(sf, u, ReduceOp::replace, "gather");
  StarForest& m = sf.multi_sf();
  auto h = make_handle(m, OpKind::gather, u, ReduceOp::replace, leafdata, multirootdata, s);
  begin_common(*h, leafdata, static_cast<size_t>(m.leaf_index_bound()) * u.bytes());
  begin_leaf_to_root(*h);
  return h;
}

void gather_end(OpHandle& h) {
  require_end(h, OpKind::gather, "gather_end");
  end_leaf_to_root(h);
  end_common(h);
}

std::unique_ptr<OpHandle> scatter_begin(StarForest& sf, const Unit& u, const void* multirootdata,
                                        void* leafdata, cudaStream_t s) {
  require_ready(sf, u, ReduceOp::replace, "scatter");
  StarForest& m = sf.multi_sf();
  auto h = make_handle(m, OpKind::scatter, u, ReduceOp::replace, multirootdata, leafdata, s);
  begin_common(*h, multirootdata, static_cast<size_t>(m.nroots()) * u.bytes());
  begin_root_to_leaf(*h);
  return h;
}

void scatter_end(OpHandle& h) {
  require_end(h, OpKind::scatter, "scatter_end");
  end_root_to_leaf(h);
  end_common(h);
}

// One-shot forms (ops.hpp:60-94: Begin + End), stream-ordered: nothing of the
// caller's can be enqueued between the two halves, so the handle is marked
// immediate (see p2p_begin). The blocking forms of the façades add a stream
// synchronisation.
void bcast(StarForest& sf, const Unit& u, const void* rootdata, void* leafdata, ReduceOp op, cudaStream_t s) {
  require_ready(sf, u, op, "bcast");
  auto h = make_handle(sf, OpKind::bcast, u, op, rootdata, leafdata, s);
  h->immediate = true;
  begin_common(*h, rootdata, static_cast<size_t>(sf.nroots()) * u.bytes());
  begin_root_to_leaf(*h);
  bcast_end(*h);
}

void reduce(StarForest& sf, const Unit& u, const void* leafdata, void* rootdata, ReduceOp op, cudaStream_t s) {
  require_ready(sf, u, op, "reduce");
  auto h = make_handle(sf, OpKind::reduce, u, op, leafdata, rootdata, s);
  h->immediate = true;
  begin_common(*h, leafdata, static_cast<size_t>(sf.leaf_index_bound()) * u.bytes());
  begin_leaf_to_root(*h);
  reduce_end(*h);
}

void fetch_and_op(StarForest& sf, const Unit& u, void* rootdata, const void* leafdata, void* leafupdate,
                  ReduceOp op, cudaStream_t s) {
  auto h = fetch_and_op_begin(sf, u, rootdata, leafdata, leafupdate, op, s);
  fetch_and_op_end(*h);
}

void gather(StarForest& sf, const Unit& u, const void* leafdata, void* multirootdata, cudaStream_t s) {
  require_ready(sf, u, ReduceOp::replace, "gather");
  StarForest& m = sf.multi_sf();
  auto h = make_handle(m, OpKind::gather, u, ReduceOp::replace, leafdata, multirootdata, s);
  h->immediate = true;
  begin_common(*h, leafdata, static_cast<size_t>(m.leaf_index_bound()) * u.bytes());
  begin_leaf_to_root(*h);
  gather_end(*h);
}

void scatter(StarForest& sf, const Unit& u, const void* multirootdata, void* leafdata, cudaStream_t s) {
  require_ready(sf, u, ReduceOp::replace, "scatter");
  StarForest& m = sf.multi_sf();
  auto h = make_handle(m, OpKind::scatter, u, ReduceOp::replace, multirootdata, leafdata, s);
  h->immediate = true;
  begin_common(*h, multirootdata, static_cast<size_t>(m.nroots()) * u.bytes());
  begin_root_to_leaf(*h);
  scatter_end(*h);
}

}  // namespace sfg
