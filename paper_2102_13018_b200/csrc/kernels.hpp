// Device-side plan descriptors and the launch interface shared by the host
// engine (ops.cpp) and the sm_100a kernels (kernels.cu).
//
// Every data movement the star-forest engine performs is a list of
// "segments" executed by ONE kernel launch:
//   SEG_PAIR         dst[dpat(i)] (op)= src[spat(i)]  (pack, unpack, local
//                    scatter; the reference's pack/unpack/scatter loops,
//                    /root/reference/proj/src/pack.cpp:111-256)
//   SEG_CSR_FOLD     root-sorted fold: root[r] = fold(root[r], contributions
//                    in the reference's deterministic order) — bit-exact with
//                    /root/reference/proj/src/ops.cpp:364,367-376
//   SEG_CSR_FETCH    serialized fetch-and-op over the same CSR
//                    (/root/reference/proj/src/ops.cpp:521-563)
// Patterns are Contiguous, Affine3D (start + x + y*s1 + z*s2) or Indexed.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sfg {

enum PatKind : uint32_t { PAT_CONTIG = 0, PAT_AFFINE = 1, PAT_INDEXED = 2 };

// Unsigned 32-bit division by a run-time constant (round-up multiplier).
// Valid for numerators < 2^31, which holds for every per-rank position.
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d == 0 ? 1 : d;
  uint32_t l = 0;
  while ((uint64_t(1) << l) < f.d) ++l;
  f.s = l;
  // m = floor(2^32 * (2^l - d) / d) + 1
  f.m = static_cast<uint32_t>(((uint64_t(1) << 32) * ((uint64_t(1) << l) - f.d)) / f.d + 1);
  return f;
}

struct DPat {
  int64_t start = 0;  // contiguous / affine base (vertex index)
  int64_t s1 = 0;     // affine row stride (vertices)
  int64_t s2 = 0;     // affine plane stride (vertices)
  const int32_t* idx = nullptr;  // indexed
  uint32_t kind = PAT_CONTIG;
  uint32_t pad = 0;
  FastDiv dx;  // affine row length
  FastDiv dy;  // affine rows per plane
};

enum SegType : int32_t {
  SEG_PAIR = 0,
  SEG_CSR_FOLD = 2,
  SEG_CSR_FETCH = 3,
  SEG_PUT_LL = 4,   // p2p: src pattern -> peer's LL128 region (lines + flag)
  SEG_RECV_LL = 5,  // p2p: my LL128 region -> dst pattern (op), polling lines
};

// LL128 messages (p2p backend, units that are a multiple of 8 bytes): a
// message of W 8-byte words travels as ceil(W/15) 128-byte lines; words
// 0..14 of a line carry data, word 15 the message number m. A warp writes a
// line with ONE 16-byte store per lane (8 lanes per line), which NVLink
// delivers as one transaction, so a receiver that sees the flag m in a line
// sees the whole line: no fence, no completion flag, and the unpack of a
// line starts as soon as it lands (NCCL's LL128 protocol). Each receive
// region holds two messages per channel (parity m & 1), so a put waits only
// for the acknowledgement of message m-2, which is long done.
constexpr int kLLIters = 4;                  // line groups per warp
constexpr int kLLLines = 8 * 4 * kLLIters;  // lines per CTA (256 threads)
constexpr int64_t kLLWideLines = 65536;    // launches moving more lines run at 3 CTAs/SM

// Buffer slots a segment can address; filled per call.
enum BufId : int32_t {
  BUF_ROOT = 0,        // user rootdata (or multiroot data)
  BUF_LEAF = 1,        // user leafdata
  BUF_LEAF_STAGE = 2,  // leaf-side staging (remote root groups, wire order)
  BUF_ROOT_STAGE = 3,  // root-side staging (remote leaf groups, wire order)
  BUF_LEAFUPDATE = 4,  // fetch-and-op leafupdate
  BUF_LEAF_REPLY = 5,  // fetch-and-op reply staging on the leaf side
  BUF_SRC_RO = 6,      // read-only source alias (leafdata for reduce/fetch)
  BUF_LL0 = 7,         // p2p LL128: my receive regions 0 (leaf), 1 (root), 2 (reply)
  BUF_PEER0 = 10,      // p2p transport: a put's peer region is BUF_PEER0 + k
  BUF_COUNT = 10 + 16
};
constexpr int kMaxPeers = BUF_COUNT - BUF_PEER0;

struct DSeg {
  DPat src;
  DPat dst;
  int64_t n = 0;  // positions (pair) or CSR roots (csr)
  // Pair segments whose two patterns are both contiguous/affine: positions
  // come in runs of `run` that are contiguous on both sides (gcd of the row
  // lengths). 0 = per-element index evaluation.
  int64_t run = 0;
  FastDiv rundiv;
  int32_t type = SEG_PAIR;
  int32_t replace = 0;  // 1: this segment moves data verbatim (pack)
  int32_t src_buf = 0;
  int32_t dst_buf = 0;
  int32_t aux_buf = 0;   // fetch: where fetched values go (same pattern as src)
  int32_t stage_buf = 0; // csr: buffer of remote entries (entry < 0)
  // CSR over distinct roots: roots[r], contributions ent[lo[r] .. hi[r])
  // entry >= 0: self leaf index into src_buf; entry < 0: staging position -e-1
  const int32_t* csr_roots = nullptr;
  const int32_t* csr_lo = nullptr;
  const int32_t* csr_hi = nullptr;
  const int32_t* csr_ent = nullptr;
  // CSR execution: 0 = one thread per root item, 1 = one warp per root item
  // (high degree). csr_seq = 1 forces the exact sequential fold order (float
  // data in deterministic mode); otherwise integer/associative ops combine
  // with a warp tree/scan, which is bit-identical for them.
  int32_t csr_warp = 0;
  int32_t csr_seq = 1;
  // L2-tiled CSR: csr_np > 1 pieces, walked piece-major by a resident grid
  // of csr_grid_threads threads (set at launch). Piece q of root r spans
  // entries [b(q), b(q+1)) with b(0) = csr_lo[r], b(np) = csr_hi[r] and
  // b(q) = csr_ptab[r * csr_pt_stride + q * csr_pt_step - 1] in between.
  int32_t csr_np = 1;
  int32_t csr_pt_stride = 0;
  int32_t csr_pt_step = 1;
  const int32_t* csr_ptab = nullptr;
  int64_t csr_grid_threads = 0;
  // One-sided put/signal (p2p backend, the paper's put + signal,
  // PAPER.md:904-922). Before touching data, every CTA of the segment waits
  // until each flag of LaunchParams::waits selected by wait_mask reaches its
  // target (a peer's "slot free" for puts, a peer's "data arrived" for
  // unpacks). After its last CTA has stored its part (stores into a peer's
  // mapped slot over NVLink), the segment advances its message counter
  // *sig_seq and publishes the new count in *sig_flag with a system-scope
  // release; sig_count is a local CTA arrival counter the last CTA resets.
  // Counters live in device memory, so a captured CUDA graph replays the
  // protocol correctly.
  uint32_t wait_mask = 0;
  // Reductions: destination roots whose bit is set are left alone (their
  // whole fold runs in another launch, see DevPlan::coupled_bits).
  const uint32_t* skip_dst = nullptr;
  unsigned int* sig_count = nullptr;
  unsigned long long* sig_flag = nullptr;
  unsigned long long* sig_seq = nullptr;
  // LL128 segments: the group's first line in the region and the words per
  // parity buffer of the region; sig_seq is the channel's message counter
  // (sent for puts, recvd for receives: message m = *sig_seq + 1).
  int64_t ll_line = 0;
  int64_t ll_par = 0;
  // LL128 put: the peer's acknowledgement count for this channel; message m
  // may overwrite parity m & 1 once it reaches m - 2.
  const unsigned long long* ll_credit = nullptr;
  // LL128 put: consecutive kLLLines chunks each CTA writes (launch_segments)
  int64_t ll_loop = 1;
};

// Wait until *flag >= *count + delta (count: a local message counter).
struct FlagWait {
  const unsigned long long* flag = nullptr;
  const unsigned long long* count = nullptr;
  long long delta = 0;  // wait for *flag >= *count + delta (nothing when <= 0)
};

constexpr int kMaxSegs = 12;
constexpr int kThreads = 256;
constexpr int kItems = 8;  // work items per thread per block
constexpr int kMaxShuffle = 16;

// Free-order fetch-and-op serialization (/root/reference/proj/src/ops.cpp:
// 531-544): the reference shuffles the order in which the contribution
// groups (self edges, then one group per remote rank) are applied, with
// Rng(mix_seed(seed ^ opid, rank)). Each root's CSR entries are stored group
// by group (self entries >= 0 first, then remote stage positions ascending),
// so the kernel walks the groups' sub-ranges in `perm` order.
struct FetchShuffle {
  int32_t n = 0;     // groups (0 or 1: stored order)
  int32_t self = 0;  // group 0 holds the self edges
  int32_t perm[kMaxShuffle] = {};
  int32_t off[kMaxShuffle + 1] = {};  // stage offset where remote group k starts (+ end)
};

struct LaunchParams {
  DSeg seg[kMaxSegs];
  int64_t block_start[kMaxSegs + 1];  // prefix of blocks per segment
  void* bufs[BUF_COUNT];
  int64_t bl = 1;  // elements per vertex
  FastDiv bldiv;
  int64_t wpv = 1;  // LL128: 8-byte words per vertex (unit bytes / 8)
  int nseg = 0;
  // p2p: flags segments wait on (bit i of DSeg::wait_mask = waits[i]) and the
  // acknowledgements the launch raises once all its CTAs are done (advance
  // the local counter *done_seq[i], publish it in a peer's "slot free" flag
  // done_flag[i]); done_count is a local CTA arrival counter.
  FlagWait waits[kMaxPeers];
  unsigned long long* done_flag[kMaxPeers];
  unsigned long long* done_seq[kMaxPeers];
  int ndone = 0;
  int done_relaxed = 0;  // LL128 channels: acknowledge with a relaxed store
  int ll_poll_ns = 20;   // LL128 receive: back-off between polls of unarrived lines
  // LL128 launches: CTAs of the receive segments (the trailing ones) are
  // dispatched interleaved with the put / local CTAs instead of after them,
  // so large messages are unpacked while they stream in. ilv_a = number of
  // blocks before the first receive segment (0 = off); launch_segments sets
  // it when requested with -1.
  int64_t ilv_a = 0;
  // Debug (SFG_TRACE_LAUNCHES): 8 words of %globaltimer marks for this
  // launch (see kernels.cu trace_mark), nullptr otherwise.
  unsigned long long* trace = nullptr;
  unsigned int* done_count = nullptr;
  FetchShuffle shuf;
};

// SFG_TRACE_LAUNCHES=N: per-launch timestamps of the first N launches of the
// process (put / receive CTA start and end, data ready, launch end), dumped by
// sfg_trace_dump. Debug only.
void trace_init();                 // allocate the buffer (outside any capture)
unsigned long long* trace_slot();  // nullptr when tracing is off or full
void trace_dump(const char* path);

// Element type the kernel instantiates for.
enum class ElemType : int32_t { u8, u16, u32, u64, i32, i64, f64 };

// Returns number of kernel launches issued (0 or 1 per call).
int launch_segments(LaunchParams& p, ElemType t, int op, cudaStream_t stream);

// p2p: ++*seq[i] and publish it in flag[i] (system-scope release) for n
// channels, after everything earlier on the stream (acknowledgements that do
// not fit one launch's parameter block).
void launch_signal(unsigned long long* const* flag, unsigned long long* const* seq, int n, cudaStream_t s);

// p2p teardown: wait until every message this slot sent was acknowledged
// (flag[i] >= *count[i]), so no peer still writes into the slot when it is
// freed. Gives up with a warning after timeout_s (a dead peer). Any n.
void launch_quiesce(const unsigned long long* const* flag, const unsigned long long* const* count, int n,
                    double timeout_s, cudaStream_t s);

// Order-independent 64-bit digest of a device buffer (debug checksum).
void launch_digest(const void* p, size_t bytes, unsigned long long* out_dev, cudaStream_t s);

}  // namespace sfg
