// One-sided put/signal data plane over NVLink peer mappings (backend "p2p").
//
// This is the paper's GPU-initiated, sync-free exchange (
// the reference emulates it on host threads with a symmetric heap and
// SendSig/RecvSig flags, /root/reference/proj/src/symheap.cpp:50-295 and
// ops.cpp:160-246,381-476,572-658). On B200 the "symmetric heap" is each
// forest's staging slots, mapped into every neighbor's address space:
//   * process per GPU: cudaIpcGetMemHandle / cudaIpcOpenMemHandle;
//   * threads of one process on distinct GPUs: the raw device pointer plus
//     cudaDeviceEnablePeerAccess.
// The pack kernel waits (in-kernel, per CTA) for the receiver's "free" flag,
// stores straight into the receiver's slot over NVLink, and its last CTA
// raises the receiver's "arrive" flag with a system-scope release. The
// receiver's unpack kernel acquires "arrive", unpacks, and its last CTA
// raises the sender's "free" flag. No host round trip, no stream memory
// operations, two kernel launches per operation when the local part is small.
// Flags are monotonic message counts (Staging), never cleared.
#include <unistd.h>

#include <cstdlib>
#include <cstring>

#include "sfg.hpp"

namespace sfg {
namespace {

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

struct SlotRecord {  // allgathered once per slot
  int32_t pid;
  int32_t device;
  uint64_t ptr;
  uint64_t root_at, reply_at, flags_at;
  int64_t par[3];  // LL128: words per parity buffer of each region
  int32_t ll;
  uint8_t uuid[16];
  cudaIpcMemHandle_t handle;
};

int64_t ll_lines(int64_t n, int64_t wpv) { return (n * wpv + 14) / 15; }

}  // namespace

// Collective over the forest's communicator: every rank creates the same slot
// in the same operation (slots are acquired in collective order).
void StarForest::p2p_attach(Staging& s) {
  DevPlan& d = dev();
  Comm& c = *comm_;
  const int P = c.size();
  const int me = c.rank();
  s.nranks = P;
  // LL128 when the unit is whole 8-byte words (kernels.hpp): each region
  // holds its groups' messages as lines, twice (parity).
  s.ll = s.unit_bytes % 8 == 0 && std::getenv("SFG_P2P_NO_LL128") == nullptr;
  size_t reg_bytes[3] = {s.leaf_bytes, s.root_bytes, s.leaf_bytes};
  if (s.ll) {
    const int64_t wpv = static_cast<int64_t>(s.unit_bytes / 8);
    int64_t lines = 0;
    s.rg_line.clear();
    for (const auto& g : d.rg) {
      s.rg_line.push_back(lines);
      lines += ll_lines(g.n, wpv);
    }
    s.ll_par[0] = s.ll_par[2] = lines * 16;
    lines = 0;
    s.lg_line.clear();
    for (const auto& g : d.lg) {
      s.lg_line.push_back(lines);
      lines += ll_lines(g.n, wpv);
    }
    s.ll_par[1] = lines * 16;
    for (int r = 0; r < 3; ++r) reg_bytes[r] = static_cast<size_t>(2 * s.ll_par[r]) * 8;
    if (s.root_bytes) SFG_CUDA(cudaMalloc(&s.plain_root, s.root_bytes));
  }
  const size_t root_at = align256(reg_bytes[0]);
  const size_t reply_at = root_at + align256(reg_bytes[1]);
  const size_t flags_at = reply_at + align256(reg_bytes[2]);
  const size_t flag_bytes = 12 * static_cast<size_t>(P) * sizeof(unsigned long long) +
                            (3 * static_cast<size_t>(P) + 1) * sizeof(unsigned int);
  const size_t total = flags_at + align256(flag_bytes);
  SFG_CUDA(cudaMalloc(&s.slot_mem, total));
  char* base = static_cast<char*>(s.slot_mem);
  if (s.ll) {
    // LL lines must start zeroed (flag 0 = no message yet)
    SFG_CUDA(cudaMemset(base, 0, flags_at));
    s.ll_region[0] = base;
    s.ll_region[1] = base + root_at;
    s.ll_region[2] = base + reply_at;
    s.leaf_stage = nullptr;
    s.root_stage = s.plain_root;
    s.leaf_reply = nullptr;
  } else {
    s.leaf_stage = s.leaf_bytes ? base : nullptr;
    s.root_stage = s.root_bytes ? base + root_at : nullptr;
    s.leaf_reply = s.leaf_bytes ? base + reply_at : nullptr;
  }
  s.flags = reinterpret_cast<unsigned long long*>(base + flags_at);
  s.seg_counts = reinterpret_cast<unsigned int*>(s.flags + 12 * P);
  s.done_count = s.seg_counts + 3 * P;
  SFG_CUDA(cudaMemset(s.flags, 0, flag_bytes));
  SFG_CUDA(cudaDeviceSynchronize());  // flags are zero before any peer can see them

  SlotRecord mine{};
  mine.pid = static_cast<int32_t>(getpid());
  mine.device = c.device();
  mine.ptr = reinterpret_cast<uint64_t>(base);
  mine.root_at = root_at;
  mine.reply_at = reply_at;
  mine.flags_at = flags_at;
  mine.ll = s.ll ? 1 : 0;
  for (int r = 0; r < 3; ++r) mine.par[r] = s.ll_par[r];
  cudaDeviceProp prop{};
  SFG_CUDA(cudaGetDeviceProperties(&prop, c.device()));
  std::memcpy(mine.uuid, &prop.uuid, sizeof(mine.uuid));
  SFG_CUDA(cudaIpcGetMemHandle(&mine.handle, base));
  std::vector<SlotRecord> all(static_cast<size_t>(P));
  c.ctrl().allgather(&mine, sizeof(mine), all.data());

  // Tell each neighbor where its group sits in my stages (vertex offsets).
  std::vector<std::vector<uint8_t>> send(static_cast<size_t>(P));
  std::vector<int64_t> leaf_off(static_cast<size_t>(P), -1), root_off(static_cast<size_t>(P), -1);
  std::vector<int64_t> leaf_line(static_cast<size_t>(P), -1), root_line(static_cast<size_t>(P), -1);
  for (size_t k = 0; k < d.rg.size(); ++k) {
    leaf_off[static_cast<size_t>(d.rg[k].rank)] = d.rg[k].stage_off;
    if (s.ll) leaf_line[static_cast<size_t>(d.rg[k].rank)] = s.rg_line[k];
  }
  for (size_t k = 0; k < d.lg.size(); ++k) {
    root_off[static_cast<size_t>(d.lg[k].rank)] = d.lg[k].stage_off;
    if (s.ll) root_line[static_cast<size_t>(d.lg[k].rank)] = s.lg_line[k];
  }
  for (int r = 0; r < P; ++r) {
    const int64_t v[4] = {leaf_off[static_cast<size_t>(r)], root_off[static_cast<size_t>(r)],
                          leaf_line[static_cast<size_t>(r)], root_line[static_cast<size_t>(r)]};
    send[static_cast<size_t>(r)].resize(sizeof(v));
    std::memcpy(send[static_cast<size_t>(r)].data(), v, sizeof(v));
  }
  auto got = c.ctrl().alltoallv(std::move(send));

  std::vector<uint8_t> is_nb(static_cast<size_t>(P), 0);
  for (const auto& g : d.rg) is_nb[static_cast<size_t>(g.rank)] = 1;
  for (const auto& g : d.lg) is_nb[static_cast<size_t>(g.rank)] = 1;
  s.peers.assign(static_cast<size_t>(P), PeerSlot{});
  for (int r = 0; r < P; ++r) {
    if (!is_nb[static_cast<size_t>(r)]) continue;
    const SlotRecord& rec = all[static_cast<size_t>(r)];
    PeerSlot& p = s.peers[static_cast<size_t>(r)];
    SFG_REQUIRE(got[static_cast<size_t>(r)].size() == 4 * sizeof(int64_t), "p2p: bad offset exchange");
    SFG_REQUIRE((rec.ll != 0) == s.ll, "p2p: ranks disagree on the LL128 protocol of a staging slot");
    int64_t v[4];
    std::memcpy(v, got[static_cast<size_t>(r)].data(), sizeof(v));
    p.leaf_off = v[0];
    p.root_off = v[1];
    p.leaf_line = v[2];
    p.root_line = v[3];
    for (int q = 0; q < 3; ++q) p.par[q] = rec.par[q];
    p.root_at = rec.root_at;
    p.reply_at = rec.reply_at;
    p.flags_at = rec.flags_at;
    if (r == me) {
      p.base = base;
      continue;
    }
    SFG_REQUIRE(std::memcmp(rec.uuid, mine.uuid, sizeof(mine.uuid)) != 0,
                "p2p backend needs one GPU per rank (ranks " + std::to_string(me) + " and " +
                    std::to_string(r) + " share a device); use the threads or nccl backend");
    int can = 0;
    if (rec.pid == mine.pid) {
      SFG_CUDA(cudaDeviceCanAccessPeer(&can, c.device(), rec.device));
      SFG_REQUIRE(can, "p2p: no peer access between devices " + std::to_string(c.device()) +
                           " and " + std::to_string(rec.device));
      const cudaError_t e = cudaDeviceEnablePeerAccess(rec.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        (void)cudaGetLastError();
      else
        SFG_CUDA(e);
      p.base = reinterpret_cast<char*>(rec.ptr);
    } else {
      void* mapped = nullptr;
      SFG_CUDA(cudaIpcOpenMemHandle(&mapped, rec.handle, cudaIpcMemLazyEnablePeerAccess));
      p.base = static_cast<char*>(mapped);
      p.ipc = true;
    }
  }
  // Every rank's flags are zeroed and mapped before anyone writes into them.
  c.ctrl().barrier();
}

}  // namespace sfg
