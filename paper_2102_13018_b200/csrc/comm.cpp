// Control plane and data-plane transports.
//
// Reference transport: /root/reference/proj/src/comm.cpp (in-process
// mailboxes, buffered isend = payload copy, gather-to-rank-0 allreduce) and
// /root/reference/proj/src/exchange.cpp (dense discovery). Here:
//   * the control plane (SetUp discovery, multi-SF slot exchange) stays on
//     the host: barrier-based slots for in-process ranks, or NCCL collectives
//     over a small device bounce buffer for one-process-per-GPU runs;
//   * the data plane never touches the host: grouped ncclSend/ncclRecv on the
//     caller's stream ("nccl"), or, for ranks that are threads of one process
//     ("threads"), a stream-ordered put protocol — the receiver publishes its
//     buffer plus a ready event, the sender's stream waits on it and copies
//     (peer copy over NVLink when the ranks sit on different GPUs) and
//     publishes an arrival event the receiver's stream waits on. This is the
//     paper's put/signal protocol (emulated on host threads
//     in /root/reference/proj/src/symheap.cpp:100-221) with CUDA events as
//     the signals.
#include <chrono>
#include <cstring>
#include <thread>

#include "sfg.hpp"

namespace sfg {

// -------------------------------------------------------------------- World

World::World(int n, double timeout_s)
    : n_(n), timeout_s_(timeout_s), slots_(static_cast<size_t>(n)),
      mail_(static_cast<size_t>(n), std::vector<std::vector<uint8_t>>(static_cast<size_t>(n))) {
  SFG_REQUIRE(n >= 1, "world needs nranks >= 1");
}

void World::barrier(const char* what) {
  std::unique_lock<std::mutex> lk(mu_);
  const uint64_t gen = generation_;
  if (++arrived_ == n_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
    return;
  }
  const auto deadline = std::chrono::steady_clock::now() +
                        std::chrono::milliseconds(static_cast<long>(timeout_s_ * 1000.0));
  while (generation_ == gen) {
    if (aborted_.load()) throw TimeoutError(std::string(what) + ": run aborted by another rank");
    if (std::chrono::steady_clock::now() >= deadline)
      throw TimeoutError(std::string(what) + ": timed out waiting for peers");
    cv_.wait_for(lk, std::chrono::milliseconds(25));
  }
}

void World::put_slot(int rank, std::vector<uint8_t> data) {
  std::lock_guard<std::mutex> lk(mu_);
  slots_[static_cast<size_t>(rank)] = std::move(data);
}

void World::put_mail(int src, int dst, std::vector<uint8_t> data) {
  std::lock_guard<std::mutex> lk(mu_);
  mail_[static_cast<size_t>(src)][static_cast<size_t>(dst)] = std::move(data);
}

std::vector<uint8_t> World::take_mail(int src, int dst) {
  std::lock_guard<std::mutex> lk(mu_);
  return std::move(mail_[static_cast<size_t>(src)][static_cast<size_t>(dst)]);
}

void World::post(const Key& k, const Post& p) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    SFG_REQUIRE(posts_.find(k) == posts_.end(), "transport: duplicate post (collective mismatch)");
    posts_[k] = p;
  }
  cv_.notify_all();
}

Post World::take(const Key& k, const char* what) {
  std::unique_lock<std::mutex> lk(mu_);
  const auto deadline = std::chrono::steady_clock::now() +
                        std::chrono::milliseconds(static_cast<long>(timeout_s_ * 1000.0));
  for (;;) {
    auto it = posts_.find(k);
    if (it != posts_.end()) {
      Post p = it->second;
      posts_.erase(it);
      return p;
    }
    if (aborted_.load()) throw TimeoutError(std::string(what) + ": run aborted by another rank");
    if (std::chrono::steady_clock::now() >= deadline)
      throw TimeoutError(std::string(what) + ": timed out waiting for rank " +
                         std::to_string(k.src == k.dst ? k.src : (k.kind == 0 ? k.dst : k.src)));
    cv_.wait_for(lk, std::chrono::milliseconds(25));
  }
}

// ------------------------------------------------------------ control planes

namespace {

class ThreadsCtrl final : public ControlPlane {
 public:
  ThreadsCtrl(World* w, int rank) : w_(w), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return w_->size(); }
  void allgather(const void* in, size_t bytes, void* out) override {
    std::vector<uint8_t> mine(bytes);
    if (bytes) std::memcpy(mine.data(), in, bytes);
    w_->put_slot(rank_, std::move(mine));
    w_->barrier("allgather");
    for (int r = 0; r < size(); ++r) {
      const auto& s = w_->slot(r);
      SFG_REQUIRE(s.size() == bytes, "allgather: size mismatch across ranks");
      if (bytes) std::memcpy(static_cast<uint8_t*>(out) + static_cast<size_t>(r) * bytes, s.data(), bytes);
    }
    w_->barrier("allgather");
  }
  std::vector<std::vector<uint8_t>> alltoallv(std::vector<std::vector<uint8_t>> send) override {
    SFG_REQUIRE(static_cast<int>(send.size()) == size(), "alltoallv: need one payload per rank");
    for (int d = 0; d < size(); ++d) w_->put_mail(rank_, d, std::move(send[static_cast<size_t>(d)]));
    w_->barrier("sparse exchange");
    std::vector<std::vector<uint8_t>> out(static_cast<size_t>(size()));
    for (int s = 0; s < size(); ++s) out[static_cast<size_t>(s)] = w_->take_mail(s, rank_);
    w_->barrier("sparse exchange");
    return out;
  }
  void barrier() override { w_->barrier("barrier"); }

 private:
  World* w_;
  int rank_;
};

class SingleCtrl final : public ControlPlane {
 public:
  int rank() const override { return 0; }
  int size() const override { return 1; }
  void allgather(const void* in, size_t bytes, void* out) override {
    if (bytes) std::memcpy(out, in, bytes);
  }
  std::vector<std::vector<uint8_t>> alltoallv(std::vector<std::vector<uint8_t>> send) override {
    return send;
  }
  void barrier() override {}
};

// Control plane over NCCL for one-process-per-GPU runs (SetUp only, so the
// host synchronisation here is by design).
class NcclCtrl final : public ControlPlane {
 public:
  NcclCtrl(ncclComm_t c, int rank, int size, int dev) : c_(c), rank_(rank), size_(size), dev_(dev) {
    SFG_CUDA(cudaSetDevice(dev_));
    SFG_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
  }
  ~NcclCtrl() override {
    if (s_) cudaStreamDestroy(s_);
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void allgather(const void* in, size_t bytes, void* out) override {
    SFG_CUDA(cudaSetDevice(dev_));
    if (bytes == 0) return;
    uint8_t* d = nullptr;
    SFG_CUDA(cudaMalloc(&d, bytes * (static_cast<size_t>(size_) + 1)));
    SFG_CUDA(cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, s_));
    SFG_NCCL(ncclAllGather(d, d + bytes, bytes, ncclUint8, c_, s_));
    SFG_CUDA(cudaMemcpyAsync(out, d + bytes, bytes * static_cast<size_t>(size_),
                             cudaMemcpyDeviceToHost, s_));
    SFG_CUDA(cudaStreamSynchronize(s_));
    SFG_CUDA(cudaFree(d));
  }
  std::vector<std::vector<uint8_t>> alltoallv(std::vector<std::vector<uint8_t>> send) override {
    SFG_CUDA(cudaSetDevice(dev_));
    const size_t n = static_cast<size_t>(size_);
    std::vector<int64_t> mine(n), all(n * n);
    for (size_t d = 0; d < n; ++d) mine[d] = static_cast<int64_t>(send[d].size());
    allgather(mine.data(), n * sizeof(int64_t), all.data());
    size_t stot = 0, rtot = 0;
    for (size_t d = 0; d < n; ++d) stot += send[d].size();
    for (size_t s = 0; s < n; ++s) rtot += static_cast<size_t>(all[s * n + static_cast<size_t>(rank_)]);
    std::vector<std::vector<uint8_t>> out(n);
    uint8_t *ds = nullptr, *dr = nullptr;
    if (stot) SFG_CUDA(cudaMalloc(&ds, stot));
    if (rtot) SFG_CUDA(cudaMalloc(&dr, rtot));
    size_t off = 0;
    std::vector<size_t> soff(n), roff(n);
    for (size_t d = 0; d < n; ++d) {
      soff[d] = off;
      if (!send[d].empty())
        SFG_CUDA(cudaMemcpyAsync(ds + off, send[d].data(), send[d].size(), cudaMemcpyHostToDevice, s_));
      off += send[d].size();
    }
    off = 0;
    for (size_t s = 0; s < n; ++s) {
      roff[s] = off;
      off += static_cast<size_t>(all[s * n + static_cast<size_t>(rank_)]);
    }
    SFG_NCCL(ncclGroupStart());
    for (size_t d = 0; d < n; ++d)
      if (!send[d].empty() && static_cast<int>(d) != rank_)
        SFG_NCCL(ncclSend(ds + soff[d], send[d].size(), ncclUint8, static_cast<int>(d), c_, s_));
    for (size_t s = 0; s < n; ++s) {
      const size_t b = static_cast<size_t>(all[s * n + static_cast<size_t>(rank_)]);
      if (b && static_cast<int>(s) != rank_)
        SFG_NCCL(ncclRecv(dr + roff[s], b, ncclUint8, static_cast<int>(s), c_, s_));
    }
    SFG_NCCL(ncclGroupEnd());
    for (size_t s = 0; s < n; ++s) {
      const size_t b = static_cast<size_t>(all[s * n + static_cast<size_t>(rank_)]);
      if (static_cast<int>(s) == rank_) {
        out[s] = std::move(send[s]);
      } else {
        out[s].resize(b);
        if (b) SFG_CUDA(cudaMemcpyAsync(out[s].data(), dr + roff[s], b, cudaMemcpyDeviceToHost, s_));
      }
    }
    SFG_CUDA(cudaStreamSynchronize(s_));
    if (ds) cudaFree(ds);
    if (dr) cudaFree(dr);
    return out;
  }
  bool alltoallv_device(const uint8_t* send, const std::vector<int64_t>& soff,
                        const std::vector<int64_t>& sbytes, uint8_t* recv, const std::vector<int64_t>& roff,
                        const std::vector<int64_t>& rbytes) override {
    SFG_CUDA(cudaSetDevice(dev_));
    SFG_CUDA(cudaStreamSynchronize(cudaStreamPerThread));  // payload written on the caller's stream
    SFG_NCCL(ncclGroupStart());
    for (int r = 0; r < size_; ++r) {
      if (r == rank_) continue;
      const size_t i = static_cast<size_t>(r);
      if (sbytes[i]) SFG_NCCL(ncclSend(send + soff[i], static_cast<size_t>(sbytes[i]), ncclUint8, r, c_, s_));
      if (rbytes[i]) SFG_NCCL(ncclRecv(recv + roff[i], static_cast<size_t>(rbytes[i]), ncclUint8, r, c_, s_));
    }
    SFG_NCCL(ncclGroupEnd());
    SFG_CUDA(cudaStreamSynchronize(s_));
    return true;
  }
  void barrier() override {
    uint8_t one = 1;
    std::vector<uint8_t> all(static_cast<size_t>(size_));
    allgather(&one, 1, all.data());
  }

 private:
  ncclComm_t c_;
  int rank_, size_, dev_;
  cudaStream_t s_ = nullptr;
};

// ------------------------------------------------------------- transports

constexpr int kReady = 0;
constexpr int kArrived = 1;

class ThreadsTransport final : public Transport {
 public:
  ThreadsTransport(World* w, int me, int dev) : w_(w), me_(me), dev_(dev) {}
  const char* name() const override { return "threads"; }

  void start(uint64_t tag, const std::vector<XferOp>& sends, const std::vector<XferOp>& recvs,
             cudaStream_t stream) override {
    // Publish every receive buffer first (never blocks), then serve sends.
    for (const auto& r : recvs) {
      Post p{r.ptr, r.bytes, nullptr, dev_};
      SFG_CUDA(cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
      SFG_CUDA(cudaEventRecord(p.ev, stream));
      w_->post(World::Key{tag, r.peer, me_, kReady}, p);
    }
    for (const auto& s : sends) {
      Post dst = w_->take(World::Key{tag, me_, s.peer, kReady}, "transport send");
      if (dst.bytes != s.bytes) {
        cudaEventDestroy(dst.ev);
        fail("transport: message size mismatch (sent " + std::to_string(s.bytes) +
             " bytes, receive posted for " + std::to_string(dst.bytes) + ")");
      }
      SFG_CUDA(cudaStreamWaitEvent(stream, dst.ev, 0));
      SFG_CUDA(cudaEventDestroy(dst.ev));
      if (s.bytes) {
        if (dst.device == dev_)
          SFG_CUDA(cudaMemcpyAsync(dst.ptr, s.ptr, s.bytes, cudaMemcpyDeviceToDevice, stream));
        else
          SFG_CUDA(cudaMemcpyPeerAsync(dst.ptr, dst.device, s.ptr, dev_, s.bytes, stream));
      }
      Post arrived{dst.ptr, s.bytes, nullptr, dev_};
      SFG_CUDA(cudaEventCreateWithFlags(&arrived.ev, cudaEventDisableTiming));
      SFG_CUDA(cudaEventRecord(arrived.ev, stream));
      w_->post(World::Key{tag, me_, s.peer, kArrived}, arrived);
      counters().bytes_sent += s.bytes;
    }
  }

  void finish(uint64_t tag, const std::vector<XferOp>& recvs, cudaStream_t stream) override {
    for (const auto& r : recvs) {
      Post p = w_->take(World::Key{tag, r.peer, me_, kArrived}, "transport receive");
      SFG_CUDA(cudaStreamWaitEvent(stream, p.ev, 0));
      SFG_CUDA(cudaEventDestroy(p.ev));
      counters().bytes_recv += r.bytes;
    }
  }

 private:
  World* w_;
  int me_, dev_;
};

class NcclTransport final : public Transport {
 public:
  NcclTransport(ncclComm_t c, int me, int dev) : c_(c), me_(me), dev_(dev) { (void)dev_; }
  const char* name() const override { return "nccl"; }

  void start(uint64_t, const std::vector<XferOp>& sends, const std::vector<XferOp>& recvs,
             cudaStream_t stream) override {
    std::vector<const XferOp*> self_sends, self_recvs;
    bool any = false;
    for (const auto& s : sends) (s.peer == me_ ? self_sends.push_back(&s) : (void)(any = true));
    for (const auto& r : recvs) (r.peer == me_ ? self_recvs.push_back(&r) : (void)(any = true));
    SFG_REQUIRE(self_sends.size() == self_recvs.size(), "transport: unmatched self message");
    for (size_t i = 0; i < self_sends.size(); ++i) {
      SFG_REQUIRE(self_sends[i]->bytes == self_recvs[i]->bytes, "transport: message size mismatch");
      if (self_sends[i]->bytes)
        SFG_CUDA(cudaMemcpyAsync(self_recvs[i]->ptr, self_sends[i]->ptr, self_sends[i]->bytes,
                                 cudaMemcpyDeviceToDevice, stream));
    }
    if (!any) return;
    SFG_NCCL(ncclGroupStart());
    for (const auto& s : sends)
      if (s.peer != me_) {
        SFG_NCCL(ncclSend(s.ptr, s.bytes, ncclUint8, s.peer, c_, stream));
        counters().bytes_sent += s.bytes;
      }
    for (const auto& r : recvs)
      if (r.peer != me_) {
        SFG_NCCL(ncclRecv(r.ptr, r.bytes, ncclUint8, r.peer, c_, stream));
        counters().bytes_recv += r.bytes;
      }
    SFG_NCCL(ncclGroupEnd());
  }

  // NCCL receives complete in stream order; nothing to do.
  void finish(uint64_t, const std::vector<XferOp>&, cudaStream_t) override {}

 private:
  ncclComm_t c_;
  int me_, dev_;
};

}  // namespace

std::unique_ptr<ControlPlane> make_threads_ctrl(World* w, int rank) {
  return std::make_unique<ThreadsCtrl>(w, rank);
}
std::unique_ptr<ControlPlane> make_single_ctrl() { return std::make_unique<SingleCtrl>(); }
std::unique_ptr<ControlPlane> make_nccl_ctrl(ncclComm_t c, int rank, int size, int dev) {
  return std::make_unique<NcclCtrl>(c, rank, size, dev);
}
std::unique_ptr<Transport> make_threads_transport(World* w, int rank, int dev, double) {
  return std::make_unique<ThreadsTransport>(w, rank, dev);
}
std::unique_ptr<Transport> make_nccl_transport(ncclComm_t c, int rank, int dev) {
  return std::make_unique<NcclTransport>(c, rank, dev);
}

// --------------------------------------------------------------------- Comm

Comm::Comm(int nranks, int rank, int device, CommConfig cfg)
    : size_(nranks), rank_(rank), device_(device), cfg_(std::move(cfg)) {
  SFG_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "comm: rank outside communicator");
}

Comm::~Comm() {
  if (device_ >= 0) cudaSetDevice(device_);
  if (cstream_) cudaStreamSynchronize(cstream_);
  transport_.reset();
  ctrl_.reset();
  if (nccl_) ncclCommDestroy(nccl_);
  if (fork_ev_) cudaEventDestroy(fork_ev_);
  if (join_ev_) cudaEventDestroy(join_ev_);
  if (cstream_) cudaStreamDestroy(cstream_);
}

cudaStream_t Comm::comm_stream() {
  if (!cstream_) {
    bind_device();
    int lo = 0, hi = 0;
    SFG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // Highest priority: the exchange should not queue behind a long local scatter.
    SFG_CUDA(cudaStreamCreateWithPriority(&cstream_, cudaStreamNonBlocking, hi));
    SFG_CUDA(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming));
    SFG_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
  }
  return cstream_;
}

void Comm::fork(cudaStream_t user) {
  cudaStream_t cs = comm_stream();
  SFG_CUDA(cudaEventRecord(fork_ev_, user));
  SFG_CUDA(cudaStreamWaitEvent(cs, fork_ev_, 0));
}

void Comm::join(cudaStream_t user) {
  cudaStream_t cs = comm_stream();
  SFG_CUDA(cudaEventRecord(join_ev_, cs));
  SFG_CUDA(cudaStreamWaitEvent(user, join_ev_, 0));
}

Transport& Comm::transport() {
  SFG_REQUIRE(transport_ != nullptr, "communicator has no data-plane transport (no device bound)");
  return *transport_;
}

void Comm::bind_device() const {
  SFG_REQUIRE(device_ >= 0, "operation needs a CUDA device; communicator was created host-only");
  SFG_CUDA(cudaSetDevice(device_));
}

}  // namespace sfg
