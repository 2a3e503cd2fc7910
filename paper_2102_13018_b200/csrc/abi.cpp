// extern "C" boundary (include/sfgpu.h). Converts C++ exceptions to status
// codes + a thread-local message, the C rendering of sf::Error.
#include "../../include/sfgpu.h"

#include <cstring>
#include <string>

#include "sfg.hpp"

struct sfg_world_s {
  sfg::World w;
  sfg_world_s(int n, double t) : w(n, t) {}
};
struct sfg_comm_s {
  std::unique_ptr<sfg::World> own_world;
  std::unique_ptr<sfg::Comm> c;
};
struct sfg_sf_s {};      // alias of sfg::StarForest
struct sfg_mat_s {};     // alias of sfg::DevMatrix
struct sfg_handle_s {};  // alias of sfg::OpHandle

namespace {

thread_local std::string g_err;

int fail_code(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return SFG_OK;
  } catch (const sfg::TimeoutError& e) {
    return fail_code(e, SFG_ERR_TIMEOUT);
  } catch (const sfg::CudaError& e) {
    return fail_code(e, SFG_ERR_CUDA);
  } catch (const std::exception& e) {
    return fail_code(e, SFG_ERR);
  }
}

sfg::StarForest* SF(sfg_sf s) {
  SFG_REQUIRE(s != nullptr, "null star forest");
  return reinterpret_cast<sfg::StarForest*>(s);
}
sfg::OpHandle* H(sfg_handle h) {
  SFG_REQUIRE(h != nullptr, "null operation handle");
  return reinterpret_cast<sfg::OpHandle*>(h);
}
sfg_handle out_h(std::unique_ptr<sfg::OpHandle> h) {
  return reinterpret_cast<sfg_handle>(h.release());
}
sfg::Unit unit(int kind, int64_t blocklen) {
  SFG_REQUIRE(kind >= 0 && kind <= 3, "unknown unit kind");
  return sfg::Unit{static_cast<sfg::Kind>(kind), blocklen};
}
sfg::ReduceOp rop(int op) {
  SFG_REQUIRE(op >= 0 && op <= 8, "unknown reduction");
  return static_cast<sfg::ReduceOp>(op);
}
cudaStream_t st(void* s) { return static_cast<cudaStream_t>(s); }

void fill_pattern(const sfg::Pattern& p, sfg_pattern* o) {
  o->kind = static_cast<int>(p.kind);
  o->has_duplicates = p.has_duplicates ? 1 : 0;
  o->count = p.count;
  o->start = p.start;
  o->dx = p.dx;
  o->dy = p.dy;
  o->dz = p.dz;
  o->s1 = p.s1;
  o->s2 = p.s2;
  o->bound = p.bound;
}

}  // namespace

extern "C" {

const char* sfg_last_error(void) { return g_err.c_str(); }
int sfg_version(void) { return SFGPU_VERSION; }

void sfg_config_default(sfg_config* cfg) {
  sfg::CommConfig c;
  cfg->deterministic = c.deterministic ? 1 : 0;
  cfg->debug_checksum = c.debug_checksum ? 1 : 0;
  cfg->force_remote = c.force_remote ? 1 : 0;
  cfg->dense_discovery_threshold = c.dense_discovery_threshold;
  cfg->seed = c.seed;
  cfg->timeout_s = c.timeout_s;
}

int sfg_world_create(int nranks, double timeout_s, sfg_world* out) {
  return guard([&] { *out = new sfg_world_s(nranks, timeout_s); });
}
int sfg_world_abort(sfg_world w) {
  return guard([&] { w->w.abort(); });
}
int sfg_world_destroy(sfg_world w) {
  return guard([&] { delete w; });
}

int sfg_nccl_unique_id(void* out, size_t bytes) {
  return guard([&] {
    SFG_REQUIRE(bytes >= sizeof(ncclUniqueId), "unique id buffer too small");
    ncclUniqueId id;
    SFG_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

}  // extern "C"

namespace {

// Control plane over caller-supplied callbacks (torch.distributed, MPI, ...).
class ExtCtrl final : public sfg::ControlPlane {
 public:
  ExtCtrl(const sfg_ctrl_ops& ops, int rank, int size) : ops_(ops), rank_(rank), size_(size) {}
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void allgather(const void* in, size_t bytes, void* out) override {
    SFG_REQUIRE(ops_.allgather(ops_.ctx, in, bytes, out) == 0, "control plane: allgather failed");
  }
  std::vector<std::vector<uint8_t>> alltoallv(std::vector<std::vector<uint8_t>> send) override {
    const size_t n = static_cast<size_t>(size_);
    std::vector<int64_t> mine(n), all(n * n), rb(n);
    for (size_t d = 0; d < n; ++d) mine[d] = static_cast<int64_t>(send[d].size());
    allgather(mine.data(), n * sizeof(int64_t), all.data());
    size_t stot = 0, rtot = 0;
    for (size_t d = 0; d < n; ++d) stot += send[d].size();
    for (size_t s = 0; s < n; ++s) {
      rb[s] = all[s * n + static_cast<size_t>(rank_)];
      rtot += static_cast<size_t>(rb[s]);
    }
    std::vector<uint8_t> sbuf(stot), rbuf(rtot);
    size_t off = 0;
    for (size_t d = 0; d < n; ++d) {
      if (!send[d].empty()) std::memcpy(sbuf.data() + off, send[d].data(), send[d].size());
      off += send[d].size();
    }
    SFG_REQUIRE(ops_.alltoallv(ops_.ctx, sbuf.data(), mine.data(), rbuf.data(), rb.data()) == 0,
                "control plane: alltoallv failed");
    std::vector<std::vector<uint8_t>> out(n);
    off = 0;
    for (size_t s = 0; s < n; ++s) {
      out[s].assign(rbuf.begin() + static_cast<std::ptrdiff_t>(off),
                    rbuf.begin() + static_cast<std::ptrdiff_t>(off + static_cast<size_t>(rb[s])));
      off += static_cast<size_t>(rb[s]);
    }
    return out;
  }
  void barrier() override {
    SFG_REQUIRE(ops_.barrier(ops_.ctx) == 0, "control plane: barrier failed");
  }

 private:
  sfg_ctrl_ops ops_;
  int rank_, size_;
};

sfg::CommConfig to_config(const sfg_config* cfg, const char* backend) {
  sfg::CommConfig cc;
  if (cfg) {
    cc.deterministic = cfg->deterministic != 0;
    cc.debug_checksum = cfg->debug_checksum != 0;
    cc.force_remote = cfg->force_remote != 0;
    cc.dense_discovery_threshold = cfg->dense_discovery_threshold;
    cc.seed = cfg->seed;
    cc.timeout_s = cfg->timeout_s;
  }
  cc.backend = backend ? backend : "threads";
  SFG_REQUIRE(cc.backend == "threads" || cc.backend == "nccl" || cc.backend == "p2p",
              "unknown transport backend '" + cc.backend + "' (threads | nccl | p2p)");
  return cc;
}

sfg_comm make_comm(sfg_world world, int nranks, int rank, int device, const sfg::CommConfig& cc,
                   const void* nccl_id, const sfg_ctrl_ops* ops) {
  auto h = std::make_unique<sfg_comm_s>();
  h->c = std::make_unique<sfg::Comm>(nranks, rank, device, cc);
  sfg::Comm& c = *h->c;
  sfg::World* w = world ? &world->w : nullptr;
  if (w) SFG_REQUIRE(w->size() == nranks, "world size does not match nranks");
  if (!w && cc.backend == "threads" && device >= 0) {
    SFG_REQUIRE(nranks == 1, "the threads backend needs an in-process world for nranks > 1");
    h->own_world = std::make_unique<sfg::World>(1, cc.timeout_s);
    w = h->own_world.get();
  }
  c.world_ = w;
  if (device >= 0) {
    SFG_CUDA(cudaSetDevice(device));
    SFG_CUDA(cudaFree(nullptr));  // create the context
    sfg::trace_init();
  }
  if (cc.backend == "p2p") SFG_REQUIRE(device >= 0, "the p2p backend needs a device");
  // p2p: NCCL only carries the control plane (SetUp, slot mapping) when the
  // ranks are processes without caller-supplied callbacks.
  if (cc.backend == "nccl" || (cc.backend == "p2p" && !w && !ops && nranks > 1)) {
    SFG_REQUIRE(device >= 0, "the nccl backend needs a device");
    ncclUniqueId id;
    if (nccl_id) {
      std::memcpy(&id, nccl_id, sizeof(id));
    } else {
      SFG_REQUIRE(nranks == 1, "nccl backend with nranks > 1 needs a shared unique id");
      SFG_NCCL(ncclGetUniqueId(&id));
    }
    SFG_NCCL(ncclCommInitRank(&c.nccl_, nranks, id, rank));
  }
  if (ops)
    c.ctrl_ = std::make_unique<ExtCtrl>(*ops, rank, nranks);
  else if (w)
    c.ctrl_ = sfg::make_threads_ctrl(w, rank);
  else if (nranks == 1)
    c.ctrl_ = sfg::make_single_ctrl();
  else {
    SFG_REQUIRE(c.nccl_ != nullptr, "nranks > 1 without a world needs the nccl backend or control-plane callbacks");
    c.ctrl_ = sfg::make_nccl_ctrl(c.nccl_, rank, nranks, device);
    // NCCL connects each peer pair on its first send/recv (~3 s on B200 for
    // the first exchange): connect every pair here, at communicator
    // creation, rather than inside the first SetUp.
    c.ctrl_->alltoallv(std::vector<std::vector<uint8_t>>(static_cast<size_t>(nranks), std::vector<uint8_t>(8, 0)));
  }
  if (device >= 0 && cc.backend != "p2p") {
    if (cc.backend == "nccl")
      c.transport_ = sfg::make_nccl_transport(c.nccl_, rank, device);
    else
      c.transport_ = sfg::make_threads_transport(w, rank, device, cc.timeout_s);
  }
  return h.release();
}

}  // namespace

extern "C" {

int sfg_comm_create(sfg_world world, int nranks, int rank, int device, const char* backend,
                    const void* nccl_id, const sfg_config* cfg, sfg_comm* out) {
  return guard([&] {
    *out = make_comm(world, nranks, rank, device, to_config(cfg, backend), nccl_id, nullptr);
  });
}

int sfg_comm_create_ext(int nranks, int rank, int device, const char* backend,
                        const void* nccl_id, const sfg_config* cfg, const sfg_ctrl_ops* ops,
                        sfg_comm* out) {
  return guard([&] {
    SFG_REQUIRE(ops && ops->allgather && ops->alltoallv && ops->barrier,
                "control-plane callbacks missing");
    *out = make_comm(nullptr, nranks, rank, device, to_config(cfg, backend), nccl_id, ops);
  });
}

int sfg_comm_destroy(sfg_comm c) {
  return guard([&] { delete c; });
}

int sfg_comm_rank(sfg_comm c, int* rank, int* size, int* device) {
  return guard([&] {
    if (rank) *rank = c->c->rank();
    if (size) *size = c->c->size();
    if (device) *device = c->c->device();
  });
}

int sfg_comm_allgather(sfg_comm c, const void* in, size_t bytes, void* out) {
  return guard([&] {
    SFG_REQUIRE(c != nullptr, "allgather needs a valid communicator");
    c->c->ctrl().allgather(in, bytes, out);
  });
}

int sfg_sf_create(sfg_comm c, sfg_sf* out) {
  return guard([&] {
    SFG_REQUIRE(c != nullptr, "star forest needs a valid communicator");
    *out = reinterpret_cast<sfg_sf>(new sfg::StarForest(c->c.get()));
  });
}

int sfg_sf_destroy(sfg_sf sf) {
  return guard([&] { delete SF(sf); });
}

int sfg_sf_set_graph(sfg_sf sf, int64_t nroots, int64_t nleaves, const int64_t* leaf_local,
                     const int32_t* remote_rank, const int64_t* remote_off) {
  return guard([&] { SF(sf)->set_graph(nroots, nleaves, leaf_local, remote_rank, remote_off); });
}

int sfg_sf_set_graph_device(sfg_sf sf, int64_t nroots, int64_t nleaves, const int64_t* leaf_local,
                            const int32_t* remote_rank, const int64_t* remote_off) {
  return guard([&] { SF(sf)->set_graph_device(nroots, nleaves, leaf_local, remote_rank, remote_off); });
}

int sfg_sf_setup(sfg_sf sf, int alg) {
  return guard([&] { SF(sf)->setup(static_cast<sfg::SetupAlg>(alg)); });
}

int sfg_sf_get_info(sfg_sf sf, sfg_sf_info* o) {
  return guard([&] {
    auto* s = SF(sf);
    o->state = static_cast<int>(s->state());
    o->nroots = s->nroots();
    o->nleaves = s->nleaves();
    o->leaf_index_bound = s->leaf_index_bound();
    o->contiguous_leaves = s->contiguous_leaves() ? 1 : 0;
    if (s->state() == sfg::SfState::set_up) {
      o->self_first = s->has_self_edges() ? 1 : 0;
      o->n_root_groups = static_cast<int>(s->root_groups().size());
      o->n_leaf_groups = static_cast<int>(s->leaf_groups().size());
    } else {
      o->self_first = 0;
      o->n_root_groups = 0;
      o->n_leaf_groups = 0;
    }
  });
}

int sfg_sf_group(sfg_sf sf, int which, int g, int* rank, int64_t* nitems, sfg_pattern* pat) {
  return guard([&] {
    const auto& gs = which == 0 ? SF(sf)->root_groups() : SF(sf)->leaf_groups();
    SFG_REQUIRE(g >= 0 && g < static_cast<int>(gs.size()), "group index out of range");
    if (rank) *rank = gs[static_cast<size_t>(g)].rank;
    if (nitems) *nitems = gs[static_cast<size_t>(g)].count();
    if (pat) fill_pattern(gs[static_cast<size_t>(g)].pat, pat);
  });
}

int sfg_sf_group_items(sfg_sf sf, int which, int g, int64_t* items) {
  return guard([&] {
    SF(sf)->host_graph();
    const auto& gs = which == 0 ? SF(sf)->root_groups() : SF(sf)->leaf_groups();
    SFG_REQUIRE(g >= 0 && g < static_cast<int>(gs.size()), "group index out of range");
    const auto& v = gs[static_cast<size_t>(g)].items;
    if (!v.empty()) std::memcpy(items, v.data(), v.size() * sizeof(int64_t));
  });
}

int sfg_sf_compute_degrees(sfg_sf sf, int64_t* out) {
  return guard([&] {
    auto d = SF(sf)->compute_degrees();
    if (!d.empty()) std::memcpy(out, d.data(), d.size() * sizeof(int64_t));
  });
}

int sfg_sf_multi_sf(sfg_sf sf, sfg_sf* out) {
  return guard([&] { *out = reinterpret_cast<sfg_sf>(&SF(sf)->multi_sf()); });
}

int sfg_sf_graph(sfg_sf sf, int64_t* leaf_index, int32_t* remote_rank, int64_t* remote_off) {
  return guard([&] {
    auto* s = SF(sf);
    s->host_graph();
    for (int64_t o = 0; o < s->nleaves(); ++o) {
      if (leaf_index) leaf_index[o] = s->leaf_index(o);
      if (remote_rank) remote_rank[o] = s->remote_rank_of(o);
      if (remote_off) remote_off[o] = s->remote_off_of(o);
    }
  });
}

int sfg_bcast_begin(sfg_sf sf, int kind, int64_t blocklen, const void* rootdata, void* leafdata,
                    int op, void* stream, sfg_handle* out) {
  return guard([&] {
    *out = out_h(sfg::bcast_begin(*SF(sf), unit(kind, blocklen), rootdata, leafdata, rop(op), st(stream)));
  });
}
int sfg_bcast_end(sfg_handle h) {
  return guard([&] { sfg::bcast_end(*H(h)); });
}

int sfg_bcast(sfg_sf sf, int kind, int64_t blocklen, const void* rootdata, void* leafdata, int op,
              void* stream) {
  return guard([&] { sfg::bcast(*SF(sf), unit(kind, blocklen), rootdata, leafdata, rop(op), st(stream)); });
}
int sfg_reduce(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata, void* rootdata, int op,
               void* stream) {
  return guard([&] { sfg::reduce(*SF(sf), unit(kind, blocklen), leafdata, rootdata, rop(op), st(stream)); });
}
int sfg_fetch_and_op(sfg_sf sf, int kind, int64_t blocklen, void* rootdata, const void* leafdata,
                     void* leafupdate, int op, void* stream) {
  return guard([&] {
    sfg::fetch_and_op(*SF(sf), unit(kind, blocklen), rootdata, leafdata, leafupdate, rop(op), st(stream));
  });
}
int sfg_gather(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata, void* multirootdata,
               void* stream) {
  return guard([&] { sfg::gather(*SF(sf), unit(kind, blocklen), leafdata, multirootdata, st(stream)); });
}
int sfg_scatter(sfg_sf sf, int kind, int64_t blocklen, const void* multirootdata, void* leafdata,
                void* stream) {
  return guard([&] { sfg::scatter(*SF(sf), unit(kind, blocklen), multirootdata, leafdata, st(stream)); });
}

int sfg_reduce_begin(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata, void* rootdata,
                     int op, void* stream, sfg_handle* out) {
  return guard([&] {
    *out = out_h(sfg::reduce_begin(*SF(sf), unit(kind, blocklen), leafdata, rootdata, rop(op), st(stream)));
  });
}
int sfg_reduce_end(sfg_handle h) {
  return guard([&] { sfg::reduce_end(*H(h)); });
}

int sfg_fetch_and_op_begin(sfg_sf sf, int kind, int64_t blocklen, void* rootdata,
                           const void* leafdata, void* leafupdate, int op, void* stream,
                           sfg_handle* out) {
  return guard([&] {
    *out = out_h(sfg::fetch_and_op_begin(*SF(sf), unit(kind, blocklen), rootdata, leafdata,
                                         leafupdate, rop(op), st(stream)));
  });
}
int sfg_fetch_and_op_end(sfg_handle h) {
  return guard([&] { sfg::fetch_and_op_end(*H(h)); });
}

int sfg_sf_compose(sfg_sf a, sfg_sf b, int inverse, sfg_sf* out) {
  return guard([&] {
    auto f = inverse ? sfg::compose_inverse(*SF(a), *SF(b)) : sfg::compose(*SF(a), *SF(b));
    *out = reinterpret_cast<sfg_sf>(f.release());
  });
}
int sfg_sf_embed(sfg_sf sf, int which, const int64_t* sel, int64_t n, sfg_sf* out) {
  return guard([&] {
    SFG_REQUIRE(n == 0 || sel != nullptr, "embed: selection pointer is null");
    auto f = which == 0 ? sfg::embed_root(*SF(sf), sel, n) : sfg::embed_leaf(*SF(sf), sel, n);
    *out = reinterpret_cast<sfg_sf>(f.release());
  });
}
int sfg_sf_identity(sfg_comm c, int64_t n, sfg_sf* out) {
  return guard([&] {
    SFG_REQUIRE(c != nullptr, "identity_sf needs a valid communicator");
    *out = reinterpret_cast<sfg_sf>(sfg::identity_sf(*c->c, n).release());
  });
}

int sfg_mat_create(sfg_comm c, int64_t rows, int64_t cols, const int64_t* rowptr,
                   const int64_t* colind, const void* vals, int kind, sfg_mat* out) {
  return guard([&] {
    SFG_REQUIRE(c != nullptr, "matrix needs a valid communicator");
    auto m = sfg::matrix_upload(*c->c, rows, cols, rowptr, colind, vals, unit(kind, 1).kind);
    *out = reinterpret_cast<sfg_mat>(m.release());
  });
}
int sfg_mat_destroy(sfg_mat m) {
  return guard([&] { delete reinterpret_cast<sfg::DevMatrix*>(m); });
}
int sfg_spmv(sfg_sf sf, sfg_mat diag, sfg_mat offdiag, const void* x_owned, void* lvec, void* y,
             void* stream) {
  return guard([&] {
    sfg::spmv(*SF(sf), *reinterpret_cast<sfg::DevMatrix*>(diag), *reinterpret_cast<sfg::DevMatrix*>(offdiag),
              x_owned, lvec, y, st(stream));
  });
}
int sfg_spmv_transpose(sfg_sf sf, sfg_mat diag, sfg_mat offdiag, const void* x_owned, void* lvec,
                       void* y, void* stream) {
  return guard([&] {
    sfg::spmv_transpose(*SF(sf), *reinterpret_cast<sfg::DevMatrix*>(diag),
                        *reinterpret_cast<sfg::DevMatrix*>(offdiag), x_owned, lvec, y, st(stream));
  });
}

int sfg_gather_begin(sfg_sf sf, int kind, int64_t blocklen, const void* leafdata,
                     void* multirootdata, void* stream, sfg_handle* out) {
  return guard([&] {
    *out = out_h(sfg::gather_begin(*SF(sf), unit(kind, blocklen), leafdata, multirootdata, st(stream)));
  });
}
int sfg_gather_end(sfg_handle h) {
  return guard([&] { sfg::gather_end(*H(h)); });
}

int sfg_scatter_begin(sfg_sf sf, int kind, int64_t blocklen, const void* multirootdata,
                      void* leafdata, void* stream, sfg_handle* out) {
  return guard([&] {
    *out = out_h(sfg::scatter_begin(*SF(sf), unit(kind, blocklen), multirootdata, leafdata, st(stream)));
  });
}
int sfg_scatter_end(sfg_handle h) {
  return guard([&] { sfg::scatter_end(*H(h)); });
}

int sfg_handle_info(sfg_handle h, int* opkind, int* op, int* ended) {
  return guard([&] {
    auto* x = H(h);
    if (opkind) *opkind = static_cast<int>(x->kind);
    if (op) *op = static_cast<int>(x->op);
    if (ended) *ended = x->ended ? 1 : 0;
  });
}

int sfg_handle_free(sfg_handle h) {
  return guard([&] {
    auto* x = reinterpret_cast<sfg::OpHandle*>(h);
    if (x && x->stg && x->sf) {
      if (!x->ended && x->sf->comm().p2p() && x->stg->flags) {
        // Begun, never ended: a peer's message may still be unconsumed in
        // the slot and its device counters are one behind, so the slot is
        // retired (never reused; freed with the forest), not returned.
        x->stg->retired = true;
        x->stg = nullptr;
        delete x;
        sfg::fail("operation freed without End on the p2p backend; its staging slot is retired "
                  "(every rank must end every operation it began)");
      }
      x->sf->release_staging(x->stg, x->stream);
    }
    delete x;
  });
}

int sfg_sf_prepare(sfg_sf sf, int kind, int64_t blocklen) {
  return guard([&] { SF(sf)->prepare(unit(kind, blocklen).bytes()); });
}

int sfg_pattern_analyze(const int64_t* idx, int64_t n, int infer_affine, int64_t ex, int64_t exy,
                        sfg_pattern* out) {
  return guard([&] { fill_pattern(sfg::Pattern::analyze(idx, n, infer_affine != 0, ex, exy), out); });
}

int sfg_trace_dump(const char* path) {
  return guard([&] { sfg::trace_dump(path); });
}

int sfg_counters_get(sfg_counters* o) {
  return guard([&] {
    auto& c = sfg::counters();
    o->pack_copies = c.pack_copies;
    o->pack_elided = c.pack_elided;
    o->unpack_copies = c.unpack_copies;
    o->unpack_elided = c.unpack_elided;
    o->replace_dup_collisions = c.replace_dup_collisions;
    o->kernel_launches = c.kernel_launches;
    o->bytes_sent = c.bytes_sent;
    o->bytes_recv = c.bytes_recv;
    o->transport_calls = c.transport_calls;
  });
}

int sfg_counters_reset(void) {
  return guard([&] { sfg::counters().reset(); });
}

int sfg_timing_enable(int on) {
  return guard([&] { sfg::timing_enable(on != 0); });
}

int sfg_timing_collect(sfg_timing* out, int cap, int* n) {
  return guard([&] {
    auto recs = sfg::timing_collect();
    int k = 0;
    for (const auto& r : recs) {
      if (k >= cap) break;
      std::memset(out[k].tag, 0, sizeof(out[k].tag));
      std::strncpy(out[k].tag, r.tag.c_str(), sizeof(out[k].tag) - 1);
      out[k].launches = r.launches;
      out[k].total_ms = r.total_ms;
      out[k].bytes = r.bytes;
      out[k].link_bytes = r.link_bytes;
      ++k;
    }
    *n = k;
  });
}

}  // extern "C"
