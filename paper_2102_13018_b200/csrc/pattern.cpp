// Index-pattern classification for the SetUp planner and the shared
// vocabulary helpers.
//
// Reference: /root/reference/proj/src/pattern.cpp:13-96 (contiguous check,
// strided detection only with GridExtents, indexed + duplicate flag). The
// planner here additionally infers Affine3D blocks without extents: the
// leading consecutive run gives dx, the first row jump gives the row stride
// s1, the number of equally spaced rows gives dy, the first plane jump gives
// s2; the whole enumeration is then verified, so a wrong guess can only fall
// back to Indexed, never mis-address.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <sstream>

#include "parallel.hpp"
#include "sfg.hpp"

namespace sfg {

// ---------------------------------------------------------------- vocabulary

const char* kind_name(Kind k) {
  switch (k) {
    case Kind::int32: return "int32";
    case Kind::int64: return "int64";
    case Kind::float64: return "float64";
    case Kind::bytes: return "bytes";
  }
  return "?";
}

const char* op_name(ReduceOp op) {
  switch (op) {
    case ReduceOp::replace: return "replace";
    case ReduceOp::sum: return "sum";
    case ReduceOp::prod: return "prod";
    case ReduceOp::max: return "max";
    case ReduceOp::min: return "min";
    case ReduceOp::land: return "land";
    case ReduceOp::lor: return "lor";
    case ReduceOp::band: return "band";
    case ReduceOp::bor: return "bor";
  }
  return "?";
}

size_t Unit::elem_size() const {
  switch (kind) {
    case Kind::int32: return 4;
    case Kind::int64: return 8;
    case Kind::float64: return 8;
    case Kind::bytes: return 1;
  }
  return 0;
}

void fail(const std::string& msg) { throw Error(msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  std::ostringstream os;
  os << "CUDA error " << cudaGetErrorName(e) << " (" << cudaGetErrorString(e) << ") in " << what
     << " at " << file << ":" << line;
  throw CudaError(os.str());
}

void nccl_check(ncclResult_t r, const char* what, const char* file, int line) {
  if (r == ncclSuccess || r == ncclInProgress) return;
  std::ostringstream os;
  os << "NCCL error " << ncclGetErrorString(r) << " in " << what << " at " << file << ":" << line;
  throw CudaError(os.str());
}

// /root/reference/proj/include/sf/unit.hpp:72-82 (same messages)
void check_unit_op(const Unit& u, ReduceOp op) {
  SFG_REQUIRE(u.blocklen >= 1, "unit blocklen must be >= 1");
  SFG_REQUIRE(static_cast<int>(u.kind) <= 3, "unknown unit kind");
  SFG_REQUIRE(static_cast<int>(op) <= 8, "unknown reduction");
  if (op == ReduceOp::replace) return;
  SFG_REQUIRE(u.kind != Kind::bytes, std::string("reduction '") + op_name(op) +
                                         "' requires a non-opaque unit kind");
  const bool logical = op == ReduceOp::land || op == ReduceOp::lor || op == ReduceOp::band ||
                       op == ReduceOp::bor;
  if (logical)
    SFG_REQUIRE(u.kind == Kind::int32 || u.kind == Kind::int64,
                std::string("reduction '") + op_name(op) + "' requires an integer unit kind");
}

void Counters::reset() {
  pack_copies = 0;
  pack_elided = 0;
  unpack_copies = 0;
  unpack_elided = 0;
  replace_dup_collisions = 0;
  kernel_launches = 0;
  bytes_sent = 0;
  bytes_recv = 0;
  transport_calls = 0;
}

Counters& counters() {
  static Counters c;
  return c;
}

// ------------------------------------------------------------------- timing

namespace {
struct TimingState {
  std::mutex mu;
  bool on = false;
  struct Pending {
    std::string tag;
    cudaEvent_t a, b;
    double bytes;
    double link_bytes;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
};
TimingState& ts() {
  static TimingState t;
  return t;
}
}  // namespace

void timing_enable(bool on) {
  std::lock_guard<std::mutex> lk(ts().mu);
  ts().on = on;
}

bool timing_enabled() { return ts().on; }

cudaEvent_t timing_event() {
  {
    std::lock_guard<std::mutex> lk(ts().mu);
    if (!ts().pool.empty()) {
      cudaEvent_t e = ts().pool.back();
      ts().pool.pop_back();
      return e;
    }
  }
  cudaEvent_t e;
  SFG_CUDA(cudaEventCreate(&e));
  return e;
}

void timing_record(const char* tag, cudaEvent_t a, cudaEvent_t b, double bytes,
                   double link_bytes) {
  std::lock_guard<std::mutex> lk(ts().mu);
  ts().pending.push_back({tag, a, b, bytes, link_bytes});
}

std::vector<TimingRec> timing_collect() {
  std::vector<TimingState::Pending> pend;
  {
    std::lock_guard<std::mutex> lk(ts().mu);
    pend.swap(ts().pending);
  }
  std::vector<TimingRec> out;
  for (auto& p : pend) {
    SFG_CUDA(cudaEventSynchronize(p.b));
    float ms = 0.f;
    SFG_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto it = std::find_if(out.begin(), out.end(), [&](const TimingRec& r) { return r.tag == p.tag; });
    if (it == out.end()) {
      out.push_back(TimingRec{p.tag, 0, 0.0, 0.0, 0.0});
      it = out.end() - 1;
    }
    it->launches++;
    it->total_ms += ms;
    it->bytes += p.bytes;
    it->link_bytes += p.link_bytes;
    std::lock_guard<std::mutex> lk(ts().mu);
    ts().pool.push_back(p.a);
    ts().pool.push_back(p.b);
  }
  return out;
}

// ------------------------------------------------------------------ pattern

namespace {

int64_t count_distinct(const HostVec<int64_t>& v, int64_t lo, int64_t hi) {
  if (v.size() < 2) return static_cast<int64_t>(v.size());
  const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
  if (span <= 4 * static_cast<uint64_t>(v.size()) + 4096) {
    std::vector<uint8_t> seen(span, 0);
    int64_t d = 0;
    for (int64_t x : v) {
      uint8_t& s = seen[static_cast<size_t>(x - lo)];
      d += s == 0;
      s = 1;
    }
    return d;
  }
  std::vector<int64_t> sorted(v.begin(), v.end());
  std::sort(sorted.begin(), sorted.end());
  return static_cast<int64_t>(std::unique(sorted.begin(), sorted.end()) - sorted.begin());
}

// Verify start + k*s2 + j*s1 + x over (dz, dy, dx), rows in parallel.
bool verify_affine(const int64_t* idx, int64_t start, int64_t dx, int64_t dy, int64_t dz,
                   int64_t s1, int64_t s2) {
  const int64_t rows = dy * dz;
  return parallel_find_first(rows, [&](int64_t r) {
           const int64_t k = r / dy, j = r - k * dy;
           const int64_t row = start + k * s2 + j * s1;
           const int64_t* p = idx + r * dx;
           for (int64_t x = 0; x < dx; ++x)
             if (p[x] != row + x) return true;
           return false;
         }) == rows;
}

}  // namespace

Pattern Pattern::contiguous_range(int64_t start, int64_t n) {
  Pattern p;
  p.kind = contiguous;
  p.start = n == 0 ? 0 : start;
  p.count = n;
  p.bound = n == 0 ? 0 : start + n;
  p.distinct = n;
  return p;
}

Pattern Pattern::analyze(const int64_t* idx, int64_t n, bool infer_affine, int64_t ex,
                         int64_t exy) {
  if (n == 0) return contiguous_range(0, 0);
  const int64_t start = idx[0];
  const int64_t run = parallel_find_first(n, [&](int64_t i) { return idx[i] != start + i; });
  if (run == n) return contiguous_range(start, n);

  auto make_affine = [&](int64_t dx, int64_t dy, int64_t dz, int64_t s1, int64_t s2) {
    Pattern p;
    p.kind = affine;
    p.count = n;
    p.start = start;
    p.dx = dx;
    p.dy = dy;
    p.dz = dz;
    p.s1 = s1;
    p.s2 = s2;
    p.bound = start + (dz - 1) * s2 + (dy - 1) * s1 + dx;
    p.distinct = n;
    return p;
  };

  if (ex > 0 && exy > 0 && exy % ex == 0) {
    // Reference-style detection with known extents (pattern.cpp:22-46).
    const int64_t dx = run;
    if (dx <= ex && n % dx == 0) {
      const int64_t rows = n / dx;
      int64_t dy = 1;
      while (dy < rows && idx[dy * dx] == start + dy * ex) ++dy;
      if (rows % dy == 0 && dy <= exy / ex) {
        const int64_t dz = rows / dy;
        if (verify_affine(idx, start, dx, dy, dz, ex, exy))
          return make_affine(dx, dy, dz, ex, exy);
      }
    }
  } else if (infer_affine && start >= 0) {
    const int64_t dx = run;
    if (n % dx == 0) {
      const int64_t rows = n / dx;
      const int64_t s1 = idx[dx] - start;
      if (s1 >= dx) {
        int64_t dy = 1;
        while (dy < rows && idx[dy * dx] == start + dy * s1) ++dy;
        if (rows % dy == 0) {
          const int64_t dz = rows / dy;
          const int64_t s2 = dz > 1 ? idx[dy * dx] - start : dy * s1;
          const bool planes_ok = dz == 1 || s2 >= (dy - 1) * s1 + dx;
          if (planes_ok && dx < (int64_t(1) << 31) && dy < (int64_t(1) << 31) &&
              verify_affine(idx, start, dx, dy, dz, s1, s2))
            return make_affine(dx, dy, dz, s1, s2);
        }
      }
    }
  }

  Pattern p;
  p.kind = indexed;
  p.count = n;
  p.idx.assign(idx, idx + n);
  int64_t lo = idx[0], hi = idx[0];
  for (int64_t i = 1; i < n; ++i) {
    lo = std::min(lo, idx[i]);
    hi = std::max(hi, idx[i]);
  }
  p.start = lo;
  p.bound = hi + 1;
  p.distinct = count_distinct(p.idx, lo, hi);
  p.has_duplicates = p.distinct < n;
  return p;
}

int64_t Pattern::index(int64_t i) const {
  switch (kind) {
    case contiguous: return start + i;
    case affine: {
      const int64_t x = i % dx;
      const int64_t r = i / dx;
      return start + x + (r % dy) * s1 + (r / dy) * s2;
    }
    case indexed: return idx[static_cast<size_t>(i)];
  }
  return 0;
}

DPat to_dpat(const Pattern& p, const int32_t* dev_idx) {
  DPat d;
  d.start = p.start;
  switch (p.kind) {
    case Pattern::contiguous: d.kind = PAT_CONTIG; break;
    case Pattern::affine:
      d.kind = PAT_AFFINE;
      d.s1 = p.s1;
      d.s2 = p.s2;
      d.dx = make_fastdiv(static_cast<uint32_t>(p.dx));
      d.dy = make_fastdiv(static_cast<uint32_t>(p.dy));
      break;
    case Pattern::indexed:
      d.kind = PAT_INDEXED;
      d.idx = dev_idx;
      break;
  }
  return d;
}

}  // namespace sfg
