// Parallel SpMV over the star forest: the consumer of the ghost exchange
// (reference /root/reference/proj/include/sf/spmv.hpp:147-169).
//
//   spmv:            bcast_begin(x_owned -> lvec); y = A x_owned; bcast_end;
//                    y += B lvec                 (spmv.hpp:149-157)
//   spmv_transpose:  y = A^T x_owned; lvec = B^T x_owned;
//                    reduce(lvec -> y, SUM)      (spmv.hpp:161-169)
//
// A (diagonal block) and B (off-diagonal block, columns = garray) live on the
// device in SELL-32 form — rows in slices of 32, each slice's entries stored
// column-major, so the 32 lanes of a warp read consecutive words — with the
// transposes (for spmv_transpose) built once at upload. One thread per row
// accumulates its row's products in CSR order with round-to-nearest multiply
// and add (no FMA contraction), which is exactly the reference's sequential
// loop (Csr::multiply / multiply_add / multiply_transpose_add): results are
// bit-identical to the reference's distributed CPU SpMV.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <type_traits>

#include "sfg.hpp"

#ifndef SPMV_UNROLL
#define SPMV_UNROLL 8
#endif

namespace sfg {
namespace {

template <class T>
__device__ __forceinline__ T mul_rn(T a, T b) {
  if constexpr (std::is_same_v<T, double>)
    return __dmul_rn(a, b);
  else
    return static_cast<T>(static_cast<unsigned long long>(a) * static_cast<unsigned long long>(b));
}
template <class T>
__device__ __forceinline__ T add_rn(T a, T b) {
  if constexpr (std::is_same_v<T, double>)
    return __dadd_rn(a, b);
  else
    return static_cast<T>(static_cast<unsigned long long>(a) + static_cast<unsigned long long>(b));
}

// acc += sum_k val * x[col] over one row's SELL slots, in CSR order. The
// matrix streams through once (evict-first loads keep L1 for x); kUnroll
// slots' loads are issued before their products so a thread keeps 2*kUnroll
// independent loads in flight.
constexpr int kUnroll = SPMV_UNROLL;
template <class T>
__device__ __forceinline__ void row_dot(int64_t base, int len, const int32_t* __restrict__ col,
                                        const T* __restrict__ val, const T* __restrict__ x, T& acc) {
  int k = 0;
  for (; k + kUnroll <= len; k += kUnroll) {
    int32_t c[kUnroll];
    T v[kUnroll], xv[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) {
      c[q] = __ldcs(col + base + static_cast<int64_t>(k + q) * 32);
      v[q] = __ldcs(val + base + static_cast<int64_t>(k + q) * 32);
    }
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) xv[q] = __ldg(x + c[q]);
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) acc = add_rn(acc, mul_rn(v[q], xv[q]));
  }
  if (k < len) {  // the tail, as one predicated batch
    int32_t c[kUnroll];
    T v[kUnroll], xv[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; ++q)
      if (k + q < len) {
        c[q] = __ldcs(col + base + static_cast<int64_t>(k + q) * 32);
        v[q] = __ldcs(val + base + static_cast<int64_t>(k + q) * 32);
      }
#pragma unroll
    for (int q = 0; q < kUnroll; ++q)
      if (k + q < len) xv[q] = __ldg(x + c[q]);
#pragma unroll
    for (int q = 0; q < kUnroll; ++q)
      if (k + q < len) acc = add_rn(acc, mul_rn(v[q], xv[q]));
  }
}

// y[r] (=|+=) sum_k vals * x[col], k in the row's CSR order.
template <class T, bool ADD, bool PLUS_ZERO>
__global__ void __launch_bounds__(256) sell_spmv_kernel(int64_t rows, const int64_t* __restrict__ slice_off,
                                                        const int32_t* __restrict__ row_len,
                                                        const int32_t* __restrict__ col,
                                                        const T* __restrict__ val, const T* __restrict__ x,
                                                        T* __restrict__ y) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t s = r >> 5;
  const int lane = static_cast<int>(r & 31);
  const int64_t base = __ldg(slice_off + s) + lane;
  const int len = __ldg(row_len + r);
  T acc = T(0);
  row_dot(base, len, col, val, x, acc);
  if constexpr (PLUS_ZERO) acc = add_rn(acc, T(0));
  y[r] = ADD ? add_rn(y[r], acc) : acc;
}

// y[r] += B_r . x over the rows that HAVE entries only (list nz_rows). For
// the other rows the reference adds an empty dot product, y[r] + 0, which
// leaves every y the diagonal product can produce unchanged bit for bit: its
// accumulator starts at +0.0 and round-to-nearest never yields -0.0 from it,
// so y is never -0.0 (the one value + 0 changes), and integers are unchanged.
template <class T>
__global__ void __launch_bounds__(256) sell_spmv_add_rows_kernel(int64_t n, const int32_t* __restrict__ rows,
                                                                 const int64_t* __restrict__ slice_off,
                                                                 const int32_t* __restrict__ row_len,
                                                                 const int32_t* __restrict__ col,
                                                                 const T* __restrict__ val,
                                                                 const T* __restrict__ x, T* __restrict__ y) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t r = __ldg(rows + t);
  const int64_t base = __ldg(slice_off + (r >> 5)) + (r & 31);
  const int len = __ldg(row_len + r);
  T acc = T(0);
  row_dot(base, len, col, val, x, acc);
  y[r] = add_rn(y[r], acc);
}

// Host SELL-32 image of a CSR matrix (rows sliced by 32, column-major inside
// a slice; padding slots are never read).
struct SellHost {
  std::vector<int64_t> slice_off;
  std::vector<int32_t> row_len, col;
  std::vector<uint8_t> val;  // elem-size bytes per slot
};

SellHost to_sell(int64_t rows, const int64_t* rowptr, const int64_t* colind, const uint8_t* vals,
                 size_t esz) {
  SellHost h;
  const int64_t nslices = (rows + 31) / 32;
  h.slice_off.resize(static_cast<size_t>(nslices) + 1);
  h.row_len.resize(static_cast<size_t>(rows));
  int64_t off = 0;
  for (int64_t s = 0; s < nslices; ++s) {
    int32_t w = 0;
    for (int64_t r = s * 32; r < std::min(rows, s * 32 + 32); ++r) {
      const int64_t len = rowptr[r + 1] - rowptr[r];
      SFG_REQUIRE(len <= INT32_MAX, "matrix row too long for the device layout");
      h.row_len[static_cast<size_t>(r)] = static_cast<int32_t>(len);
      w = std::max(w, static_cast<int32_t>(len));
    }
    h.slice_off[static_cast<size_t>(s)] = off;
    off += static_cast<int64_t>(w) * 32;
  }
  h.slice_off[static_cast<size_t>(nslices)] = off;
  h.col.assign(static_cast<size_t>(off), 0);
  h.val.assign(static_cast<size_t>(off) * esz, 0);
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t base = h.slice_off[static_cast<size_t>(r >> 5)] + (r & 31);
    for (int64_t i = rowptr[r], k = 0; i < rowptr[r + 1]; ++i, ++k) {
      const int64_t slot = base + k * 32;
      SFG_REQUIRE(colind[i] >= 0 && colind[i] <= INT32_MAX, "matrix column index outside the int32 range");
      h.col[static_cast<size_t>(slot)] = static_cast<int32_t>(colind[i]);
      std::memcpy(&h.val[static_cast<size_t>(slot) * esz], vals + static_cast<size_t>(i) * esz, esz);
    }
  }
  return h;
}

// CSR of the transpose with every column's entries in ascending original
// row — the order in which Csr::multiply_transpose_add visits them.
void transpose_csr(int64_t rows, int64_t cols, const int64_t* rowptr, const int64_t* colind,
                   const uint8_t* vals, size_t esz, std::vector<int64_t>& trp, std::vector<int64_t>& tci,
                   std::vector<uint8_t>& tv) {
  const int64_t nnz = rowptr[rows];
  trp.assign(static_cast<size_t>(cols) + 1, 0);
  for (int64_t i = 0; i < nnz; ++i) ++trp[static_cast<size_t>(colind[i]) + 1];
  std::partial_sum(trp.begin(), trp.end(), trp.begin());
  std::vector<int64_t> cur(trp.begin(), trp.end() - 1);
  tci.resize(static_cast<size_t>(nnz));
  tv.resize(static_cast<size_t>(nnz) * esz);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t i = rowptr[r]; i < rowptr[r + 1]; ++i) {
      const int64_t p = cur[static_cast<size_t>(colind[i])]++;
      tci[static_cast<size_t>(p)] = r;
      std::memcpy(&tv[static_cast<size_t>(p) * esz], vals + static_cast<size_t>(i) * esz, esz);
    }
}

void upload_sell(const SellHost& h, size_t esz, DevMatrix::Sell& d, std::vector<void*>& allocs) {
  auto up = [&](const void* src, size_t bytes) -> void* {
    void* p = nullptr;
    SFG_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    if (bytes) SFG_CUDA(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
    allocs.push_back(p);
    return p;
  };
  d.rows = static_cast<int64_t>(h.row_len.size());
  d.slice_off = static_cast<int64_t*>(up(h.slice_off.data(), h.slice_off.size() * sizeof(int64_t)));
  d.row_len = static_cast<int32_t*>(up(h.row_len.data(), h.row_len.size() * sizeof(int32_t)));
  d.col = static_cast<int32_t*>(up(h.col.data(), h.col.size() * sizeof(int32_t)));
  d.val = up(h.val.data(), h.val.size());
  d.slots = static_cast<int64_t>(h.col.size());
  std::vector<int32_t> nz;
  for (size_t r = 0; r < h.row_len.size(); ++r)
    if (h.row_len[r] > 0) nz.push_back(static_cast<int32_t>(r));
  d.n_nz_rows = static_cast<int64_t>(nz.size());
  d.nz_rows = static_cast<int32_t*>(up(nz.data(), nz.size() * sizeof(int32_t)));
  (void)esz;
}

// y += B lvec over B's non-empty rows only (see sell_spmv_add_rows_kernel):
// valid when y holds a product this library computed (never -0.0).
template <class T>
void launch_add_rows(const DevMatrix::Sell& m, const void* x, void* y, cudaStream_t s) {
  if (m.n_nz_rows == 0) return;
  const unsigned blocks = static_cast<unsigned>((m.n_nz_rows + 255) / 256);
  const bool timed = timing_enabled();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    e0 = timing_event();
    e1 = timing_event();
    SFG_CUDA(cudaEventRecord(e0, s));
  }
  sell_spmv_add_rows_kernel<T><<<blocks, 256, 0, s>>>(m.n_nz_rows, m.nz_rows, m.slice_off, m.row_len, m.col,
                                                      static_cast<const T*>(m.val), static_cast<const T*>(x),
                                                      static_cast<T*>(y));
  SFG_CUDA(cudaGetLastError());
  counters().kernel_launches++;
  if (timed) {
    SFG_CUDA(cudaEventRecord(e1, s));
    const double nnz = static_cast<double>(m.nnz);
    const double b = nnz * (sizeof(T) + 4) + static_cast<double>(m.cols) * sizeof(T) +
                     static_cast<double>(m.n_nz_rows) * (sizeof(T) * 2 + 8);
    timing_record("spmv_offdiag", e0, e1, b);
  }
}

template <class T, bool ADD, bool PLUS_ZERO>
void launch_sell(const DevMatrix::Sell& m, const void* x, void* y, cudaStream_t s) {
  if (m.rows == 0) return;
  const unsigned blocks = static_cast<unsigned>((m.rows + 255) / 256);
  const bool timed = timing_enabled();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    e0 = timing_event();
    e1 = timing_event();
    SFG_CUDA(cudaEventRecord(e0, s));
  }
  sell_spmv_kernel<T, ADD, PLUS_ZERO><<<blocks, 256, 0, s>>>(m.rows, m.slice_off, m.row_len, m.col,
                                                  static_cast<const T*>(m.val), static_cast<const T*>(x),
                                                  static_cast<T*>(y));
  SFG_CUDA(cudaGetLastError());
  counters().kernel_launches++;
  if (timed) {
    SFG_CUDA(cudaEventRecord(e1, s));
    // compulsory bytes: stored entries (value + int32 column), x per entry
    // (gathered; cached re-reads not counted twice would need the matrix
    // structure), y written (and read when accumulating), row lengths.
    const double nnz = static_cast<double>(m.nnz);
    const double b = nnz * (sizeof(T) + 4) + static_cast<double>(m.cols) * sizeof(T) +
                     static_cast<double>(m.rows) * (sizeof(T) * (ADD ? 2 : 1) + 4);
    timing_record(ADD ? "spmv_offdiag" : "spmv_diag", e0, e1, b);
  }
}

template <bool ADD, bool PLUS_ZERO = false>
void run_sell(Kind k, const DevMatrix::Sell& m, const void* x, void* y, cudaStream_t s) {
  if (k == Kind::float64)
    launch_sell<double, ADD, PLUS_ZERO>(m, x, y, s);
  else
    launch_sell<int64_t, ADD, PLUS_ZERO>(m, x, y, s);
}

}  // namespace

DevMatrix::~DevMatrix() {
  if (device >= 0) cudaSetDevice(device);
  for (void* p : allocs) cudaFree(p);
}

std::unique_ptr<DevMatrix> matrix_upload(Comm& comm, int64_t rows, int64_t cols, const int64_t* rowptr,
                                         const int64_t* colind, const void* vals, Kind kind) {
  SFG_REQUIRE(kind == Kind::float64 || kind == Kind::int64, "SpMV supports float64 and int64 matrices");
  SFG_REQUIRE(rows >= 0 && cols >= 0 && rowptr != nullptr && rowptr[0] == 0, "matrix: bad CSR row pointer");
  // row numbers (of the matrix and of its transpose) are int32 on the device
  SFG_REQUIRE(rows <= INT32_MAX && cols <= INT32_MAX, "matrix dimensions outside the int32 range");
  for (int64_t r = 0; r < rows; ++r) SFG_REQUIRE(rowptr[r + 1] >= rowptr[r], "matrix: bad CSR row pointer");
  const int64_t nnz = rowptr[rows];
  for (int64_t i = 0; i < nnz; ++i)
    SFG_REQUIRE(colind[i] >= 0 && colind[i] < cols, "matrix: column index outside the matrix");
  comm.bind_device();
  auto m = std::make_unique<DevMatrix>();
  m->device = comm.device();
  m->kind = kind;
  m->rows = rows;
  m->cols = cols;
  m->nnz = nnz;
  const size_t esz = 8;
  const auto* v = static_cast<const uint8_t*>(vals);
  upload_sell(to_sell(rows, rowptr, colind, v, esz), esz, m->fwd, m->allocs);
  std::vector<int64_t> trp, tci;
  std::vector<uint8_t> tv;
  transpose_csr(rows, cols, rowptr, colind, v, esz, trp, tci, tv);
  upload_sell(to_sell(cols, trp.data(), tci.data(), tv.data(), esz), esz, m->bwd, m->allocs);
  m->fwd.nnz = m->bwd.nnz = nnz;
  m->fwd.cols = cols;
  m->bwd.cols = rows;
  return m;
}

// spmv.hpp:149-157
void spmv(StarForest& sf, const DevMatrix& diag, const DevMatrix& off, const void* x_owned, void* lvec,
          void* y, cudaStream_t s) {
  SFG_REQUIRE(diag.kind == off.kind, "spmv: diagonal and off-diagonal blocks differ in kind");
  SFG_REQUIRE(diag.cols == sf.nroots() && off.cols == sf.leaf_index_bound() && diag.rows == off.rows,
              "spmv: matrix blocks do not match the ghost forest");
  const Unit u{diag.kind, 1};
  auto h = bcast_begin(sf, u, x_owned, lvec, ReduceOp::replace, s);
  // y = A x overlaps the ghost exchange. With an empty off-diagonal block the
  // reference's `y += 0` is folded into it (acc + 0, the same bits).
  if (off.nnz == 0)
    run_sell<false, true>(diag.kind, diag.fwd, x_owned, y, s);
  else
    run_sell<false>(diag.kind, diag.fwd, x_owned, y, s);
  bcast_end(*h);
  if (off.nnz != 0) {
    if (off.kind == Kind::float64)
      launch_add_rows<double>(off.fwd, lvec, y, s);
    else
      launch_add_rows<int64_t>(off.fwd, lvec, y, s);
  }
}

// spmv.hpp:161-169
void spmv_transpose(StarForest& sf, const DevMatrix& diag, const DevMatrix& off, const void* x_owned,
                    void* lvec, void* y, cudaStream_t s) {
  SFG_REQUIRE(diag.kind == off.kind, "spmv_transpose: diagonal and off-diagonal blocks differ in kind");
  SFG_REQUIRE(diag.cols == sf.nroots() && off.cols == sf.leaf_index_bound() && diag.rows == off.rows,
              "spmv_transpose: matrix blocks do not match the ghost forest");
  const Unit u{diag.kind, 1};
  run_sell<false>(diag.kind, diag.bwd, x_owned, y, s);  // y = A^T x
  run_sell<false>(off.kind, off.bwd, x_owned, lvec, s);  // lvec = B^T x
  auto h = reduce_begin(sf, u, lvec, y, ReduceOp::sum, s);
  reduce_end(*h);
}

}  // namespace sfg
