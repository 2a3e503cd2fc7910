/* TEST INFRASTRUCTURE ONLY — the CPU oracle of the star-forest data path.
 *
 * A plain-C restatement of the reference's sequential oracle and operation
 * semantics, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER. The product path (paper_2102_13018_b200)
 * never links, imports or calls this file.
 *
 * What it restates (file:line in /root/reference/proj):
 *   edge list of a global graph       src/oracle.cpp:12-26 (GlobalGraph::from_specs)
 *   op semantics                      src/pack.cpp:19-45, src/oracle.cpp:51-63
 *   bcast                             src/oracle.cpp:65-77
 *   reduce, deterministic fold order  src/oracle.cpp:79-101 (key: root rank,
 *                                     root offset, self first, leaf rank, leaf idx)
 *   degrees                           src/oracle.cpp:103-110
 *   gather / scatter slot order       src/oracle.cpp:115-164
 *   serialized fetch-and-op           src/oracle.cpp:166-188
 * The reference oracle is int64-only; this one covers every kind the path
 * supports (int32, int64, float64 and opaque bytes for replace) and any
 * blocklen, with the library's typed semantics (pack.cpp functors; integer
 * arithmetic wraps). Parity is pinned against the reference's golden vectors
 * (tests/golden/fig2.json, from tests/test_sfops.cpp) and against outputs of
 * the reference library itself (tests/golden/ref_random.npz, made by
 * tests/golden/make_golden.py through oracle/_ref).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { K_I32 = 0, K_I64 = 1, K_F64 = 2, K_BYTES = 3 };
enum { OP_REPLACE = 0, OP_SUM, OP_PROD, OP_MAX, OP_MIN, OP_LAND, OP_LOR, OP_BAND, OP_BOR };

typedef struct {
  int32_t root_rank;
  int32_t remote; /* 0 for self edges, which sort first */
  int32_t leaf_rank;
  int64_t root_off;
  int64_t leaf_idx;
  int64_t id; /* original edge position */
} key_t_;

static int cmp_key(const void* pa, const void* pb) {
  const key_t_* a = (const key_t_*)pa;
  const key_t_* b = (const key_t_*)pb;
  if (a->root_rank != b->root_rank) return a->root_rank < b->root_rank ? -1 : 1;
  if (a->root_off != b->root_off) return a->root_off < b->root_off ? -1 : 1;
  /* self?-1:leaf_rank */
  int64_t ra = a->remote ? a->leaf_rank : -1, rb = b->remote ? b->leaf_rank : -1;
  if (ra != rb) return ra < rb ? -1 : 1;
  if (a->leaf_idx != b->leaf_idx) return a->leaf_idx < b->leaf_idx ? -1 : 1;
  return 0;
}

static size_t kind_size(int kind) {
  switch (kind) {
    case K_I32: return 4;
    case K_I64: return 8;
    case K_F64: return 8;
    default: return 1;
  }
}

/* a (op)= b, one element (pack.cpp:19-45) */
static void apply(int kind, int op, void* a, const void* b) {
  if (op == OP_REPLACE) {
    memcpy(a, b, kind_size(kind));
    return;
  }
  if (kind == K_F64) {
    double x = *(double*)a, y = *(const double*)b;
    switch (op) {
      case OP_SUM: x = x + y; break;
      case OP_PROD: x = x * y; break;
      case OP_MAX: if (y > x) x = y; break;
      case OP_MIN: if (y < x) x = y; break;
      default: break;
    }
    *(double*)a = x;
  } else if (kind == K_I64) {
    int64_t x = *(int64_t*)a, y = *(const int64_t*)b;
    switch (op) {
      case OP_SUM: x = (int64_t)((uint64_t)x + (uint64_t)y); break;
      case OP_PROD: x = (int64_t)((uint64_t)x * (uint64_t)y); break;
      case OP_MAX: if (y > x) x = y; break;
      case OP_MIN: if (y < x) x = y; break;
      case OP_LAND: x = (x && y) ? 1 : 0; break;
      case OP_LOR: x = (x || y) ? 1 : 0; break;
      case OP_BAND: x = x & y; break;
      case OP_BOR: x = x | y; break;
    }
    *(int64_t*)a = x;
  } else if (kind == K_I32) {
    int32_t x = *(int32_t*)a, y = *(const int32_t*)b;
    switch (op) {
      case OP_SUM: x = (int32_t)((uint32_t)x + (uint32_t)y); break;
      case OP_PROD: x = (int32_t)((uint32_t)x * (uint32_t)y); break;
      case OP_MAX: if (y > x) x = y; break;
      case OP_MIN: if (y < x) x = y; break;
      case OP_LAND: x = (x && y) ? 1 : 0; break;
      case OP_LOR: x = (x || y) ? 1 : 0; break;
      case OP_BAND: x = x & y; break;
      case OP_BOR: x = x | y; break;
    }
    *(int32_t*)a = x;
  }
}

static void apply_vertex(int kind, int64_t bl, int op, char* dst, const char* src) {
  if (kind == K_BYTES) {
    memcpy(dst, src, (size_t)bl);
    return;
  }
  const size_t es = kind_size(kind);
  for (int64_t b = 0; b < bl; ++b) apply(kind, op, dst + (size_t)b * es, src + (size_t)b * es);
}

static key_t_* sorted_keys(int64_t ne, const int32_t* rr, const int64_t* ro, const int32_t* lr,
                           const int64_t* li) {
  key_t_* k = (key_t_*)malloc(sizeof(key_t_) * (size_t)(ne ? ne : 1));
  for (int64_t e = 0; e < ne; ++e) {
    k[e].root_rank = rr[e];
    k[e].root_off = ro[e];
    k[e].leaf_rank = lr[e];
    k[e].leaf_idx = li[e];
    k[e].remote = lr[e] != rr[e];
    k[e].id = e;
  }
  qsort(k, (size_t)ne, sizeof(key_t_), cmp_key);
  return k;
}

/* bcast: oracle.cpp:65-77 (each leaf has one root, so order is immaterial) */
int oracle_bcast(int64_t ne, const int32_t* rr, const int64_t* ro, const int32_t* lr,
                 const int64_t* li, int kind, int64_t bl, int op, char* const* rootdata,
                 char* const* leafdata) {
  const size_t ub = kind_size(kind) * (size_t)bl;
  for (int64_t e = 0; e < ne; ++e)
    apply_vertex(kind, bl, op, leafdata[lr[e]] + (size_t)li[e] * ub,
                 rootdata[rr[e]] + (size_t)ro[e] * ub);
  return 0;
}

/* reduce: oracle.cpp:79-101 */
int oracle_reduce(int64_t ne, const int32_t* rr, const int64_t* ro, const int32_t* lr,
                  const int64_t* li, int kind, int64_t bl, int op, char* const* leafdata,
                  char* const* rootdata) {
  const size_t ub = kind_size(kind) * (size_t)bl;
  key_t_* k = sorted_keys(ne, rr, ro, lr, li);
  for (int64_t e = 0; e < ne; ++e)
    apply_vertex(kind, bl, op, rootdata[k[e].root_rank] + (size_t)k[e].root_off * ub,
                 leafdata[k[e].leaf_rank] + (size_t)k[e].leaf_idx * ub);
  free(k);
  return 0;
}

/* fetch-and-op: oracle.cpp:166-188; leafupdate gets the pre-value */
int oracle_fetch_and_op(int64_t ne, const int32_t* rr, const int64_t* ro, const int32_t* lr,
                        const int64_t* li, int kind, int64_t bl, int op, char* const* rootdata,
                        char* const* leafdata, char* const* leafupdate) {
  if (op == OP_REPLACE || kind == K_BYTES) return 1;
  const size_t ub = kind_size(kind) * (size_t)bl;
  key_t_* k = sorted_keys(ne, rr, ro, lr, li);
  for (int64_t e = 0; e < ne; ++e) {
    char* root = rootdata[k[e].root_rank] + (size_t)k[e].root_off * ub;
    memcpy(leafupdate[k[e].leaf_rank] + (size_t)k[e].leaf_idx * ub, root, ub);
    apply_vertex(kind, bl, op, root, leafdata[k[e].leaf_rank] + (size_t)k[e].leaf_idx * ub);
  }
  free(k);
  return 0;
}

/* degrees: oracle.cpp:103-110 (deg[r] arrays pre-zeroed by the caller) */
int oracle_degrees(int64_t ne, const int32_t* rr, const int64_t* ro, int64_t* const* deg) {
  for (int64_t e = 0; e < ne; ++e) ++deg[rr[e]][ro[e]];
  return 0;
}

/* multiroot slot of every edge, in the deterministic gather order
 * (oracle.cpp:115-139). slot[e] is indexed by the ORIGINAL edge order. */
static void slots(int64_t ne, const int32_t* rr, const int64_t* ro, const int32_t* lr,
                  const int64_t* li, int nranks, const int64_t* nroots, int64_t* slot_of) {
  int64_t** next = (int64_t**)calloc((size_t)nranks, sizeof(int64_t*));
  for (int r = 0; r < nranks; ++r) next[r] = (int64_t*)calloc((size_t)nroots[r] + 1, sizeof(int64_t));
  for (int64_t e = 0; e < ne; ++e) ++next[rr[e]][ro[e] + 1];
  for (int r = 0; r < nranks; ++r)
    for (int64_t i = 0; i < nroots[r]; ++i) next[r][i + 1] += next[r][i];
  key_t_* k = sorted_keys(ne, rr, ro, lr, li);
  for (int64_t s = 0; s < ne; ++s) {
    const int64_t e = k[s].id;
    slot_of[e] = next[rr[e]][ro[e]]++;
  }
  for (int r = 0; r < nranks; ++r) free(next[r]);
  free(next);
  free(k);
}

int oracle_gather(int64_t ne, const int32_t* rr, const int64_t* ro, const int32_t* lr,
                  const int64_t* li, int nranks, const int64_t* nroots, int kind, int64_t bl,
                  char* const* leafdata, char* const* multiroot) {
  const size_t ub = kind_size(kind) * (size_t)bl;
  int64_t* s = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne ? ne : 1));
  slots(ne, rr, ro, lr, li, nranks, nroots, s);
  for (int64_t e = 0; e < ne; ++e)
    memcpy(multiroot[rr[e]] + (size_t)s[e] * ub, leafdata[lr[e]] + (size_t)li[e] * ub, ub);
  free(s);
  return 0;
}

int oracle_scatter(int64_t ne, const int32_t* rr, const int64_t* ro, const int32_t* lr,
                   const int64_t* li, int nranks, const int64_t* nroots, int kind, int64_t bl,
                   char* const* multiroot, char* const* leafdata) {
  const size_t ub = kind_size(kind) * (size_t)bl;
  int64_t* s = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne ? ne : 1));
  slots(ne, rr, ro, lr, li, nranks, nroots, s);
  for (int64_t e = 0; e < ne; ++e)
    memcpy(leafdata[lr[e]] + (size_t)li[e] * ub, multiroot[rr[e]] + (size_t)s[e] * ub, ub);
  free(s);
  return 0;
}
