/* TEST INFRASTRUCTURE ONLY — see oracle.h.  Plain-C restatement of the
 * reference hot paths; every function cites the reference lines it follows.
 * Compiled with -ffp-contract=off semantics (no FMA on x86-64 SSE anyway). */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ST_OK 0
#define ST_INVALID (-1)
#define ST_UNKNOWN_TABLE (-5)

static const uint64_t kGamma = 0x9E3779B97F4A7C15ULL; /* inc/rng.hpp:25 */
static const uint64_t kProfileStream = 0x70726f66ULL;  /* profiler.cpp:29 */

/* inc/rng.hpp:27-31 — SplitMix64 finalizer */
uint64_t or_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* inc/rng.hpp:61-64 */
uint64_t or_derive_stream(uint64_t master, uint64_t a, uint64_t b) {
  uint64_t s = or_mix64(master ^ (kGamma * (a + 1)));
  return or_mix64(s ^ (0xD1B54A32D192ED03ULL * (b + 1)));
}

/* inc/rng.hpp:38-44: first next_double() of a fresh stream */
static double first_double(uint64_t seed) {
  uint64_t st = seed + kGamma;
  return (double)(or_mix64(st) >> 11) * 0x1.0p-53;
}

/* inc/workload.hpp:28-31 */
int or_hash_value(uint64_t raw, uint64_t hash_size, uint32_t* out) {
  if (hash_size == 0) return ST_INVALID;
  *out = (uint32_t)(or_mix64(raw) % hash_size);
  return ST_OK;
}

int or_hash_batch(const uint64_t* raw, uint64_t n, uint64_t hash_size,
                  uint32_t* out) {
  if (hash_size == 0) return ST_INVALID;
  for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)(or_mix64(raw[i]) % hash_size);
  return ST_OK;
}

static int table_index(uint32_t J, const uint32_t* table_ids, uint32_t id) {
  for (uint32_t j = 0; j < J; ++j)
    if (table_ids[j] == id) return (int)j;
  return -1;
}

/* core/src/profiler.cpp:60-112 */
int or_profile_counts(uint32_t J, const uint32_t* table_ids,
                      const uint64_t* hash_sizes, uint64_t num_samples,
                      uint64_t R, const uint64_t* rec_sample,
                      const uint32_t* rec_table, const uint64_t* rec_offset,
                      const uint32_t* rec_len, const uint32_t* ids,
                      const uint64_t* raw_ids, double rate, uint64_t seed,
                      uint64_t* counts, uint64_t* present, uint64_t* accesses,
                      uint64_t* selected_count) {
  if (num_samples < 1 || J == 0) return ST_INVALID;         /* :62-63 */
  if (!(rate > 0.0 && rate <= 1.0)) return ST_INVALID;       /* :64-65 */
  unsigned char* sel = (unsigned char*)malloc(num_samples);
  uint64_t nsel = 0;
  for (uint64_t s = 0; s < num_samples; ++s) {               /* :68-74 */
    sel[s] = rate >= 1.0 ||
             first_double(or_derive_stream(seed, s, kProfileStream)) < rate;
    nsel += sel[s];
  }
  if (nsel == 0) { free(sel); return ST_INVALID; }           /* :75-76 */
  uint64_t* base = (uint64_t*)malloc(sizeof(uint64_t) * J);
  uint64_t acc = 0;
  for (uint32_t j = 0; j < J; ++j) { base[j] = acc; acc += hash_sizes[j]; present[j] = 0; accesses[j] = 0; }
  int st = ST_OK;
  for (uint64_t r = 0; r < R; ++r) {                          /* :101-112 */
    if (!sel[rec_sample[r]]) continue;
    int j = table_index(J, table_ids, rec_table[r]);
    if (j < 0) { st = ST_UNKNOWN_TABLE; break; }
    present[j] += 1;
    accesses[j] += rec_len[r];
    uint64_t* c = counts + base[j];
    for (uint64_t i = rec_offset[r]; i < rec_offset[r] + rec_len[r]; ++i) {
      uint64_t row = raw_ids ? or_mix64(raw_ids[i]) % hash_sizes[j] : ids[i];
      c[row] += 1;
    }
  }
  if (selected_count) *selected_count = nsel;
  free(base);
  free(sel);
  return st;
}

typedef struct { uint64_t count; uint32_t row; } ranked_t;

static int cmp_ranked(const void* a, const void* b) {       /* :136-139 */
  const ranked_t* x = (const ranked_t*)a;
  const ranked_t* y = (const ranked_t*)b;
  if (x->count != y->count) return x->count > y->count ? -1 : 1;
  return x->row < y->row ? -1 : (x->row > y->row);
}

/* core/src/profiler.cpp:31-45 — integer ICDF walk over sorted counts */
static void icdf_from_sorted(const uint64_t* sorted, uint64_t total,
                             uint64_t* icdf) {
  uint64_t prefix = 0, k = 0;
  icdf[0] = 0;
  for (int i = 1; i <= 100; ++i) {
    while (prefix * 100 < (uint64_t)i * total) prefix += sorted[k++];
    icdf[i] = k;
  }
}

/* core/src/profiler.cpp:114-159 */
int or_rank_table(const uint64_t* counts, uint64_t H, uint64_t total,
                  uint32_t* rows_by_rank, double* cdf, uint64_t* icdf101,
                  uint64_t* distinct) {
  uint64_t n = 0;
  for (uint64_t r = 0; r < H; ++r) n += counts[r] != 0;
  ranked_t* rk = (ranked_t*)malloc(sizeof(ranked_t) * (n ? n : 1));
  n = 0;
  for (uint64_t r = 0; r < H; ++r)
    if (counts[r]) { rk[n].count = counts[r]; rk[n].row = (uint32_t)r; ++n; }
  qsort(rk, n, sizeof(ranked_t), cmp_ranked);
  uint64_t* sorted = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  uint64_t cum = 0;
  for (uint64_t r = 0; r < n; ++r) {
    sorted[r] = rk[r].count;
    rows_by_rank[r] = rk[r].row;
    cum += rk[r].count;
    cdf[r] = (double)cum / (double)total;
  }
  if (total == 0) memset(icdf101, 0, 101 * sizeof(uint64_t));
  else icdf_from_sorted(sorted, total, icdf101);
  *distinct = n;
  free(sorted);
  free(rk);
  return ST_OK;
}

static int cmp_u64_desc(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x > y ? -1 : (x < y);
}

/* core/src/profiler.cpp:49-58 */
int or_build_icdf(const uint64_t* counts, uint64_t n, uint64_t* icdf101) {
  uint64_t total = 0;
  for (uint64_t i = 0; i < n; ++i) total += counts[i];
  if (total == 0) return ST_INVALID;
  uint64_t* s = (uint64_t*)malloc(sizeof(uint64_t) * n);
  memcpy(s, counts, sizeof(uint64_t) * n);
  qsort(s, n, sizeof(uint64_t), cmp_u64_desc);
  icdf_from_sorted(s, total, icdf101);
  free(s);
  return ST_OK;
}

/* core/src/remap.cpp:40-105 */
int or_build_remap(uint64_t hash_size, uint64_t hbm_rows,
                   const uint32_t* rows_by_rank, uint64_t distinct,
                   int omit_unaccessed, int32_t* entries,
                   uint64_t* slow_rows_allocated) {
  const int32_t kUnset = INT32_MIN;
  if (hash_size > 0x7FFFFFFFULL) return ST_INVALID;          /* :42-46 */
  if (hbm_rows > hash_size) return ST_INVALID;               /* :47-51 */
  for (uint64_t r = 0; r < hash_size; ++r) entries[r] = kUnset;
  uint64_t ranked = hbm_rows < distinct ? hbm_rows : distinct;
  for (uint64_t r = 0; r < ranked; ++r) entries[rows_by_rank[r]] = (int32_t)r;
  uint64_t fast_next = ranked;                               /* :71-78 */
  for (uint64_t row = 0; row < hash_size && fast_next < hbm_rows; ++row)
    if (entries[row] == kUnset) entries[row] = (int32_t)fast_next++;
  uint64_t slow_next = 0;
  if (omit_unaccessed) {                                     /* :85-96 */
    unsigned char* acc = (unsigned char*)calloc(hash_size ? hash_size : 1, 1);
    for (uint64_t r = 0; r < distinct; ++r) acc[rows_by_rank[r]] = 1;
    for (uint64_t row = 0; row < hash_size; ++row)
      if (entries[row] == kUnset && acc[row])
        entries[row] = (int32_t)(-(int64_t)(slow_next++) - 1);
    *slow_rows_allocated = slow_next;
    for (uint64_t row = 0; row < hash_size; ++row)
      if (entries[row] == kUnset)
        entries[row] = (int32_t)(-(int64_t)(slow_next++) - 1);
    free(acc);
  } else {                                                   /* :97-103 */
    for (uint64_t row = 0; row < hash_size; ++row)
      if (entries[row] == kUnset)
        entries[row] = (int32_t)(-(int64_t)(slow_next++) - 1);
    *slow_rows_allocated = slow_next;
  }
  return ST_OK;
}

/* core/src/simulator.cpp:72-94 */
int or_simulate_counts(uint32_t J, const uint32_t* table_ids, uint64_t R,
                       const uint64_t* rec_sample, const uint32_t* rec_table,
                       const uint64_t* rec_offset, const uint32_t* rec_len,
                       const uint32_t* ids, const uint32_t* table_gpu,
                       const int32_t* const* remaps, uint32_t num_gpus,
                       uint64_t sample_limit, uint64_t* hbm_count,
                       uint64_t* uvm_count, uint64_t* table_fast,
                       uint64_t* table_total) {
  for (uint32_t g = 0; g < num_gpus; ++g) hbm_count[g] = uvm_count[g] = 0;
  for (uint32_t j = 0; j < J; ++j) table_fast[j] = table_total[j] = 0;
  for (uint64_t r = 0; r < R; ++r) {
    if (rec_sample[r] >= sample_limit) continue;
    int j = table_index(J, table_ids, rec_table[r]);
    if (j < 0) return ST_UNKNOWN_TABLE;
    uint64_t fast = 0;
    for (uint64_t i = rec_offset[r]; i < rec_offset[r] + rec_len[r]; ++i)
      fast += remaps[j][ids[i]] >= 0;
    hbm_count[table_gpu[j]] += fast;
    uvm_count[table_gpu[j]] += rec_len[r] - fast;
    table_fast[j] += fast;
    table_total[j] += rec_len[r];
  }
  return ST_OK;
}

float or_init_weight(uint64_t seed, uint32_t table_id, uint64_t row,
                     uint32_t d, float scale) {
  uint64_t u = or_mix64(or_derive_stream(seed, table_id, row) + d) >> 40;
  float x = (float)u * 0x1.0p-24f - 0.5f;
  return x * scale;
}

void or_init_table(uint64_t seed, uint32_t table_id, uint64_t H, uint32_t D,
                   float scale, float* W) {
  for (uint64_t r = 0; r < H; ++r)
    for (uint32_t d = 0; d < D; ++d)
      W[r * D + d] = or_init_weight(seed, table_id, r, d, scale);
}

int or_emb_forward(uint32_t T, uint64_t B, const uint32_t* D,
                   const uint64_t* col_off, uint64_t out_stride,
                   const uint64_t* offsets, const uint32_t* indices,
                   const float* const* W, float* out) {
  for (uint32_t t = 0; t < T; ++t) {
    for (uint64_t b = 0; b < B; ++b) {
      float* o = out + b * out_stride + col_off[t];
      for (uint32_t d = 0; d < D[t]; ++d) o[d] = 0.0f;
      for (uint64_t l = offsets[t * B + b]; l < offsets[t * B + b + 1]; ++l) {
        const float* w = W[t] + (uint64_t)indices[l] * D[t];
        for (uint32_t d = 0; d < D[t]; ++d) o[d] = o[d] + w[d];
      }
    }
  }
  return ST_OK;
}

/* Lanes per row and the per-lane / xor-butterfly order of the kernel's
 * sum-of-squares (paper_2201_10095_b200/csrc/emb_bwd.cuh). */
static uint32_t lanes_for(uint32_t D) {
  uint32_t v = D / 4, L = 1;
  while (L < v && L < 32) L <<= 1;
  return L;
}

static float rowwise_sumsq(const float* g, uint32_t D) {
  uint32_t L = lanes_for(D), V = D / 4;
  float part[32];
  for (uint32_t l = 0; l < L; ++l) {
    float s = 0.0f;
    for (uint32_t v = l; v < V; v += L)
      for (int k = 0; k < 4; ++k) {
        float x = g[4 * v + k];
        float sq = x * x;
        s = s + sq;
      }
    part[l] = s;
  }
  for (uint32_t off = L / 2; off >= 1; off >>= 1) {
    float nxt[32];
    for (uint32_t l = 0; l < L; ++l) nxt[l] = part[l] + part[l ^ off];
    memcpy(part, nxt, sizeof(float) * L);
  }
  return part[0];
}

/* One lookup of the batch: global key = key_base[t] + storage slot (key_base =
 * sum of earlier tables' hash sizes), l = position in the table-major index
 * list. */
typedef struct { uint64_t key; uint64_t l; } lk_t;
static int cmp_lk(const void* a, const void* b) {
  const lk_t* x = (const lk_t*)a;
  const lk_t* y = (const lk_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->l < y->l ? -1 : (x->l > y->l);
}

#define OR_CHUNK 32 /* csrc/emb_bwd.cuh kChunk (positions per piece) */
#define OR_GROUP 64 /* csrc/emb_bwd.cuh kGroupPieces (pieces per group) */

int or_emb_backward(uint32_t T, uint64_t B, const uint32_t* D,
                    const uint64_t* H, const uint64_t* col_off,
                    uint64_t grad_stride, const uint64_t* offsets,
                    const uint32_t* indices, const float* grad_out, int opt,
                    float lr, float eps, float* const* W,
                    float* const* momentum, const int32_t* const* remap,
                    const uint64_t* hbm_rows) {
  const uint64_t L = offsets[(uint64_t)T * B];
  if (L == 0) return ST_OK;
  uint64_t* kb = (uint64_t*)malloc(sizeof(uint64_t) * (T + 1));
  kb[0] = 0;
  for (uint32_t t = 0; t < T; ++t) kb[t + 1] = kb[t] + H[t];
  lk_t* lk = (lk_t*)malloc(sizeof(lk_t) * L);
  uint64_t* bag = (uint64_t*)malloc(sizeof(uint64_t) * L);
  uint32_t* tab = (uint32_t*)malloc(sizeof(uint32_t) * L);
  for (uint32_t t = 0; t < T; ++t)
    for (uint64_t b = 0; b < B; ++b)
      for (uint64_t l = offsets[t * B + b]; l < offsets[t * B + b + 1]; ++l) {
        if (indices[l] >= H[t]) { free(kb); free(lk); free(bag); free(tab); return ST_INVALID; }
        uint64_t slot = indices[l];
        if (remap) {
          const int32_t e = remap[t][indices[l]];
          slot = e >= 0 ? (uint64_t)e : hbm_rows[t] + (uint64_t)(-(int64_t)e - 1);
          if (slot >= H[t]) { free(kb); free(lk); free(bag); free(tab); return ST_INVALID; }
        }
        lk[l].key = kb[t] + slot;
        lk[l].l = l;
        bag[l] = b;
        tab[l] = t;
      }
  qsort(lk, L, sizeof(lk_t), cmp_lk); /* stable by construction (l breaks ties) */
  uint32_t dmax = 0;
  for (uint32_t t = 0; t < T; ++t) dmax = D[t] > dmax ? D[t] : dmax;
  float* g = (float*)malloc(sizeof(float) * dmax);
  float* piece = (float*)malloc(sizeof(float) * dmax);
  float* gs = (float*)malloc(sizeof(float) * dmax);
  uint64_t i = 0;
  while (i < L) {
    const uint64_t key = lk[i].key;
    const uint32_t t = tab[lk[i].l];
    const uint32_t row = indices[lk[i].l]; /* the remap is a bijection: one row per slot */
    const uint32_t d = D[t];
    uint64_t e = i;
    while (e < L && lk[e].key == key) ++e;
    /* The kernel's reduction tree (csrc/emb_bwd.cuh), anchored at the
     * segment's first sorted position i, length L = e - i: pieces of
     * OR_CHUNK positions from i, each summed in sorted order from +0.0f; for
     * L <= OR_CHUNK the single piece is g.  Otherwise groups of OR_GROUP
     * consecutive pieces are added left to right (first piece as the
     * accumulator) and g = the group sums left to right (first as the
     * accumulator). */
    int first_group = 1;
    uint64_t p = i;
    while (p < e) {
      uint64_t ge = p + (uint64_t)OR_CHUNK * OR_GROUP;
      if (ge > e) ge = e;
      int first_piece = 1;
      for (uint64_t q0 = p; q0 < ge; q0 += OR_CHUNK) {
        uint64_t pe = q0 + OR_CHUNK;
        if (pe > ge) pe = ge;
        for (uint32_t k = 0; k < d; ++k) piece[k] = 0.0f;
        for (uint64_t q = q0; q < pe; ++q) {
          const float* go = grad_out + bag[lk[q].l] * grad_stride + col_off[t];
          for (uint32_t k = 0; k < d; ++k) piece[k] = piece[k] + go[k];
        }
        if (first_piece) memcpy(gs, piece, sizeof(float) * d);
        else for (uint32_t k = 0; k < d; ++k) gs[k] = gs[k] + piece[k];
        first_piece = 0;
      }
      if (first_group) memcpy(g, gs, sizeof(float) * d);
      else for (uint32_t k = 0; k < d; ++k) g[k] = g[k] + gs[k];
      first_group = 0;
      p = ge;
    }
    float* w = W[t] + (uint64_t)row * d;
    if (opt == 0) {
      for (uint32_t k = 0; k < d; ++k) {
        float step = lr * g[k];
        w[k] = w[k] - step;
      }
    } else {
      float s = rowwise_sumsq(g, d);
      float m = momentum[t][row] + s / (float)d;
      momentum[t][row] = m;
      float mult = lr / (sqrtf(m) + eps);
      for (uint32_t k = 0; k < d; ++k) {
        float step = mult * g[k];
        w[k] = w[k] - step;
      }
    }
    i = e;
  }
  free(gs);
  free(piece);
  free(g);
  free(tab);
  free(bag);
  free(lk);
  free(kb);
  return ST_OK;
}
