/*
 * kv_alloc_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference merged-block allocator
 * `seasim::UnifiedKvCache` (/root/reference/proj/include/seasim/kv_cache.hpp:46-267)
 * and its shape helpers (kv_cache.hpp:17-33).  Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline leg may load this code.
 *
 * Parity pins: tests/test_oracle_alloc.py replays the reference's own
 * known-answer tests (proj/tests/kv_cache_test.cpp:26-235) against this file,
 * and diffs seeded op streams against the reference itself compiled from
 * /root/reference into oracle/_ref/libref_kv.so (oracle/ref_kv.cpp).
 *
 * The std::set free list / per-model partial sets of the reference become
 * bitmaps scanned from a low-water hint; "lowest id first" is preserved.
 * Every double the reference accumulates is accumulated here with the same
 * operations in the same order (fragmentation quirk Q1 included).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define SKVO_MAX_MODELS 64

enum { SKVO_OK = 0, SKVO_FULL = 1, SKVO_ECONFIG = -1, SKVO_EVALIDATION = -2, SKVO_ELOGIC = -3 };

typedef struct {
  int model;
  long tokens;
  int nslots, cap;
  int32_t *pairs; /* (block, sub) interleaved, token order */
} skvo_entry;

typedef struct {
  uint64_t key;
  int32_t ent; /* -1 empty, -2 tombstone */
} skvo_hslot;

typedef struct skvo_cache {
  int M, tpb;
  size_t P;
  double merged;
  double native[SKVO_MAX_MODELS];
  int sub[SKVO_MAX_MODELS];
  size_t open[SKVO_MAX_MODELS];
  size_t nwords;
  uint64_t *freebits;            /* 1 = block on the free list */
  size_t free_count, free_hint;  /* hint: lowest word that may hold a set bit */
  uint64_t *partial;             /* [M][nwords], 1 = claimed & not full */
  size_t partial_hint[SKVO_MAX_MODELS];
  int *blk_model, *blk_occ;
  int maxsub;
  uint64_t *owner; /* [P][maxsub], 0 = empty (Q2: id 0 is indistinguishable) */
  /* request table: open addressing id -> entry index */
  skvo_hslot *ht;
  size_t ht_cap, ht_used;
  skvo_entry *ents;
  size_t ents_len, ents_cap;
  int32_t *free_ents;
  size_t free_ents_len, free_ents_cap;
  /* stats (kv_cache.hpp:260-266) */
  size_t current_entries;
  uint64_t peak_entries, stats_rw;
  double slot_frag, token_waste, peak_frag, peak_used;
} skvo_cache;

/* kv_cache.hpp:17-22 */
int skvo_native_block_bytes(int layers, int heads, int head_dim, int dtype_bytes, int tpb, int tp,
                            double *out) {
  if (tp == 0 || heads % tp != 0) return SKVO_ECONFIG;
  *out = (double)tpb * layers * 2.0 * (heads / tp) * head_dim * dtype_bytes;
  return SKVO_OK;
}

/* kv_cache.hpp:26-33 */
int skvo_plan_merged_shape(int M, const int *layers, const int *heads, const int *head_dim,
                           const int *dtype_bytes, int tpb, int tp, double *out) {
  if (M <= 0) return SKVO_ECONFIG;
  double merged = 0.0;
  for (int m = 0; m < M; ++m) {
    double nb;
    if (skvo_native_block_bytes(layers[m], heads[m], head_dim[m], dtype_bytes[m], tpb, tp, &nb))
      return SKVO_ECONFIG;
    if (nb > merged) merged = nb;
  }
  *out = merged;
  return SKVO_OK;
}

static uint64_t hmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static void ht_rehash(skvo_cache *c, size_t ncap) {
  skvo_hslot *old = c->ht;
  size_t ocap = c->ht_cap;
  c->ht = (skvo_hslot *)malloc(ncap * sizeof(skvo_hslot));
  for (size_t i = 0; i < ncap; ++i) c->ht[i].ent = -1;
  c->ht_cap = ncap;
  c->ht_used = 0;
  for (size_t i = 0; i < ocap; ++i) {
    if (old[i].ent < 0) continue;
    size_t h = hmix(old[i].key) & (ncap - 1);
    while (c->ht[h].ent != -1) h = (h + 1) & (ncap - 1);
    c->ht[h] = old[i];
    c->ht_used++;
  }
  free(old);
}

static long ht_find(const skvo_cache *c, uint64_t key) {
  size_t h = hmix(key) & (c->ht_cap - 1);
  for (;;) {
    const skvo_hslot *s = &c->ht[h];
    if (s->ent == -1) return -1;
    if (s->ent >= 0 && s->key == key) return (long)h;
    h = (h + 1) & (c->ht_cap - 1);
  }
}

static int32_t new_entry(skvo_cache *c) {
  int32_t e;
  if (c->free_ents_len) {
    e = c->free_ents[--c->free_ents_len];
  } else {
    if (c->ents_len == c->ents_cap) {
      c->ents_cap = c->ents_cap ? c->ents_cap * 2 : 64;
      c->ents = (skvo_entry *)realloc(c->ents, c->ents_cap * sizeof(skvo_entry));
    }
    e = (int32_t)c->ents_len++;
    c->ents[e].pairs = NULL;
    c->ents[e].cap = 0;
  }
  c->ents[e].model = -1;
  c->ents[e].tokens = 0;
  c->ents[e].nslots = 0;
  return e;
}

/* table_[id] — registers on first touch (kv_cache.hpp:106) */
static int32_t ht_get_or_insert(skvo_cache *c, uint64_t key) {
  long f = ht_find(c, key);
  if (f >= 0) return c->ht[f].ent;
  if ((c->ht_used + 1) * 2 > c->ht_cap) ht_rehash(c, c->ht_cap * 2);
  size_t h = hmix(key) & (c->ht_cap - 1);
  while (c->ht[h].ent >= 0) h = (h + 1) & (c->ht_cap - 1);
  if (c->ht[h].ent == -1) c->ht_used++;
  c->ht[h].key = key;
  c->ht[h].ent = new_entry(c);
  return c->ht[h].ent;
}

skvo_cache *skvo_create(int M, const int *layers, const int *heads, const int *head_dim,
                        const int *dtype_bytes, int tpb, int tp, size_t pool, int *status) {
  *status = SKVO_OK;
  if (M > SKVO_MAX_MODELS) { *status = SKVO_ECONFIG; return NULL; }
  double merged;
  if (skvo_plan_merged_shape(M, layers, heads, head_dim, dtype_bytes, tpb, tp, &merged)) {
    *status = SKVO_ECONFIG;
    return NULL;
  }
  skvo_cache *c = (skvo_cache *)calloc(1, sizeof(skvo_cache));
  c->M = M;
  c->tpb = tpb;
  c->P = pool;
  c->merged = merged;
  c->maxsub = 1;
  for (int m = 0; m < M; ++m) {
    skvo_native_block_bytes(layers[m], heads[m], head_dim[m], dtype_bytes[m], tpb, tp, &c->native[m]);
    c->sub[m] = (int)(merged / c->native[m]); /* kv_cache.hpp:62 */
    if (c->sub[m] > c->maxsub) c->maxsub = c->sub[m];
  }
  c->nwords = (pool + 63) / 64;
  c->freebits = (uint64_t *)calloc(c->nwords ? c->nwords : 1, 8);
  for (size_t b = 0; b < pool; ++b) c->freebits[b >> 6] |= 1ULL << (b & 63);
  c->free_count = pool;
  c->partial = (uint64_t *)calloc((c->nwords ? c->nwords : 1) * (size_t)M, 8);
  c->blk_model = (int *)malloc((pool ? pool : 1) * sizeof(int));
  c->blk_occ = (int *)calloc(pool ? pool : 1, sizeof(int));
  for (size_t b = 0; b < pool; ++b) c->blk_model[b] = -1;
  c->owner = (uint64_t *)calloc((pool ? pool : 1) * (size_t)c->maxsub, 8);
  c->ht_cap = 64;
  c->ht = (skvo_hslot *)malloc(c->ht_cap * sizeof(skvo_hslot));
  for (size_t i = 0; i < c->ht_cap; ++i) c->ht[i].ent = -1;
  return c;
}

void skvo_destroy(skvo_cache *c) {
  if (!c) return;
  for (size_t i = 0; i < c->ents_len; ++i) free(c->ents[i].pairs);
  free(c->ents);
  free(c->free_ents);
  free(c->ht);
  free(c->freebits);
  free(c->partial);
  free(c->blk_model);
  free(c->blk_occ);
  free(c->owner);
  free(c);
}

int skvo_sub_slots(const skvo_cache *c, int m) { return c->sub[m]; }
double skvo_merged_block_bytes(const skvo_cache *c) { return c->merged; }
size_t skvo_free_blocks(const skvo_cache *c) { return c->free_count; }
size_t skvo_allocated_blocks(const skvo_cache *c) { return c->P - c->free_count; }
size_t skvo_table_entries(const skvo_cache *c) { return c->current_entries; }
size_t skvo_native_blocks_for(const skvo_cache *c, long tokens) {
  return (size_t)((tokens + c->tpb - 1) / c->tpb); /* kv_cache.hpp:81-83 */
}
int skvo_registered(const skvo_cache *c, uint64_t id) { return ht_find(c, id) >= 0; }
size_t skvo_available_slots(const skvo_cache *c, int m) { /* kv_cache.hpp:88-90 */
  return c->open[m] + c->free_count * (size_t)c->sub[m];
}

/* kv_cache.hpp:92-99 */
int skvo_can_grow_to(const skvo_cache *c, uint64_t id, int m, long tokens) {
  size_t need = skvo_native_blocks_for(c, tokens), have = 0;
  long f = ht_find(c, id);
  if (f >= 0) have = (size_t)c->ents[c->ht[f].ent].nslots;
  if (need <= have) return 1;
  return skvo_available_slots(c, m) >= need - have;
}

/* kv_cache.hpp:184-189 */
static double entry_token_waste(const skvo_cache *c, const skvo_entry *e) {
  if (e->model < 0) return 0.0;
  const double cap_tokens = (double)e->nslots * c->tpb;
  const double per_token = c->native[e->model] / c->tpb;
  return (cap_tokens - (double)e->tokens) * per_token;
}

static size_t lowest_set(const uint64_t *bits, size_t nwords, size_t *hint) {
  for (size_t w = *hint; w < nwords; ++w) {
    if (bits[w]) {
      *hint = w;
      return w * 64 + (size_t)__builtin_ctzll(bits[w]);
    }
  }
  *hint = nwords;
  return (size_t)-1;
}

/* kv_cache.hpp:191-222 */
static int claim_slot(skvo_cache *c, skvo_entry *e, int m, uint64_t id) {
  c->token_waste -= entry_token_waste(c, e);
  int block, slot;
  uint64_t *pm = c->partial + (size_t)m * c->nwords;
  size_t pb = lowest_set(pm, c->nwords, &c->partial_hint[m]);
  if (pb != (size_t)-1) {
    block = (int)pb;
    uint64_t *own = c->owner + (size_t)block * c->maxsub;
    slot = 0;
    while (own[slot] != 0) ++slot;
    own[slot] = id;
    c->blk_occ[block]++;
    c->open[m]--;
    c->slot_frag -= c->native[m];
    if (c->blk_occ[block] == c->sub[m]) pm[block >> 6] &= ~(1ULL << (block & 63));
  } else {
    size_t fb = lowest_set(c->freebits, c->nwords, &c->free_hint);
    if (fb == (size_t)-1) return SKVO_ELOGIC; /* "claim_slot: pool exhausted" */
    block = (int)fb;
    c->freebits[fb >> 6] &= ~(1ULL << (fb & 63));
    c->free_count--;
    c->blk_model[block] = m;
    c->blk_occ[block] = 1;
    uint64_t *own = c->owner + (size_t)block * c->maxsub;
    for (int s = 0; s < c->maxsub; ++s) own[s] = 0;
    own[0] = id;
    slot = 0;
    c->open[m] += (size_t)(c->sub[m] - 1);
    c->slot_frag += c->merged - c->native[m];
    if (c->sub[m] > 1) {
      pm[block >> 6] |= 1ULL << (block & 63);
      if ((size_t)(block >> 6) < c->partial_hint[m]) c->partial_hint[m] = (size_t)(block >> 6);
    }
  }
  if (e->nslots == e->cap) {
    e->cap = e->cap ? e->cap * 2 : 8;
    e->pairs = (int32_t *)realloc(e->pairs, (size_t)e->cap * 2 * sizeof(int32_t));
  }
  e->pairs[2 * e->nslots] = block;
  e->pairs[2 * e->nslots + 1] = slot;
  e->nslots++;
  c->current_entries++;
  c->token_waste += entry_token_waste(c, e);
  return SKVO_OK;
}

/* kv_cache.hpp:224-240 */
static void release_slot(skvo_cache *c, int block, int slot, int m) {
  c->owner[(size_t)block * c->maxsub + slot] = 0;
  c->blk_occ[block]--;
  uint64_t *pm = c->partial + (size_t)m * c->nwords;
  if (c->blk_occ[block] == 0) {
    pm[block >> 6] &= ~(1ULL << (block & 63));
    c->open[m] -= (size_t)(c->sub[m] - 1);
    c->slot_frag -= c->merged - c->native[m];
    c->blk_model[block] = -1;
    c->freebits[block >> 6] |= 1ULL << (block & 63);
    c->free_count++;
    if ((size_t)(block >> 6) < c->free_hint) c->free_hint = (size_t)(block >> 6);
  } else {
    pm[block >> 6] |= 1ULL << (block & 63);
    if ((size_t)(block >> 6) < c->partial_hint[m]) c->partial_hint[m] = (size_t)(block >> 6);
    c->open[m]++;
    c->slot_frag += c->native[m];
  }
}

/* kv_cache.hpp:242-246 */
static void note_watermarks(skvo_cache *c) {
  if (c->current_entries > c->peak_entries) c->peak_entries = c->current_entries;
  double used = (double)(c->P - c->free_count);
  if (used > c->peak_used) c->peak_used = used;
  double frag = c->slot_frag + c->token_waste;
  if (frag > c->peak_frag) c->peak_frag = frag;
}

/* kv_cache.hpp:104-123.  Returns SKVO_OK (granted), SKVO_FULL (CacheFull -> false),
 * SKVO_EVALIDATION (negative tokens), SKVO_ELOGIC (model change / exhausted). */
int skvo_try_allocate(skvo_cache *c, uint64_t id, int m, long tokens) {
  if (tokens < 0) return SKVO_EVALIDATION;
  int32_t ei = ht_get_or_insert(c, id);
  skvo_entry *e = &c->ents[ei];
  if (e->nslots == 0) e->model = m;
  if (e->model != m) return SKVO_ELOGIC;
  const size_t need = skvo_native_blocks_for(c, tokens);
  if (need > (size_t)e->nslots && skvo_available_slots(c, m) < need - (size_t)e->nslots)
    return SKVO_FULL;
  c->token_waste -= entry_token_waste(c, e);
  while ((size_t)e->nslots < need) {
    int rc = claim_slot(c, e, m, id);
    if (rc) return rc;
  }
  if (tokens > e->tokens) {
    c->stats_rw += (uint64_t)(tokens - e->tokens);
    e->tokens = tokens;
  }
  c->token_waste += entry_token_waste(c, e);
  note_watermarks(c);
  return SKVO_OK;
}

/* kv_cache.hpp:126-134 */
int skvo_free_request(skvo_cache *c, uint64_t id) {
  long f = ht_find(c, id);
  if (f < 0) return SKVO_ELOGIC;
  int32_t ei = c->ht[f].ent;
  skvo_entry *e = &c->ents[ei];
  for (int i = 0; i < e->nslots; ++i) release_slot(c, e->pairs[2 * i], e->pairs[2 * i + 1], e->model);
  c->current_entries -= (size_t)e->nslots;
  c->token_waste -= entry_token_waste(c, e);
  c->ht[f].ent = -2; /* tombstone */
  if (c->free_ents_len == c->free_ents_cap) {
    c->free_ents_cap = c->free_ents_cap ? c->free_ents_cap * 2 : 64;
    c->free_ents = (int32_t *)realloc(c->free_ents, c->free_ents_cap * sizeof(int32_t));
  }
  c->free_ents[c->free_ents_len++] = ei;
  return SKVO_OK;
}

/* kv_cache.hpp:138-142 */
void skvo_record_context_read(skvo_cache *c, uint64_t id) {
  long f = ht_find(c, id);
  if (f < 0) return;
  c->stats_rw += (uint64_t)c->ents[c->ht[f].ent].nslots;
}

/* kv_cache.hpp:144-148.  Returns the entry count (pairs copied up to cap) or -1. */
long skvo_block_table(const skvo_cache *c, uint64_t id, int32_t *pairs, size_t cap) {
  long f = ht_find(c, id);
  if (f < 0) return SKVO_ELOGIC;
  const skvo_entry *e = &c->ents[c->ht[f].ent];
  size_t n = (size_t)e->nslots < cap ? (size_t)e->nslots : cap;
  if (pairs && n) memcpy(pairs, e->pairs, n * 2 * sizeof(int32_t));
  return e->nslots;
}

/* kv_cache.hpp:150-154 */
uint64_t skvo_owner_of(const skvo_cache *c, int block, int slot) {
  if (slot >= c->maxsub) return 0;
  if (c->blk_model[block] < 0) return 0; /* slot_owner cleared on release */
  if (slot >= c->sub[c->blk_model[block]]) return 0;
  return c->owner[(size_t)block * c->maxsub + slot];
}

int skvo_request_model(const skvo_cache *c, uint64_t id) {
  long f = ht_find(c, id);
  return f < 0 ? -1 : c->ents[c->ht[f].ent].model;
}
long skvo_request_tokens(const skvo_cache *c, uint64_t id) {
  long f = ht_find(c, id);
  return f < 0 ? -1 : c->ents[c->ht[f].ent].tokens;
}

double skvo_fragmentation_bytes(const skvo_cache *c) { return c->slot_frag + c->token_waste; }

/* CacheStats (kv_cache.hpp:35-40, 163-170) */
typedef struct {
  uint64_t block_table_entries, native_reads_writes;
  double internal_fragmentation_bytes, peak_utilization;
} skvo_stats;

void skvo_get_stats(const skvo_cache *c, skvo_stats *s) {
  s->block_table_entries = c->peak_entries;
  s->native_reads_writes = c->stats_rw;
  s->internal_fragmentation_bytes = c->peak_frag;
  s->peak_utilization = c->P == 0 ? 0.0 : c->peak_used / (double)c->P;
}

/* open_slots_ mirror (kv_cache.hpp:254), exposed for differential tests */
size_t skvo_open_slots(const skvo_cache *c, int m) { return c->open[m]; }

/* Replay driver for timing: applies n ops {kind,id,model,tokens}; kind 0=grow 1=free.
 * Returns the number of granted grows; -1 on a protocol error. */
typedef struct {
  int32_t kind, model;
  uint64_t id;
  int64_t tokens;
} skvo_op;

long skvo_replay(skvo_cache *c, const skvo_op *ops, size_t n) {
  long granted = 0;
  for (size_t i = 0; i < n; ++i) {
    if (ops[i].kind == 0) {
      int rc = skvo_try_allocate(c, ops[i].id, ops[i].model, (long)ops[i].tokens);
      if (rc == SKVO_OK) granted++;
      else if (rc != SKVO_FULL) return -1;
    } else {
      if (skvo_free_request(c, ops[i].id)) return -1;
    }
  }
  return granted;
}

/* ---- Split-scheme accounting (kv_cache.hpp:277-348) and compare_schemes (:352-369) ----
 * Per-layer-per-head blocks: each native block of model m costs L*H table
 * entries and every token touches L*H blocks.  All wastes are integer-valued
 * doubles (< 2^53), so the reference's std::map iteration order does not
 * change the sum; entries are visited in insertion order here. */
typedef struct {
  uint64_t id;
  int model, live;
  long blocks, tokens;
} skvo_split_ent;

int skvo_compare_schemes(int M, const int *layers, const int *heads, const int *head_dim,
                         const int *dtype_bytes, int tpb, int tp, const skvo_op *ops, size_t n,
                         size_t pool, double *out) {
  int st;
  skvo_cache *c = skvo_create(M, layers, heads, head_dim, dtype_bytes, tpb, tp, pool, &st);
  if (!c) return st;
  skvo_split_ent *se = (skvo_split_ent *)calloc(n ? n : 1, sizeof(skvo_split_ent));
  size_t nse = 0;
  uint64_t cur = 0, peak = 0, rw = 0;
  double frag = 0.0;
  int rc = SKVO_OK;
  for (size_t i = 0; i < n && rc == SKVO_OK; ++i) {
    const skvo_op *op = &ops[i];
    if (op->kind == 0) {
      int g = skvo_try_allocate(c, op->id, op->model, (long)op->tokens);
      if (g == SKVO_FULL) { rc = SKVO_EVALIDATION; break; } /* "pool too small" */
      if (g) { rc = g; break; }
      /* SplitCacheCounter::grow (:286-302) */
      size_t k = 0;
      while (k < nse && !(se[k].live && se[k].id == op->id)) ++k;
      if (k == nse) { se[nse].id = op->id; se[nse].live = 1; se[nse].blocks = 0; se[nse].tokens = 0; nse++; }
      se[k].model = op->model;
      const long need = (op->tokens + tpb - 1) / tpb;
      const uint64_t factor = (uint64_t)layers[op->model] * (uint64_t)heads[op->model];
      if (need > se[k].blocks) { cur += (uint64_t)(need - se[k].blocks) * factor; se[k].blocks = need; }
      if (op->tokens > se[k].tokens) { rw += (uint64_t)(op->tokens - se[k].tokens) * factor; se[k].tokens = op->tokens; }
      if (cur > peak) peak = cur;
      double waste = 0.0;
      for (size_t j = 0; j < nse; ++j) {
        if (!se[j].live) continue;
        const int mm = se[j].model;
        const double per_token = 2.0 * layers[mm] * heads[mm] * head_dim[mm] * dtype_bytes[mm];
        waste += ((double)se[j].blocks * tpb - se[j].tokens) * per_token;
      }
      if (waste > frag) frag = waste;
    } else {
      if (skvo_free_request(c, op->id)) { rc = SKVO_ELOGIC; break; }
      for (size_t j = 0; j < nse; ++j)
        if (se[j].live && se[j].id == op->id) {
          cur -= (uint64_t)se[j].blocks * (uint64_t)layers[se[j].model] * (uint64_t)heads[se[j].model];
          se[j].live = 0;
        }
    }
  }
  if (rc == SKVO_OK) {
    skvo_stats s;
    skvo_get_stats(c, &s);
    out[0] = (double)s.block_table_entries;
    out[1] = (double)s.native_reads_writes;
    out[2] = s.internal_fragmentation_bytes;
    out[3] = s.peak_utilization;
    out[4] = (double)peak;
    out[5] = (double)rw;
    out[6] = frag;
    out[7] = 0.0;
  }
  free(se);
  skvo_destroy(c);
  return rc;
}
