/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for parity tests, smoke() and
 * bench.py's cpu_baseline leg.  Never linked into or called by the product
 * path (paper_1111_1373_b200/), which fails loudly without its CUDA library.
 *
 * A plain-C restatement of the reference "spectree" algorithms on the
 * classification hot path.  Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj/core).  It is pinned two
 * ways (tests/test_oracle.py):
 *   - against SURVEY.md Appendix A golden hashes (computed with the
 *     reference itself) for every canonical config, and
 *   - against the compiled reference (oracle/_ref, built by oracle/Makefile
 *     from the unmodified sources) on fuzz seeds, when that build exists.
 *
 * Node layout: 16 bytes {u32 attribute, f32 threshold, u32 child, u32 class}
 * (include/spectree/tree.hpp:43-55).  kNoClass = 0xFFFFFFFF (tree.hpp:15-16).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ST_NO_CLASS 0xFFFFFFFFu

typedef struct {
  uint32_t attribute;
  float threshold;
  uint32_t child;
  uint32_t class_id;
} or_node;

/* ---------------------------------------------------------------------- */
/* std::mt19937_64 (the reference draws from it: synthetic.cpp:97,157)    */
/* ---------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt64_next(mt64* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* bounded draw: (rng() * bound) >> 64 (synthetic.cpp:20-23, dataset.cpp:52-55) */
static uint64_t bounded(mt64* r, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)mt64_next(r) * bound) >> 64);
}

/* ---------------------------------------------------------------------- */
/* generate_synthetic_tree (synthetic.cpp:82-154)                          */
/* ---------------------------------------------------------------------- */
#define GRID_BITS 23u /* kGridBits synthetic.cpp:17 */
#define GRID_SIZE (1u << GRID_BITS)

typedef struct {
  uint32_t attribute;
  float threshold;
  int32_t left, right; /* -1 = none */
  int64_t class_val;   /* -1 = none */
} lnode;

typedef struct {
  int32_t node;
  uint32_t depth;
  uint32_t* lo; /* arity entries, owned */
  uint32_t* hi;
} gleaf;

typedef struct {
  lnode* v;
  size_t n, cap;
} lvec;

static int32_t lvec_push(lvec* L) {
  if (L->n == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 64;
    L->v = (lnode*)realloc(L->v, L->cap * sizeof(lnode));
  }
  lnode z = {0, 0.0f, -1, -1, -1};
  L->v[L->n] = z;
  return (int32_t)L->n++;
}

static int splittable(const gleaf* g, uint32_t arity) { /* synthetic.cpp:34-41 */
  for (uint32_t a = 0; a < arity; ++a)
    if (g->hi[a] - g->lo[a] >= 2) return 1;
  return 0;
}

/* pick_wide_attribute (synthetic.cpp:67-80); returns arity on exhaustion */
static uint32_t pick_wide(const gleaf* g, uint32_t arity, mt64* rng, uint32_t* scratch) {
  uint32_t nw = 0;
  for (uint32_t a = 0; a < arity; ++a)
    if (g->hi[a] - g->lo[a] >= 2) scratch[nw++] = a;
  if (nw == 0) return arity;
  return scratch[bounded(rng, nw)];
}

/* split_leaf (synthetic.cpp:46-65): the leaf becomes a split at its box
 * midpoint; `left` reuses the leaf's slot, `right` is returned. */
static void split_leaf(lvec* L, gleaf* g, uint32_t attribute, uint32_t arity, gleaf* right) {
  uint32_t mid = g->lo[attribute] + (g->hi[attribute] - g->lo[attribute]) / 2;
  int32_t l = lvec_push(L);
  int32_t r = lvec_push(L);
  lnode* node = &L->v[g->node];
  node->class_val = -1;
  node->attribute = attribute;
  node->threshold = (float)mid / (float)GRID_SIZE;
  node->left = l;
  node->right = r;
  right->node = r;
  right->depth = g->depth + 1;
  right->lo = (uint32_t*)malloc(arity * 4);
  right->hi = (uint32_t*)malloc(arity * 4);
  memcpy(right->lo, g->lo, arity * 4);
  memcpy(right->hi, g->hi, arity * 4);
  right->lo[attribute] = mid;
  g->node = l;
  g->depth += 1;
  g->hi[attribute] = mid;
}

/* Returns the node count (> 0) and writes *out (malloc'd, caller frees);
 * returns 0 on an infeasible shape (the reference throws ArgumentError). */
uint32_t or_gen_tree(uint32_t depth, uint32_t leaf_count, uint32_t arity,
                     uint32_t class_count, uint64_t seed, or_node** out) {
  *out = NULL;
  if (arity == 0 || class_count == 0) return 0;
  if (depth == 0) {
    if (leaf_count != 1) return 0;
  } else {
    if (leaf_count < depth + 1) return 0;
    if (depth < 32 && (uint64_t)leaf_count > (1ULL << depth)) return 0;
  }
  mt64 rng;
  mt64_seed(&rng, seed);
  lvec L = {0};
  int32_t root = lvec_push(&L);
  gleaf* leaves = (gleaf*)malloc(sizeof(gleaf) * (leaf_count + 1));
  size_t nleaves = 1;
  leaves[0].node = root;
  leaves[0].depth = 0;
  leaves[0].lo = (uint32_t*)calloc(arity, 4);
  leaves[0].hi = (uint32_t*)malloc(arity * 4);
  for (uint32_t a = 0; a < arity; ++a) leaves[0].hi[a] = GRID_SIZE;
  uint32_t* scratch = (uint32_t*)malloc(arity * 4);
  size_t* eligible = (size_t*)malloc(sizeof(size_t) * (leaf_count + 1));
  int ok = 1;

  /* spine: always re-split slot 0, which holds the newest left child
   * (synthetic.cpp:113-127) */
  for (uint32_t d = 0; d < depth && ok; ++d) {
    gleaf* g = &leaves[0];
    uint32_t preferred = d % arity;
    uint32_t attribute = preferred;
    if (!(g->hi[preferred] - g->lo[preferred] >= 2)) {
      attribute = pick_wide(g, arity, &rng, scratch);
      if (attribute == arity) { ok = 0; break; }
    }
    split_leaf(&L, g, attribute, arity, &leaves[nleaves]);
    nleaves++;
  }
  /* fill: split a uniformly drawn eligible leaf (synthetic.cpp:129-147) */
  while (ok && nleaves < leaf_count) {
    size_t ne = 0;
    for (size_t i = 0; i < nleaves; ++i)
      if (leaves[i].depth < depth && splittable(&leaves[i], arity)) eligible[ne++] = i;
    if (ne == 0) { ok = 0; break; }
    size_t pick = eligible[bounded(&rng, ne)];
    uint32_t attribute = pick_wide(&leaves[pick], arity, &rng, scratch);
    if (attribute == arity) { ok = 0; break; }
    split_leaf(&L, &leaves[pick], attribute, arity, &leaves[nleaves]);
    nleaves++;
  }
  if (ok) {
    /* classes in leaf-list order (synthetic.cpp:149-152) */
    for (size_t i = 0; i < nleaves; ++i)
      L.v[leaves[i].node].class_val = (int64_t)bounded(&rng, class_count);
  }
  for (size_t i = 0; i < nleaves; ++i) {
    free(leaves[i].lo);
    free(leaves[i].hi);
  }
  free(leaves);
  free(scratch);
  free(eligible);
  if (!ok) {
    free(L.v);
    return 0;
  }
  /* encode_breadth_first (tree.cpp:72-113) */
  or_node* nodes = (or_node*)malloc(sizeof(or_node) * L.n);
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * L.n);
  size_t qn = 1;
  queue[0] = root;
  uint32_t child_counter = 1;
  for (size_t i = 0; i < qn; ++i) {
    const lnode* nd = &L.v[queue[i]];
    or_node e;
    if (nd->left < 0) { /* leaf: self-loop, +inf, class */
      e.attribute = 0;
      e.threshold = INFINITY;
      e.child = (uint32_t)i;
      e.class_id = (uint32_t)nd->class_val;
    } else {
      e.attribute = nd->attribute;
      e.threshold = nd->threshold;
      e.child = child_counter;
      e.class_id = ST_NO_CLASS;
      queue[qn++] = nd->left;
      queue[qn++] = nd->right;
      child_counter += 2;
    }
    nodes[i] = e;
  }
  free(queue);
  free(L.v);
  *out = nodes;
  return (uint32_t)qn;
}

void or_free(void* p) { free(p); }

/* ---------------------------------------------------------------------- */
/* generate_synthetic_dataset (synthetic.cpp:156-182)                      */
/* ---------------------------------------------------------------------- */
void or_gen_dataset(uint64_t count, uint32_t arity, uint64_t seed, int gaussian, float* out) {
  mt64 rng;
  mt64_seed(&rng, seed);
  const uint64_t total = count * (uint64_t)arity;
  if (!gaussian) {
    for (uint64_t i = 0; i < total; ++i) out[i] = (float)(mt64_next(&rng) >> 40) * 0x1p-24f;
  } else {
    const double pi = 3.141592653589793238462643383279502884; /* std::numbers::pi */
    for (uint64_t i = 0; i < total; ++i) {
      const double u1 = ((double)(mt64_next(&rng) >> 40) + 1.0) * 0x1p-24;
      const double u2 = (double)(mt64_next(&rng) >> 40) * 0x1p-24;
      const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * pi * u2);
      out[i] = (float)(0.5 + 0.15 * z);
    }
  }
}

/* Fisher-Yates record permutation (dataset.cpp:59-74); writes the order. */
void or_shuffle_order(uint64_t count, uint64_t seed, uint64_t* order) {
  for (uint64_t i = 0; i < count; ++i) order[i] = i;
  mt64 rng;
  mt64_seed(&rng, seed);
  for (uint64_t i = count; i > 1; --i) {
    uint64_t j = bounded(&rng, i);
    uint64_t t = order[i - 1];
    order[i - 1] = order[j];
    order[j] = t;
  }
}

/* ---------------------------------------------------------------------- */
/* hashes                                                                   */
/* ---------------------------------------------------------------------- */
static uint64_t fnv_mix(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = (const unsigned char*)p;
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* FNV-1a-64 over raw bytes (tree_fnv, labels_fnv) */
uint64_t or_fnv1a(const void* p, uint64_t n) { return fnv_mix(0xcbf29ce484222325ULL, p, n); }

/* dataset_checksum (dataset.cpp:76-93): arity(u32), count(u64), values */
uint64_t or_dataset_checksum(const float* x, uint64_t count, uint32_t arity) {
  uint64_t h = 0xcbf29ce484222325ULL;
  h = fnv_mix(h, &arity, 4);
  h = fnv_mix(h, &count, 8);
  return fnv_mix(h, x, count * arity * 4);
}

/* ---------------------------------------------------------------------- */
/* evaluators                                                               */
/* ---------------------------------------------------------------------- */
/* EncodedTree::max_attribute over ALL nodes incl. leaves (tree.cpp:47) */
uint32_t or_max_attribute(const or_node* nodes, uint32_t n) {
  uint32_t m = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (nodes[i].attribute > m) m = nodes[i].attribute;
  return m;
}

/* classify (eval_serial.cpp:21-29): i = child + (x[attr] > thr) until leaf */
static inline uint32_t classify(const or_node* nodes, const float* rec) {
  uint32_t i = 0;
  while (nodes[i].class_id == ST_NO_CLASS)
    i = nodes[i].child + (uint32_t)(rec[nodes[i].attribute] > nodes[i].threshold);
  return nodes[i].class_id;
}

/* eval_serial (eval_serial.cpp:33-41).  Returns 2 (ArgumentError) when
 * max_attribute >= arity (check_attribute_range, eval_serial.cpp:10-17). */
int or_eval_serial(const or_node* nodes, uint32_t n, const float* x, uint64_t m,
                   uint32_t arity, uint32_t* out) {
  if (or_max_attribute(nodes, n) >= arity) return 2;
  for (uint64_t r = 0; r < m; ++r) out[r] = classify(nodes, x + r * arity);
  return 0;
}

/* traversal_depths (eval_serial.cpp:77-93) */
int or_traversal_depths(const or_node* nodes, uint32_t n, const float* x, uint64_t m,
                        uint32_t arity, uint32_t* out) {
  if (or_max_attribute(nodes, n) >= arity) return 2;
  for (uint64_t r = 0; r < m; ++r) {
    const float* rec = x + r * arity;
    uint32_t i = 0, e = 0;
    while (nodes[i].class_id == ST_NO_CLASS) {
      i = nodes[i].child + (uint32_t)(rec[nodes[i].attribute] > nodes[i].threshold);
      ++e;
    }
    out[r] = e;
  }
  return 0;
}

/* Mapped-lane speculative evaluation, barrier-separated mode
 * (eval_speculative.cpp:127-204, mapped branch :151-155 and :170-181):
 * node-eval over internal nodes, then while root unresolved apply k
 * snapshot doublings.  iters/steps (nullable) receive SpeculativeStats. */
int or_eval_speculative(const or_node* nodes, uint32_t n, const float* x, uint64_t m,
                        uint32_t arity, uint32_t k, uint32_t* out, uint32_t* iters,
                        uint32_t* steps) {
  if (k == 0) return 2;
  if (or_max_attribute(nodes, n) >= arity) return 2;
  uint32_t* cur = (uint32_t*)malloc(4 * n);
  uint32_t* alt = (uint32_t*)malloc(4 * n);
  uint32_t* mapped = (uint32_t*)malloc(4 * n);
  uint32_t nm = 0;
  for (uint32_t i = 0; i < n; ++i) {
    cur[i] = alt[i] = i; /* identity-seeded (make_path_array :14-19) */
    if (nodes[i].class_id == ST_NO_CLASS) mapped[nm++] = i; /* processor_node_map */
  }
  for (uint64_t r = 0; r < m; ++r) {
    const float* rec = x + r * arity;
    for (uint32_t j = 0; j < nm; ++j) {
      const or_node* nd = &nodes[mapped[j]];
      cur[mapped[j]] = nd->child + (uint32_t)(rec[nd->attribute] > nd->threshold);
    }
    uint32_t it = 0, st = 0;
    while (nodes[cur[0]].class_id == ST_NO_CLASS) {
      for (uint32_t s = 0; s < k; ++s) {
        for (uint32_t j = 0; j < nm; ++j) alt[mapped[j]] = cur[cur[mapped[j]]];
        uint32_t* t = cur;
        cur = alt;
        alt = t;
        ++st;
      }
      ++it;
    }
    out[r] = nodes[cur[0]].class_id;
    if (iters) iters[r] = it;
    if (steps) steps[r] = st;
  }
  free(cur);
  free(alt);
  free(mapped);
  return 0;
}

/* Random-forest majority vote (no reference: SURVEY §8a row a13).  Per
 * sample, count each tree's eval_serial label; the winner is the class with
 * the highest count, smallest class id on ties.  Trees are concatenated in
 * `nodes` with tree t occupying [offsets[t], offsets[t+1]).  Classes must be
 * < n_classes. */
int or_eval_forest(const or_node* nodes, const uint64_t* offsets, uint32_t t_count,
                   const float* x, uint64_t m, uint32_t arity, uint32_t n_classes,
                   uint32_t* out) {
  for (uint32_t t = 0; t < t_count; ++t) {
    const or_node* tn = nodes + offsets[t];
    uint32_t tn_n = (uint32_t)(offsets[t + 1] - offsets[t]);
    if (or_max_attribute(tn, tn_n) >= arity) return 2;
    for (uint32_t i = 0; i < tn_n; ++i)
      if (tn[i].class_id != ST_NO_CLASS && tn[i].class_id >= n_classes) return 2;
  }
  uint32_t* counts = (uint32_t*)calloc(n_classes, 4);
  for (uint64_t r = 0; r < m; ++r) {
    const float* rec = x + r * arity;
    memset(counts, 0, 4 * n_classes);
    for (uint32_t t = 0; t < t_count; ++t) counts[classify(nodes + offsets[t], rec)]++;
    uint32_t best = 0;
    for (uint32_t c = 1; c < n_classes; ++c)
      if (counts[c] > counts[best]) best = c;
    out[r] = best;
  }
  free(counts);
  return 0;
}
