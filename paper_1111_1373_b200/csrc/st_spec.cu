// Speculative-decomposition kernel dispatch (K2 k_spec_ring / k_spec / k_spec_exact_cta).
#include "st_internal.cuh"

namespace sti {

// ---- speculative kernel dispatch -----------------------------------------
template <int A, int LOADER, bool WS, bool EXACT, int STEPS>
void launch_spec_k(const SpecArgs& sa, const Staging& stg, size_t smem, int dev, uint32_t bps,
                   cudaStream_t s) {
  auto fn = k_spec<A, LOADER, WS, EXACT, STEPS>;
  const uint64_t n_tiles = (sa.p.m + 31) / 32;
  const int blocks = blocks_for((const void*)fn, smem, dev, bps, n_tiles, stg.warps);
  clear_stale_error();
  fn<<<blocks, stg.warps * 32, smem, s>>>(sa, stg.tmap);
  check_launch();
}

// Fast path: the doubling count is a compile-time constant for the usual
// window heights (steps 0..3); EXACT (reference counters) and taller windows
// use a runtime count.
template <int A, int LOADER, bool WS>
void launch_spec_steps(const SpecArgs& sa, const Staging& stg, size_t smem, int dev, uint32_t bps,
                       cudaStream_t s) {
  if (sa.iters) return launch_spec_k<A, LOADER, WS, true, -1>(sa, stg, smem, dev, bps, s);
  switch (sa.smax) {
    case 0: return launch_spec_k<A, LOADER, WS, false, 0>(sa, stg, smem, dev, bps, s);
    case 1: return launch_spec_k<A, LOADER, WS, false, 1>(sa, stg, smem, dev, bps, s);
    case 2: return launch_spec_k<A, LOADER, WS, false, 2>(sa, stg, smem, dev, bps, s);
    case 3: return launch_spec_k<A, LOADER, WS, false, 3>(sa, stg, smem, dev, bps, s);
    default: return launch_spec_k<A, LOADER, WS, false, -1>(sa, stg, smem, dev, bps, s);
  }
}

template <int A, bool WS, int STEPS, int SR, bool CW = false, int RT = 1, int SL = 0, int L3 = 0>
void launch_spec_ring_k(const SpecRingArgs& ra, const Staging& stg, size_t smem, int dev,
                        uint32_t warps, cudaStream_t s) {
  auto fn = k_spec_ring<A, WS, STEPS, SR, CW, RT, SL, L3>;
  constexpr uint64_t R = L3 ? (L3 == 3 ? kTripleSlot * 3 / 2 : kTripleSlot) : 32 * RT;
  const uint64_t n_tiles = (ra.s.p.m + R - 1) / R;
  const int blocks = blocks_for((const void*)fn, smem, dev, 0, n_tiles * warps, warps);
  clear_stale_error();
  fn<<<blocks, warps * 32, smem, s>>>(ra, stg.tmap);
  check_launch();
}

template <int A, bool WS, int STEPS, bool CW = false>
void launch_spec_ring_sr(uint32_t sr, const SpecRingArgs& ra, const Staging& stg, size_t smem, int dev,
                         uint32_t warps, cudaStream_t s, int sl = 0) {
  // two record streams: shared window table and records inside one 128-byte row
  if constexpr (WS && (A == 8 || A == 16 || A == 32)) {
    if constexpr (CW) {
      if (sl == 1 && sr >= 2) {  // self-loop codes (WinTable::sl_*), predicated advance
        if (ra.tile_mult == 2) return launch_spec_ring_k<A, WS, STEPS, 2, CW, 2, 1>(ra, stg, smem, dev, warps, s);
        return launch_spec_ring_k<A, WS, STEPS, 2, CW, 1, 1>(ra, stg, smem, dev, warps, s);
      }
      if (sl == 3 && sr >= 2) {  // self-loop codes, fixed trip count
        if (ra.tile_mult == 0) {  // lane triples, 80- or 120-record slots (ra.triple 1 / 3)
          if (ra.triple == 3) return launch_spec_ring_k<A, WS, STEPS, 2, CW, 1, 3, 3>(ra, stg, smem, dev, warps, s);
          return launch_spec_ring_k<A, WS, STEPS, 2, CW, 1, 3, 1>(ra, stg, smem, dev, warps, s);
        }
        if (ra.tile_mult == 2) return launch_spec_ring_k<A, WS, STEPS, 2, CW, 2, 3>(ra, stg, smem, dev, warps, s);
        return launch_spec_ring_k<A, WS, STEPS, 2, CW, 1, 3>(ra, stg, smem, dev, warps, s);
      }
      if (sl == 2 && sr >= 2) {  // self-loop codes, branchy advance
        if (ra.tile_mult == 2) return launch_spec_ring_k<A, WS, STEPS, 2, CW, 2, 2>(ra, stg, smem, dev, warps, s);
        return launch_spec_ring_k<A, WS, STEPS, 2, CW, 1, 2>(ra, stg, smem, dev, warps, s);
      }
      if (sr >= 2 && ra.tile_mult == 2) return launch_spec_ring_k<A, WS, STEPS, 2, CW, 2>(ra, stg, smem, dev, warps, s);
    }
    if (sr >= 2) return launch_spec_ring_k<A, WS, STEPS, 2, CW>(ra, stg, smem, dev, warps, s);
  }
  return launch_spec_ring_k<A, WS, STEPS, 1, CW>(ra, stg, smem, dev, warps, s);
}

template <int A>
void launch_spec_ring(bool ws, uint32_t sr, bool cw, int sl, const SpecRingArgs& ra, const Staging& stg,
                      size_t smem, int dev, uint32_t warps, cudaStream_t s) {
  // 8-byte window entries (shared table, window loop)
  if (cw && sr != 0) {
    switch (ra.s.smax) {
      case 0: return launch_spec_ring_sr<A, true, 0, true>(sr, ra, stg, smem, dev, warps, s, sl);
      case 1: return launch_spec_ring_sr<A, true, 1, true>(sr, ra, stg, smem, dev, warps, s, sl);
      case 2: return launch_spec_ring_sr<A, true, 2, true>(sr, ra, stg, smem, dev, warps, s, sl);
      case 3: return launch_spec_ring_sr<A, true, 3, true>(sr, ra, stg, smem, dev, warps, s, sl);
      default: return launch_spec_ring_sr<A, true, -1, true>(sr, ra, stg, smem, dev, warps, s, sl);
    }
  }
  // one window, pointer jumping with self-loop leaf codes
  if (sr == 0 && ws && sl && ra.s.smax <= 5) {
    switch (ra.s.smax) {
      case 0: return launch_spec_ring_k<A, true, 0, 0, false, 1, 1>(ra, stg, smem, dev, warps, s);
      case 1: return launch_spec_ring_k<A, true, 1, 0, false, 1, 1>(ra, stg, smem, dev, warps, s);
      case 2: return launch_spec_ring_k<A, true, 2, 0, false, 1, 1>(ra, stg, smem, dev, warps, s);
      case 3: return launch_spec_ring_k<A, true, 3, 0, false, 1, 1>(ra, stg, smem, dev, warps, s);
      case 4: return launch_spec_ring_k<A, true, 4, 0, false, 1, 1>(ra, stg, smem, dev, warps, s);
      default: return launch_spec_ring_k<A, true, 5, 0, false, 1, 1>(ra, stg, smem, dev, warps, s);
    }
  }
  // the whole tree in one window (sr == 0): hoisted entry, independent
  // passes, the doubling count (<= 5 for <= 32 lanes) always compile-time so
  // the passes interleave
  if (sr == 0 && ws && ra.s.smax <= 5) {
    switch (ra.s.smax) {
      case 0: return launch_spec_ring_k<A, true, 0, 0>(ra, stg, smem, dev, warps, s);
      case 1: return launch_spec_ring_k<A, true, 1, 0>(ra, stg, smem, dev, warps, s);
      case 2: return launch_spec_ring_k<A, true, 2, 0>(ra, stg, smem, dev, warps, s);
      case 3: return launch_spec_ring_k<A, true, 3, 0>(ra, stg, smem, dev, warps, s);
      case 4: return launch_spec_ring_k<A, true, 4, 0>(ra, stg, smem, dev, warps, s);
      default: return launch_spec_ring_k<A, true, 5, 0>(ra, stg, smem, dev, warps, s);
    }
  }
  if (sr == 0) sr = 1;
#define ST_RING(WSV, ST) return launch_spec_ring_sr<A, WSV, ST>(sr, ra, stg, smem, dev, warps, s)
  if (ws) {
    switch (ra.s.smax) {
      case 0: ST_RING(true, 0);
      case 1: ST_RING(true, 1);
      case 2: ST_RING(true, 2);
      case 3: ST_RING(true, 3);
      default: ST_RING(true, -1);
    }
  }
  switch (ra.s.smax) {
    case 0: ST_RING(false, 0);
    case 1: ST_RING(false, 1);
    case 2: ST_RING(false, 2);
    case 3: ST_RING(false, 3);
    default: ST_RING(false, -1);
  }
#undef ST_RING
}

template <int A, int LOADER>
void launch_spec_t(bool win_shared, const SpecArgs& sa, const Staging& stg, size_t smem, int dev,
                   uint32_t bps, cudaStream_t s) {
  if (win_shared) return launch_spec_steps<A, LOADER, true>(sa, stg, smem, dev, bps, s);
  return launch_spec_steps<A, LOADER, false>(sa, stg, smem, dev, bps, s);
}

// speculative ring: tile slots beyond one per warp -- few where the walk is
// shared-memory bound (lane triples: a slot fewer buys a resident warp),
// more where the ring streams at HBM speed (one-window ballot, C2's 4-lane
// groups: more tiles in flight)
constexpr uint32_t kRingExtraTriple = 4, kRingExtra = 12;

// Lane triples apply to the fixed-trip loop over G = 4 three-node windows
// with TMA-staged records inside one 128-byte row.
// (8 / 16 attributes: 80-record slots of 2.5 / 5 KB; 32-attribute ones
// would take 10 KB and cost resident warps -- C2 +19 %).
static bool triple_ok(const st_geom& g, uint32_t G, const WinTable& wt, const float* x, uint64_t m, uint32_t a,
                      uint64_t ld, int layout) {
  return !(g.variant & ST_VAR_SPEC_QUAD) && G == 4 && wt.sl_ws == 3 && m >= kTripleSlot && (a == 8 || a == 16) &&
         tma_ok(x, m, a, ld, layout, 1);
}

void spec_geometry(const st_tree* t, const st_geom& g, uint32_t& G, uint32_t& H) {
  G = g.group_lanes;
  if (G == 0) {
    const uint32_t I = std::max<uint32_t>(1, t->info.internal);
    if (I <= 32) {
      // whole tree in one record group: the paper's Proc. 5 geometry
      // (15 internal nodes -> its half-warp of 16 lanes)
      G = 1;
      while (G < I) G *= 2;
    } else {
      // larger trees: 3-node windows in 4-lane groups (two levels per window,
      // one shfl doubling) measured fastest on C2 among genuine speculation
      G = 4;
    }
  }
  if (G > 32 || (G & (G - 1)) != 0)
    fail(ST_ERR_ARGUMENT, "group_lanes must be a power of two <= 32 on the GPU, got " +
                              std::to_string(g.group_lanes));
  H = g.window_levels;
  if (H == 0) {
    if (t->info.internal <= G) {
      // whole tree in one window: the paper's Proc. 5 geometry (mapped lanes)
      H = std::max<uint32_t>(1, t->info.depth);
    } else {
      // complete-level windows: largest H with 2^H - 1 <= G
      H = 1;
      while ((2u << H) - 1 <= G) ++H;
    }
  }
}

// Reference counters for trees with more than 32 internal nodes: CTA-scope
// whole-tree speculation (k_spec_exact_cta).
void eval_spec_exact_cta(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                         int layout, uint32_t k, uint32_t* labels, st_stats* stats, cudaStream_t s,
                         int dev) {
  st_tree::Dev& dv = t->device(dev);
  const DevProps pr = dev_props(dev);
  SpecExactArgs ea{};
  ea.p = pipe_args(x, m, a, ld, layout);
  ea.nodes = dv.wide;
  ea.map = dv.internal_map;
  ea.n = (uint32_t)t->nodes.size();
  ea.I = t->info.internal;
  ea.k = k ? k : 1;
  ea.labels = labels;
  ea.iters = stats->iterations;
  ea.steps = stats->doubling_steps;
  // the two path arrays (+ the root word) per CTA: shared memory when they
  // fit, else a per-CTA slice of a stream-ordered global buffer
  const bool global_bufs = 8ull * t->nodes.size() + 16 > pr.smem_optin;
  const size_t smem = global_bufs ? 0 : 8ull * t->nodes.size() + 16;
  const uint32_t threads = std::min<uint32_t>(1024, std::max<uint32_t>(32, (ea.I + 31) / 32 * 32));
  auto fn = k_spec_exact_cta<0>;
  static std::mutex mu;
  static std::map<int, bool> attr;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!attr.count(dev)) {
      CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)pr.smem_optin));
      attr[dev] = true;
    }
  }
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, (int)threads, smem));
  const uint64_t blocks = std::min<uint64_t>(m, (uint64_t)pr.sms * std::max(occ, 1));
  if (global_bufs) {
    const size_t bytes = (size_t)blocks * (2ull * t->nodes.size() + 1) * 4;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&ea.gbuf), bytes, s));
  }
  clear_stale_error();
  fn<<<(unsigned)blocks, threads, smem, s>>>(ea);
  check_launch();
  if (global_bufs) CK(cudaFreeAsync(ea.gbuf, s));
}

// The resident frame stream with the speculative kernel (st_frames.cu): the
// fixed-trip ring loop (G = 4 three-node windows, 8-byte self-loop tables)
// in k_spec_ring<..., FR = true>.
template <int A, int L3>
static void launch_spec_frames_k(const SpecRingArgs& ra, const Staging& stg, size_t smem, int dev,
                                 uint32_t warps, uint32_t max_ctas, cudaStream_t s) {
  auto fn = k_spec_ring<A, true, 1, 2, true, 1, 3, L3, true>;
  int blocks = blocks_for((const void*)fn, smem, dev, 0, ra.tpf * warps, warps);
  if (max_ctas) blocks = std::min<int>(blocks, (int)max_ctas);
  clear_stale_error();
  fn<<<blocks, warps * 32, smem, s>>>(ra, stg.tmap);
  check_launch();
}

static void launch_spec_frames(uint32_t a, uint32_t triple, const SpecRingArgs& ra, const Staging& stg, size_t smem,
                               int dev, uint32_t warps, uint32_t max_ctas, cudaStream_t s) {
  if (a == 8 && triple == 3) return launch_spec_frames_k<8, 3>(ra, stg, smem, dev, warps, max_ctas, s);
  if (a == 8 && triple == 1) return launch_spec_frames_k<8, 1>(ra, stg, smem, dev, warps, max_ctas, s);
  if (a == 8 && triple == 0) return launch_spec_frames_k<8, 0>(ra, stg, smem, dev, warps, max_ctas, s);
  if (a == 16 && triple == 1) return launch_spec_frames_k<16, 1>(ra, stg, smem, dev, warps, max_ctas, s);
  if (a == 16 && triple == 0) return launch_spec_frames_k<16, 0>(ra, stg, smem, dev, warps, max_ctas, s);
  if (a == 32 && triple == 0) return launch_spec_frames_k<32, 0>(ra, stg, smem, dev, warps, max_ctas, s);
  fail(ST_ERR_ARGUMENT, "speculative frame stream: no kernel for this arity / slot layout");
}

void eval_spec_device(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom& g, uint32_t* labels, st_stats* stats, cudaStream_t s, int dev,
                      SpecFrames* fr) {
  if (fr && (stats || t->info.internal <= 32))
    fail(ST_ERR_ARGUMENT, "speculative frame streams need a multi-window tree (> 32 internal nodes) and no counters");
  if (stats && t->info.internal > 32) {
    // counters are defined by whole-tree speculation (the reference law)
    return eval_spec_exact_cta(t, x, m, a, ld, layout, g.reductions, labels, stats, s, dev);
  }
  st_geom gg = g;
  if (stats) {
    // whole tree in one record group so the counters follow the reference law
    uint32_t G = 1;
    while (G < std::max<uint32_t>(1, t->info.internal)) G *= 2;
    gg.group_lanes = G;
    gg.window_levels = std::max<uint32_t>(1, t->info.depth);
  }
  uint32_t G, H;
  spec_geometry(t, gg, G, H);
  if (4ull * t->info.max_attribute >= (1u << 24))
    fail(ST_ERR_ARGUMENT, "speculative kernel requires attribute indices < 2^22");
  auto wt = t->windows(G, H);
  SEntry* wdev = t->device_windows(dev, G, H, *wt);
  st_tree::Dev& dv = t->device(dev);
  const DevProps pr = dev_props(dev);
  SpecArgs sa{};
  sa.p = pipe_args(x, m, a, ld, layout);
  sa.win = wdev;
  sa.n_entries = wt->base_units;
  sa.root_code = wt->root_code;
  sa.G = G;
  sa.smax = wt->max_steps;
  sa.k = g.reductions;
  sa.leaf_class = dv.leaf_tbl;
  sa.labels = labels;
  sa.lab_mask = kLeafBit - 1u;  // ring label rows: kLeafBit | class (per-format overrides below)
  if (stats) {
    sa.iters = stats->iterations;
    sa.steps = stats->doubling_steps;
    if (!sa.iters || !sa.steps) fail(ST_ERR_ARGUMENT, "st_stats requires both arrays");
    if (sa.k == 0) sa.k = 1;  // counters follow the reference loop (k per root check)
  } else if (sa.k != 0) {
    // k without counters: same labels; the fixed-step path is used
    sa.k = 0;
  }
  const uint32_t win_bytes = round1024((size_t)wt->base_units * sizeof(SEntry));
  bool win_shared = win_bytes <= 96 * 1024;
  Staging stg = plan_staging(x, m, a, ld, layout, 1, g.stages, win_shared ? win_bytes : 0, pr);
  if (win_shared && win_bytes + 1024 + stg.tile_smem() > pr.smem_optin) {
    win_shared = false;
    stg = plan_staging(x, m, a, ld, layout, 1, g.stages, 0, pr);
  }
  sa.win_bytes = win_shared ? win_bytes : 0;
  if (stg.loader == kDirect) stg.ns = 1, stg.stage_bytes = 0;
  // speculative is issue/latency-bound: several 8-warp CTAs per SM (the
  // occupancy maximum) beat one wide CTA (C2: 0.52 vs 0.68 ms)
  stg.warps = g.warps_per_cta ? pick_warps(g.warps_per_cta, stg, sa.win_bytes, pr) : kWarpsPerCta;
  sa.ns = stg.ns;
  sa.stage_bytes = stg.stage_bytes;
  const size_t smem = 1024 + sa.win_bytes + (size_t)stg.warps * stg.ns * (stg.stage_bytes + 8u) +
                      (size_t)stg.warps * 3 * 128;  // + per-warp label/counter rows
  const uint32_t bps = g.blocks_per_sm;  // speculative is latency-bound: keep every resident CTA
  // CTA-shared ring (default for the fast path): up to 32 warps on one SM
  // share NS = warps + 4 (lane triples) or + 12 tile slots.
  if (stg.loader == kTma && !stats && g.pipeline != 1) {
    const bool onewin = wt->windows == 1 && win_shared && !(g.variant & ST_VAR_SPEC_GENERAL);
    SpecArgs rs = sa;
    bool ws = win_shared, cw = false;
    // 8-byte window entries when the tree's fields fit (half the entry
    // wavefronts); ST_VAR_SPEC_WIDE keeps the 16-byte format
    if (!onewin && wt->cw_units && !(g.variant & ST_VAR_SPEC_WIDE)) {
      const uint32_t cb = round1024((size_t)wt->cw_units * sizeof(SEntry));
      if (cb <= 96 * 1024) {
        cw = ws = true;
        rs.win = wdev + wt->cw_off;
        rs.n_entries = wt->cw_units;
        rs.win_bytes = cb;
        const uint32_t ab = wt->cw_abits, cb2 = wt->cw_cbits;
        rs.cw_amask = (1u << ab) - 1u;
        rs.cw_lsh = ab;
        rs.cw_rsh = ab + cb2;
        rs.cw_cmask = (1u << cb2) - 1u;
        rs.cw_leaf = 1u << (cb2 - 1u);
        rs.cw_emask = (1u << (cb2 - 2u)) - 1u;
        rs.cw_wstride = 8u * G;
        rs.lab_mask = rs.cw_leaf - 1u;
      }
    }
    // record streams per group (samples_per_thread): two independent window
    // chains per lane.  With 8-byte entries they win on every canonical tree
    // (C2 0.357 vs 0.386 ms, C5 d8 0.281 vs 0.295, C1, C3, C5 d16;
    // profiles/r1_sweep_*_spec2_cw.json); with 16-byte entries only on large
    // trees (C5 d16: 0.61 vs 0.68 ms; C2, 255 internal: 0.399 vs 0.390 ms;
    // profiles/r1_sweep_*_spec2d.json, *_spec2e.json)
    uint32_t sr = g.samples_per_thread ? g.samples_per_thread : ((cw || t->info.internal > 511) ? 2u : 1u);
    if (onewin) sr = 0;  // whole tree in one window
    // Self-loop codes (WinTable::sl_*): a terminal code's low bits name its
    // own lane, so every pointer-jumping step is one shfl with no select,
    // and the two-stream loop advances a resolved stream by a constant
    // record-address step under predication.  Needs the stream step to keep
    // the tile's 128B-swizzle phase (row step = 0 or 4 mod 8).
    // ST_VAR_SPEC_SELECT keeps the select-per-step loop.
    int sl = 0;
    uint32_t lg = 0;
    while ((1u << lg) < G) ++lg;
    const bool want_sl = !(g.variant & ST_VAR_SPEC_SELECT);
    if (!(g.variant & ST_VAR_SPEC_SELECT)) {
      const uint32_t ng = 32u / G;
      const uint32_t adv = 2u * ng * 4u * a, rows_step = adv / 128u;
      if (want_sl && cw && sr >= 2 && wt->sl_units && (a == 8 || a == 16 || a == 32) && adv % 128u == 0 &&
          (rows_step % 8u == 0 || rows_step % 8u == 4) &&
          round1024((size_t)wt->sl_units * sizeof(SEntry)) <= 96 * 1024) {
        // Loop shape.  Round 2 chose by tree balance (profiles/r2_spec_sl_ab.txt):
        // the fixed trip (leaves absorbing, no per-step test) for balanced
        // trees, a predicated stream advance for skewed ones (C5 d16 - d20,
        // C2), a divergent advance otherwise.  With lane triples and the
        // warp's batch ending once every stream is absorbed (one vote per
        // step, sl_wcheck below), the fixed trip wins everywhere (same-box
        // A/B): C5 d18 / d20 -5 / -3 % vs predicated, d16 -9 %, C2 -1.5 %
        // (4-lane groups: its 32-attribute records would make 10 KB triple
        // slots).  ST_VAR_SPEC_PRED / _BRANCH force the others.
        sl = (g.variant & ST_VAR_SPEC_PRED) ? 1 : (g.variant & ST_VAR_SPEC_BRANCH) ? 2 : 3;
        rs.sl_wmax = wt->sl_wmax;
        // early batch exit (one vote per step) only where the deepest record
        // visits clearly more windows than the mean
        rs.sl_wcheck = (wt->sl_wmax > 1.25 * wt->sl_wmean) ? std::max<uint32_t>(1u, (uint32_t)wt->sl_wmean)
                                                           : wt->sl_wmax;
        rs.sl_ws = wt->sl_ws;
        rs.sl_wmul = 8u * wt->sl_ws / G;  // code units (w << log2 G) -> byte offset of window w
        rs.win = wdev + wt->sl_off;
        rs.n_entries = wt->sl_units;
        rs.win_bytes = round1024((size_t)wt->sl_units * sizeof(SEntry));
        rs.cw_amask = (1u << wt->sl_abits) - 1u;
        rs.cw_lsh = wt->sl_abits;
        rs.cw_rsh = wt->sl_abits + wt->sl_cbits;
        rs.sl_xmask = ((1u << wt->sl_cbits) - 1u) & ~(G - 1u);
        rs.sl_leafmin = wt->sl_nw << lg;
        rs.sl_adv = adv;
        rs.sl_xor = rows_step % 8u == 4 ? 0x40u : 0u;
        rs.lab_mask = 0xFFFFFFFFu;
        rs.lab_shift = lg;
        rs.lab_sub = wt->sl_nw;
      }
      if (onewin && (g.variant & ST_VAR_SPEC_JUMP) && wt->sl1_off) {
        sl = 1;  // one window: pointer jumping with self-loop leaf codes
        rs.lab_mask = ~kLeafBit;
        rs.lab_shift = 5;
      }
    }
    // 64-record ring slots for the two-stream 8-byte-window loop: the slot's
    // records are shared by 16 streams, 4 each instead of 2, which evens out
    // the streams' window counts and halves the per-slot overhead -- taken
    // when the slot stays at 4 KB (16 attributes: C5 d8 / d12 / d16 / d20
    // -5 / -10 / -8 / -6 %, C1 even).  Larger slots cost resident warps (C2,
    // 8 KB: +44 %); 2 KB ones gained nothing (C3 +2 %).  st_geom.slot_records
    // = 1 / 2 forces 32 / 64 (profiles/r1_spec_tile_ab.txt).
    uint32_t rt = 1;
    Staging rstg = stg;
    if (g.slot_records > 3) fail(ST_ERR_ARGUMENT, "slot_records must be 0-3");
    const uint32_t want_rt = g.slot_records ? std::min<uint32_t>(g.slot_records, 2u) : (a == 16 ? 2u : 1u);
    if (cw && sr >= 2 && (a == 8 || a == 16 || a == 32) && want_rt == 2 && m >= 64) {
      Staging s2 = plan_staging(x, m, a, ld, layout, 2, g.stages, rs.win_bytes, pr);
      if (s2.loader == kTma && s2.S == 2) rt = 2, rstg = s2;
    }
    // Lane triples (fixed-trip loop over G = 4 three-node windows): 10
    // record groups per warp instead of 8, 80-record slots -- C1 / C3 / C5
    // d8..d14 -8 / -10 / -9 % (same-box A/B); ST_VAR_SPEC_QUAD keeps the
    // 4-lane groups.
    // Triple slots hold 80 or 120 records (8 or 12 per group): 120 for
    // 8-attribute records (4 KB slots: C3 -1.3 % per frame, -2.1 % on 32
    // frames), 80 otherwise (120 would make 16-attribute slots 8 KB: C5 d12
    // +17 %); st_geom.slot_records = 2 / 3 forces 80 / 120.
    uint32_t triple = 0;
    if (sl == 3 && triple_ok(g, G, *wt, x, m, a, ld, layout)) {
      triple = g.slot_records == 3 ? 3u : g.slot_records == 2 ? 1u : a == 8 ? 3u : 1u;
      const uint32_t recs = triple == 3 ? kTripleSlot * 3 / 2 : kTripleSlot;
      Staging s3 = stg;
      s3.S = 1;
      s3.stage_bytes = round1024((uint64_t)recs * a * 4);
      make_tmap(s3, x, m, a, recs);
      rstg = s3;
      rt = 0;
    }
    const size_t slot_recs = rt ? 32u * rt : (size_t)(triple == 3 ? kTripleSlot * 3 / 2 : kTripleSlot);
    const size_t lb = 32 + 32 * 4 * slot_recs;  // generation padding + ticket + per-warp label rows (<= 32 warps)
    const size_t budget = pr.smem_optin - 1024 - rs.win_bytes - lb;
    const size_t max_slots = budget / (rstg.stage_bytes + 16u);
    // warps + extra slots: the slots beyond one per warp keep refills in
    // flight while every warp walks a tile; each slot fewer buys a resident
    // warp where shared memory binds (same-box A/B,
    // profiles/r2_spec_ring_slots_ab.txt: lane triples with + 4 vs + 12: C3
    // -4 %, C5 d16 / d20 -1.5 / -2.8 %; but the paper tree +5 %, C2 +1.3 %)
    const uint32_t extra = triple ? kRingExtraTriple : kRingExtra;
    const uint32_t warps = (uint32_t)std::min<size_t>(32, max_slots > extra ? max_slots - extra : 0);
    if (warps >= 4) {
      SpecRingArgs ra{};
      ra.s = rs;
      ra.n_slots = (uint32_t)std::min<size_t>(max_slots, warps + extra);
      // stress knob: any ring depth >= 1 must give exact labels
      if (g.ring_slots) ra.n_slots = std::min<uint32_t>(ra.n_slots, g.ring_slots);
      ra.ns_magic = (uint32_t)std::min<uint64_t>(0xFFFFFFFFull, (1ull << 32) / ra.n_slots);
      ra.bulk_win = (g.variant & ST_VAR_TREE_LOOP) ? 0u : 1u;
      ra.tile_mult = rt;
      ra.triple = triple;
      ra.s.stage_bytes = rstg.stage_bytes;
      const size_t rsmem = 1024 + rs.win_bytes + (size_t)ra.n_slots * (rstg.stage_bytes + 8u) +
                           (((size_t)4 * ra.n_slots + 15) & ~size_t(15)) + 16 + (size_t)warps * 4 * slot_recs;
      // one window: ballot + leaf path masks unless pointer jumping is asked
      // for (pm_off then names the self-loop entries, or 0: select per step)
      if (onewin) ra.s.pm_off = (g.variant & ST_VAR_SPEC_JUMP) ? (sl ? wt->sl1_off : 0u) : wt->pm_off;
      if (fr) {
        if (!(cw && sl == 3 && sr >= 2 && rt <= 1 && ra.s.smax == 1 && (a == 8 || a == 16 || a == 32)))
          fail(ST_ERR_ARGUMENT, "speculative frame stream needs the fixed-trip window loop (G = 4 windows, "
                                "8-byte self-loop tables, 8 / 16 / 32 attributes)");
        if (m % slot_recs != 0)
          fail(ST_ERR_ARGUMENT, "records per frame must be a multiple of " + std::to_string(slot_recs) +
                                    " (whole speculative ring slots per frame)");
        make_tmap(rstg, x, fr->ring_records, a, (uint32_t)slot_recs);
        ra.fctl = fr->fctl;
        ra.ring = fr->ring;
        ra.frame_rows = (uint32_t)(m * a / 32);
        ra.tpf = m / slot_recs;
        ra.idle_ns = fr->idle_ns;
        fr->tiles = ra.tpf;
        return launch_spec_frames(a, triple, ra, rstg, rsmem, dev, warps, fr->max_ctas, s);
      }
      switch (ct_arity(a) ? a : 0) {
        case 8: return launch_spec_ring<8>(ws, sr, cw, sl, ra, rstg, rsmem, dev, warps, s);
        case 16: return launch_spec_ring<16>(ws, sr, cw, sl, ra, rstg, rsmem, dev, warps, s);
        case 32: return launch_spec_ring<32>(ws, sr, cw, sl, ra, rstg, rsmem, dev, warps, s);
        case 64: return launch_spec_ring<64>(ws, sr, cw, sl, ra, rstg, rsmem, dev, warps, s);
        default: return launch_spec_ring<0>(ws, sr, cw, sl, ra, rstg, rsmem, dev, warps, s);
      }
    }
  }
  if (fr) fail(ST_ERR_ARGUMENT, "speculative frame stream needs the TMA-staged ring kernel");
  if (stg.loader == kTma && ct_arity(a)) {
    switch (a) {
      case 8: return launch_spec_t<8, kTma>(win_shared, sa, stg, smem, dev, bps, s);
      case 16: return launch_spec_t<16, kTma>(win_shared, sa, stg, smem, dev, bps, s);
      case 32: return launch_spec_t<32, kTma>(win_shared, sa, stg, smem, dev, bps, s);
      case 64: return launch_spec_t<64, kTma>(win_shared, sa, stg, smem, dev, bps, s);
    }
  }
  switch (stg.loader) {
    case kTma: return launch_spec_t<0, kTma>(win_shared, sa, stg, smem, dev, bps, s);
    case kDirect: return launch_spec_t<0, kDirect>(win_shared, sa, stg, smem, dev, bps, s);
    default: return launch_spec_t<0, kScalar>(win_shared, sa, stg, smem, dev, bps, s);
  }
}


}  // namespace sti
