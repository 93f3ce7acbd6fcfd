// Data-decomposition kernel dispatch (K1 k_data, st_kernels.cuh).
#include "st_internal.cuh"

namespace sti {

// ---- data kernel dispatch ------------------------------------------------
template <int A, int S, int TLOC, int LOADER, int CAP, bool DEPTH>
void launch_data_t(const DataArgs& d, const Staging& stg, const ConstTree<CAP>* ct, size_t smem,
                   int dev, uint32_t bps, cudaStream_t s) {
  auto fn = k_data<A, S, TLOC, LOADER, CAP, DEPTH>;
  const uint64_t n_tiles = (d.p.m + 32 * S - 1) / (32 * S);
  const int blocks = blocks_for((const void*)fn, smem, dev, bps, n_tiles, stg.warps);
  static const ConstTree<1> dummy{};
  clear_stale_error();
  if (d.pdl) {
    // programmatic dependent launch: the prologue (barrier init, tree copy)
    // may overlap the previous kernel in the stream; the kernel waits for it
    // (griddepcontrol.wait) before touching records or labels
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(stg.warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if constexpr (CAP == 1) CK(cudaLaunchKernelEx(&cfg, fn, d, stg.tmap, ct ? *ct : dummy));
    else CK(cudaLaunchKernelEx(&cfg, fn, d, stg.tmap, *ct));
  } else if constexpr (CAP == 1) {
    fn<<<blocks, stg.warps * 32, smem, s>>>(d, stg.tmap, ct ? *ct : dummy);
  } else {
    fn<<<blocks, stg.warps * 32, smem, s>>>(d, stg.tmap, *ct);
  }
  check_launch();
}

// DEPTH (traversal depths beside the labels): record-major walks only, the
// tree in shared memory, global memory (L1) or the 16-byte original nodes.
template <int A, int S, int LOADER, bool DEPTH>
void launch_data_tloc(int tloc, const DataArgs& d, const Staging& stg, const st_tree* t,
                      size_t smem, int dev, uint32_t bps, cudaStream_t s) {
  switch (tloc) {
    case ST_TREE_SHARED:
      if constexpr ((A == 8 || A == 16) && LOADER == kTma && !DEPTH) {
        if (d.record_regs == 2) return launch_data_t<A, S, kSharedT, LOADER, 1, DEPTH>(d, stg, nullptr, smem, dev, bps, s);
        if (d.record_regs) return launch_data_t<A, S, kSharedReg, LOADER, 1, DEPTH>(d, stg, nullptr, smem, dev, bps, s);
      }
      return launch_data_t<A, S, kShared, LOADER, 1, DEPTH>(d, stg, nullptr, smem, dev, bps, s);
    case ST_TREE_GLOBAL:
      return launch_data_t<A, S, kGlobal, LOADER, 1, DEPTH>(d, stg, nullptr, smem, dev, bps, s);
    case ST_TREE_CONSTANT: {
      if constexpr (LOADER == kTma && !DEPTH) {
        if (t->compact.size() <= 512) {
          ConstTree<512> ct{};
          std::copy(t->compact.begin(), t->compact.end(), ct.n);
          return launch_data_t<A, S, kConst, LOADER, 512, DEPTH>(d, stg, &ct, smem, dev, bps, s);
        }
        auto ct = std::make_unique<ConstTree<4000>>();
        std::copy(t->compact.begin(), t->compact.end(), ct->n);
        return launch_data_t<A, S, kConst, LOADER, 4000, DEPTH>(d, stg, ct.get(), smem, dev, bps, s);
      }
      break;
    }
    default:
      break;
  }
  return launch_data_t<A, S, kWide, LOADER, 1, DEPTH>(d, stg, nullptr, smem, dev, bps, s);
}


uint32_t choose_S(uint32_t a, uint32_t want, bool small) {
  // instantiated: a=8 {1,2,4}, a=16 {1,2,4}, a=32 {1,2}, others {1}
  const uint32_t maxS = (a == 8 || a == 16) ? 4 : a == 32 ? 2 : 1;
  // predicated walk (k_data data_step): independent chains per lane pay off
  // where a tile is small -- C3 (a = 8): S = 4 0.63 ms vs S = 2 0.67 ms for 32
  // frames; C2 (a = 32): S = 2 0.307 vs S = 1 0.321 ms (profiles/r1_sweep_*);
  // C5 (a = 16, one stage per warp): S = 4 vs 1: d12 -7 %, d16 -16 %, d20
  // -10 %, d8 even (profiles/r1_ab_stages.txt).  Small inputs keep S = 1
  // (C1 with a shared tree: S = 2, eval_data_device).
  if (want == 0) want = a <= 8 ? 4 : a == 32 ? 2 : (a == 16 && !small) ? 4 : 1;
  uint32_t S = 1;
  while (S * 2 <= std::min(want, maxS)) S *= 2;
  return S;
}

template <int A, bool DEPTH>
void launch_data_a(const Staging& stg, int tloc, const DataArgs& d, const st_tree* t, size_t smem,
                   int dev, uint32_t bps, cudaStream_t s) {
  if constexpr (A == 8 || A == 16) {
    if (stg.S == 4) return launch_data_tloc<A, 4, kTma, DEPTH>(tloc, d, stg, t, smem, dev, bps, s);
  }
  if constexpr (A == 8 || A == 16 || A == 32) {
    if (stg.S == 2) return launch_data_tloc<A, 2, kTma, DEPTH>(tloc, d, stg, t, smem, dev, bps, s);
  }
  return launch_data_tloc<A, 1, kTma, DEPTH>(tloc, d, stg, t, smem, dev, bps, s);
}

template <bool DEPTH>
void launch_data(const Staging& stg, int tloc, const DataArgs& d, const st_tree* t, size_t smem,
                 int dev, uint32_t bps, cudaStream_t s, uint32_t a) {
  if (stg.loader == kTma && ct_arity(a)) {
    switch (a) {
      case 8: return launch_data_a<8, DEPTH>(stg, tloc, d, t, smem, dev, bps, s);
      case 16: return launch_data_a<16, DEPTH>(stg, tloc, d, t, smem, dev, bps, s);
      case 32: return launch_data_a<32, DEPTH>(stg, tloc, d, t, smem, dev, bps, s);
      case 64: return launch_data_a<64, DEPTH>(stg, tloc, d, t, smem, dev, bps, s);
    }
  }
  switch (stg.loader) {
    case kTma: return launch_data_tloc<0, 1, kTma, DEPTH>(tloc, d, stg, t, smem, dev, bps, s);
    case kDirect:
      return launch_data_tloc<0, 1, kDirect, DEPTH>(tloc == ST_TREE_CONSTANT ? ST_TREE_GLOBAL : tloc, d,
                                                    stg, t, smem, dev, bps, s);
    default:
      return launch_data_tloc<0, 1, kScalar, DEPTH>(tloc == ST_TREE_CONSTANT ? ST_TREE_GLOBAL : tloc, d,
                                                    stg, t, smem, dev, bps, s);
  }
}

DataPlan plan_data(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                   const st_geom& g0, uint32_t* labels, uint32_t* depths, int dev) {
  st_geom g = g0;
  if (depths) {
    // traversal depths come from the record-major walks; the constant-bank
    // tree is a paper comparison variant without a depth counter
    g.record_regs = 2;
    if (g.tree_loc == ST_TREE_CONSTANT) g.tree_loc = ST_TREE_GLOBAL;
  }
  st_tree::Dev& dv = t->device(dev);
  const DevProps pr = dev_props(dev);
  DataArgs d{};
  d.p = pipe_args(x, m, a, ld, layout);
  d.nodes = dv.compact;
  d.wide = dv.wide;
  d.n_nodes = (uint32_t)t->nodes.size();
  d.abits = t->abits;
  d.leaf_class = dv.leaf_tbl;
  d.labels = labels;
  d.depths = depths;
  // records walked from registers: default for 8-attribute records; 16 on request
  // 8/16-attribute records: walk from registers (1), from the record-major
  // shared tile (0), or from the tile transposed in place to attribute-major
  // (2) -- the default for 8 attributes (C3: -4 % per frame, -0.6 % on 32
  // frames vs registers; profiles/r1_ab_stages.txt); 16-attribute records
  // walk the record-major tile (C5 d12 / d16: transposed +10 / +11 %)
  d.record_regs = g.record_regs == 1 ? 1u : 0u;
  if ((a == 8 || a == 16) && (g.record_regs == 3 || (g.record_regs == 0 && a == 8))) d.record_regs = 2u;
  d.bulk_tree = (g.variant & ST_VAR_TREE_LOOP) ? 0u : 1u;


  // fewer than 8 tiles of 32 records per warp at 32 warps on every SM
  // (trees read through L1 / the constant bank keep S = 1 as well)
  const bool small = m < (uint64_t)pr.sms * 32 * 8 * 32 || g.tree_loc == ST_TREE_GLOBAL ||
                     g.tree_loc == ST_TREE_CONSTANT;

  // the folded tree (leaf pairs inside terminals) serves the shared-tree TMA
  // walks over 8/16/32-attribute records of large trees; every other path
  // reads `compact`.  Same-box A/B (profiles/r1_fold_ab.txt): C5 d12 -6 %,
  // C1 -5 %, C5 d16 / d20 -3 / -2 %; on small trees the post-loop terminal
  // step only lengthens each tile (C2 +4 %, C5 d8 +3 %), hence >= 2047 nodes.
  const bool fold = t->fold_ok && t->nodes.size() >= (g.fold_min ? g.fold_min : 2047u) &&
                    (a == 8 || a == 16 || a == 32) &&
                    !(g.variant & ST_VAR_NO_FOLD) &&
                    (g.tree_loc == ST_TREE_AUTO || g.tree_loc == ST_TREE_SHARED) &&
                    tma_ok(x, m, a, ld, layout, ct_arity(a) ? choose_S(a, g.samples_per_thread, small) : 1);
  uint32_t tree_bytes = round1024((fold ? t->folded.size() : t->nodes.size()) * sizeof(CNode));
  int tloc = g.tree_loc;
  if (!t->compact_ok) tloc = kWide;
  else if (tloc == ST_TREE_AUTO) tloc = tree_bytes <= 96 * 1024 ? ST_TREE_SHARED : ST_TREE_GLOBAL;
  if (tloc == ST_TREE_CONSTANT && t->compact.size() > 4000) tloc = ST_TREE_GLOBAL;
  // shared trees are rebased to absolute shared addresses inside the compact
  // child field: the largest address must fit below the leaf bit
  if (tloc == ST_TREE_SHARED && ((uint64_t)pr.smem_optin << t->abits) >= (1ull << 31)) tloc = ST_TREE_GLOBAL;
  uint32_t S0 = ct_arity(a) ? choose_S(a, g.samples_per_thread, small) : 1;
  // small 16-attribute inputs walking a shared tree (C1): S = 2 with one
  // stage per warp, 15.6 vs 15.9-16.6 us for S = 1 with one or two stages
  // (profiles/r2_small_sweep_C1.json)
  const bool small16 = !g.samples_per_thread && a == 16 && small && tloc == ST_TREE_SHARED &&
                       g.tree_loc != ST_TREE_GLOBAL && g.tree_loc != ST_TREE_CONSTANT &&
                       tma_ok(x, m, a, ld, layout, 2);
  if (small16) S0 = 2;
  // Records walked from registers release their tile before the walk, so one
  // stage per warp already double-buffers (next TMA in flight during the
  // walk) and the saved shared memory buys twice the warps (C3 x 32 frames:
  // 0.566 vs 0.615 ms, profiles/r1_sweep_C3x32_regs1.json).
  // Shared-tree walks over large inputs: one stage per warp too -- the
  // smem it frees holds S-record tiles for as many warps, and the S chains
  // per lane hide the tree latency better than a second tile in flight
  // (same-box A/B, profiles/r1_ab_stages.txt: C2 -1.9 %, C5 d16 -16 %).
  // Small inputs keep two, except 16-attribute records at S = 2 (above).
  const uint32_t want_ns =
      g.stages ? g.stages : ((d.record_regs == 1 || !small || small16) && tloc == ST_TREE_SHARED ? 1u : 0u);
  Staging stg = plan_staging(x, m, a, ld, layout, S0, want_ns,
                             tloc == ST_TREE_SHARED ? tree_bytes : 0, pr);
  if (tloc == ST_TREE_SHARED && tree_bytes + 1024 + stg.tile_smem() > pr.smem_optin) {
    tloc = ST_TREE_GLOBAL;
    stg = plan_staging(x, m, a, ld, layout, S0, g.stages, 0, pr);
  }
  if (tloc == ST_TREE_CONSTANT && stg.loader != kTma) tloc = ST_TREE_GLOBAL;
  // A large shared-memory tree is staged once per CTA: widen the CTA so that
  // one copy serves up to 32 warps instead of capping the SM at one 8-warp CTA.
  stg.warps = pick_warps(g.warps_per_cta, stg, tloc == ST_TREE_SHARED ? tree_bytes : 0, pr);
  uint32_t want_bps = g.blocks_per_sm;
  // Small inputs (< 8 tiles per warp at 32 warps/SM, e.g. C1's 1M records)
  // are ramp-up bound: four 8-warp CTAs per SM stage their tree copies
  // faster than one 32-warp CTA (C1: 17.0 vs 19.3 us, profiles/r1_sweep_C1x1_small_flush.json).
  const uint64_t tiles_total = m / (32ull * stg.S);
  if (!g.warps_per_cta && !g.blocks_per_sm && stg.loader == kTma && tloc == ST_TREE_SHARED &&
      tiles_total < (uint64_t)pr.sms * 32 * 8 &&
      4 * (1024 + tree_bytes + (size_t)kWarpsPerCta * stg.ns * (stg.stage_bytes + 8u)) <= pr.smem_per_sm) {
    stg.warps = kWarpsPerCta;
    want_bps = 4;
  }
  // transposed tiles: the scaled attribute field widens the meta's low part
  // by log2(32) bits; the absolute child address must still fit below bit 31
  if (d.record_regs == 2) {
    if (stg.loader != kTma || ((uint64_t)pr.smem_optin << (t->abits + 5u)) >= (1ull << 31)) d.record_regs = 0;
  }
  d.ns = stg.ns;
  d.stage_bytes = stg.stage_bytes;
  if (fold && tloc == ST_TREE_SHARED) {
    if (stg.loader != kTma) fail(ST_ERR_CUDA, "internal: folded tree without the TMA walk");
    d.nodes = dv.folded;
    d.n_nodes = (uint32_t)t->folded.size();
  }
  d.tree_bytes = tloc == ST_TREE_SHARED ? tree_bytes : 0;
  const size_t smem = 1024 + d.tree_bytes + stg.tile_smem();
  const uint32_t bps = default_bps(want_bps, stg, m, pr);
  // Programmatic dependent launch: the prologue (barrier init, tree copy)
  // overlaps the previous kernel's tail.  Dependents are triggered early only
  // when one of their CTAs fits beside the ones launched per SM (small inputs:
  // C1 -6 % per launch in a back-to-back stream); otherwise the trigger is the
  // implicit one at exit (C1 / C3 -2 %; an early trigger without room cost
  // C3 +5 %; tools/pdl_ab.py, profiles/r1_pdl_ab.txt).  st_geom.pdl: 0 auto,
  // 1 early, 2 at exit, 3 off.
  {
    const size_t cta = smem + 1024;  // + the per-CTA shared-memory reservation
    const bool room = bps > 0 && (size_t)(bps + 1) * cta <= pr.smem_per_sm;
    if (g.pdl > 3) fail(ST_ERR_ARGUMENT, "pdl must be 0-3");
    d.pdl = g.pdl == 0 ? (room ? 1u : 2u) : g.pdl == 3 ? 0u : g.pdl;
  }
  DataPlan pl;
  pl.stg = stg;
  pl.tloc = tloc;
  pl.d = d;
  pl.smem = smem;
  pl.bps = bps;
  return pl;
}

void eval_data_device(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom& g, uint32_t* labels, uint32_t* depths, cudaStream_t s, int dev) {
  const DataPlan pl = plan_data(t, x, m, a, ld, layout, g, labels, depths, dev);
  if (depths) return launch_data<true>(pl.stg, pl.tloc, pl.d, t, pl.smem, dev, pl.bps, s, a);
  return launch_data<false>(pl.stg, pl.tloc, pl.d, t, pl.smem, dev, pl.bps, s, a);
}


}  // namespace sti
