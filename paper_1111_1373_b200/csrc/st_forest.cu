// Forest kernel dispatch (K3 k_forest_smem / k_forest).
#include "st_internal.cuh"

namespace sti {

// ---- forest ----------------------------------------------------------------
template <int A, int LOADER>
void launch_forest_t(bool packed, const ForestArgs& fa, const Staging& stg, size_t smem, int dev,
                     cudaStream_t s) {
  const uint64_t n_tiles = (fa.p.m + 31) / 32;
  if (packed) {
    auto fn = k_forest<A, LOADER, true>;
    const int blocks = blocks_for((const void*)fn, smem, dev, 0, n_tiles, stg.warps);
    clear_stale_error();
    fn<<<blocks, stg.warps * 32, smem, s>>>(fa, stg.tmap);
  } else {
    auto fn = k_forest<A, LOADER, false>;
    const int blocks = blocks_for((const void*)fn, smem, dev, 0, n_tiles, stg.warps);
    clear_stale_error();
    fn<<<blocks, stg.warps * 32, smem, s>>>(fa, stg.tmap);
  }
  check_launch();
}

template <int A, int S, int U>
void launch_forest_smem(const Forest2Args& fa, const Staging& stg, size_t smem, int dev,
                        cudaStream_t s) {
  auto fn = k_forest_smem<A, S, U>;
  const uint64_t n_tiles = (fa.p.m + 32 * S - 1) / (32 * S);
  // warp 0 of each CTA is the tree producer: tiles are spread over warps - 1
  const int blocks = blocks_for((const void*)fn, smem, dev, 0,
                                n_tiles * stg.warps / std::max<uint32_t>(1, stg.warps - 1), stg.warps);
  clear_stale_error();
  fn<<<blocks, stg.warps * 32, smem, s>>>(fa, stg.tmap);
  check_launch();
}

template <int A, int S>
void launch_forest_u(uint32_t U, const Forest2Args& fa, const Staging& stg, size_t smem, int dev,
                     cudaStream_t s) {
  if constexpr (S == 1 && A > 0 && A <= 64) {  // the transposed-tile walk takes U chains
    if (U >= 4) return launch_forest_smem<A, S, 4>(fa, stg, smem, dev, s);
    if (U == 3) return launch_forest_smem<A, S, 3>(fa, stg, smem, dev, s);
    if (U == 2) return launch_forest_smem<A, S, 2>(fa, stg, smem, dev, s);
  }
  return launch_forest_smem<A, S, 1>(fa, stg, smem, dev, s);
}


// Trees streamed through shared memory (packed votes, TMA-staged records).
bool forest_smem_path(st_forest* f, int lay, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                      int layout, const st_geom& g, uint32_t* labels, cudaStream_t s, int dev,
                      const DevProps& pr) {
  const st_forest::Layout& L = f->lay[lay];
  if (!(f->n_classes <= 8 && f->t_count <= 255) || L.max_tree_bytes > 48 * 1024) return false;
  // one record per lane (the tile is transposed to attribute-major once per
  // round, which needs the record in registers); parallelism from wide CTAs
  const uint32_t S = 1;
  if (!tma_ok(x, m, a, ld, layout, S)) return false;
  Staging stg;
  stg.loader = kTma;
  stg.S = S;
  stg.ns = 1;
  stg.stage_bytes = round1024(32ull * S * a * 4);
  // Geometry: U trees walked per lane at once (U dependent-load chains), a
  // ring of NT tree slots, and as many consumer warps as the rest of shared
  // memory holds record tiles for.  With folded trees (~10 KB for C4) the
  // sweep (profiles/r1_forest_sweep_fold.json) puts U = 3, NT = 6 first
  // (7.76 ms; U = 2, NT = 4: 7.95 ms; unfolded U = 2, NT = 4: 8.33 ms): the
  // walk is bound by shared-memory wavefronts of the node loads, so more
  // chains only add ring slots at the expense of record tiles.
  const bool transposed = S == 1 && a <= 64 && ct_arity(a);
  const uint32_t U = std::max<uint32_t>(1, std::min<uint32_t>(4, g.forest_chains ? g.forest_chains
                                                                                 : (transposed ? 3u : 1u)));
  uint32_t nt = g.forest_slots;
  if (nt == 0) nt = U + 3;
  if (!transposed && U != 1) return false;
  stg.warps = 0;
  size_t fixed = 0;
  for (uint32_t n = nt; n >= std::max<uint32_t>(2, U) && !stg.warps; --n) {
    const size_t region = round1024((uint64_t)n * L.max_tree_bytes);
    const size_t base = 1024 + region + 16u * n;
    if (base >= pr.smem_optin) continue;
    uint32_t w = (uint32_t)std::min<size_t>(kForestMaxThreads / 32, 1 + (pr.smem_optin - base) / (stg.stage_bytes + 8u));
    if (g.warps_per_cta) w = std::min(w, g.warps_per_cta);
    if (w < 2) continue;
    stg.warps = w;
    nt = n;
    fixed = base;
  }
  if (!stg.warps) return false;
  make_tmap(stg, x, m, a);
  st_forest::Dev& dv = f->device(dev, lay);
  Forest2Args fa{};
  fa.p = pipe_args(x, m, a, ld, layout);
  fa.nodes = dv.nodes;
  fa.offsets = dv.offsets;
  fa.t_count = f->t_count;
  fa.n_classes = f->n_classes;
  fa.abits = f->abits;
  fa.labels = labels;
  fa.stage_bytes = stg.stage_bytes;
  fa.tree_buf_bytes = L.max_tree_bytes;
  fa.n_tree_bufs = nt;
  fa.tree_region = round1024((uint64_t)nt * L.max_tree_bytes);
  fa.tree_bytes = dv.tree_bytes;
  const size_t smem = fixed + (size_t)(stg.warps - 1) * (stg.stage_bytes + 8u);
  switch (a) {
    case 8: return launch_forest_u<8, 1>(U, fa, stg, smem, dev, s), true;
    case 16: return launch_forest_u<16, 1>(U, fa, stg, smem, dev, s), true;
    case 32: return launch_forest_u<32, 1>(U, fa, stg, smem, dev, s), true;
    case 64: return launch_forest_u<64, 1>(U, fa, stg, smem, dev, s), true;
    default: return launch_forest_u<0, 1>(U, fa, stg, smem, dev, s), true;
  }
}

void forest_device_impl(st_forest* f, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                        int layout, const st_geom& g, uint32_t* labels, cudaStream_t s) {
  if (!f) fail(ST_ERR_ARGUMENT, "null forest");
  check_common(m, a, ld, layout, f->max_attribute);
  if (m == 0) return;
  if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
  if (g.forest_chains > 4) fail(ST_ERR_ARGUMENT, "forest_chains must be 0-4");
  const int dev = current_device();
  const DevProps pr = dev_props(dev);
  const int lay = (g.variant & ST_VAR_NO_FOLD) ? 1 : 0;
  if (forest_smem_path(f, lay, x, m, a, ld, layout, g, labels, s, dev, pr)) return;
  st_forest::Dev& dv = f->device(dev, lay);
  ForestArgs fa{};
  fa.p = pipe_args(x, m, a, ld, layout);
  fa.nodes = dv.nodes;
  fa.offsets = dv.offsets;
  fa.t_count = f->t_count;
  fa.n_classes = f->n_classes;
  fa.abits = f->abits;
  fa.labels = labels;
  const bool packed = f->n_classes <= 8 && f->t_count <= 255;
  const size_t cnt_bytes = packed ? 0 : (size_t)kWarpsPerCta * 32 * f->n_classes * 4;  // 8-warp CTAs
  Staging stg = plan_staging(x, m, a, ld, layout, 1, 0, cnt_bytes, pr);
  fa.ns = stg.ns;
  fa.stage_bytes = stg.stage_bytes;
  const size_t smem = 1024 + stg.tile_smem() + cnt_bytes;
  if (stg.loader == kTma && ct_arity(a)) {
    switch (a) {
      case 8: return launch_forest_t<8, kTma>(packed, fa, stg, smem, dev, s);
      case 16: return launch_forest_t<16, kTma>(packed, fa, stg, smem, dev, s);
      case 32: return launch_forest_t<32, kTma>(packed, fa, stg, smem, dev, s);
      case 64: return launch_forest_t<64, kTma>(packed, fa, stg, smem, dev, s);
    }
  }
  switch (stg.loader) {
    case kTma: return launch_forest_t<0, kTma>(packed, fa, stg, smem, dev, s);
    case kDirect: return launch_forest_t<0, kDirect>(packed, fa, stg, smem, dev, s);
    default: return launch_forest_t<0, kScalar>(packed, fa, stg, smem, dev, s);
  }
}


}  // namespace sti
