// gemm.cu — fused multiplexed-LoRA linear for sm_100a (tcgen05 cta_group::2 +
// TMEM + TMA), one persistent warp-specialized kernel per call.
//
// For all segments of an hTask at once (spatial batching of the BaseOp, Eq. 1
// P:484-489 / Eq. 2) plus every segment's LoRA adapter (north_star
// formula), fused horizontally across tasks:
//
//   fwd:  Y  = X W^T            + Hs B_t^T      Hs = bf16(s_t X A_t^T)
//   bwd:  dX = dY W             + Gs A_t        Gs = bf16(s_t dY B_t)
//
// Execution unit = a CTA pair (cluster of 2 on one TPC).  The leader CTA's
// single MMA thread issues tcgen05.mma.cta_group::2 with M = 256: each CTA
// stages its own 128 rows of A and half (128 columns) of the B tile, and owns
// 128 TMEM lanes of the fp32 accumulator.  Each CTA therefore streams 32 KB per
// 64-deep k-block for a 128x256 output slab (half the B traffic of a 1-CTA
// 128x256 tile), with a 6-stage TMA ring.
//
// Work items, static round-robin over clusters:
//   * side tiles (one per 256-row block m): the shrink Hs/Gs[m] = s_t X_m A_t^T
//     (MMA N = 128; CTA 0's half of B holds the rank-padded A_t, CTA 1's half
//     is TMA zero fill), written to global and published by release-adds on
//     flags[m] (8 = all epilogue warps of the pair);
//   * main tiles (m, n): the backbone product over the whole reduction, then one
//     "extension" k-block per task present in the tile: A = Hs/Gs tile,
//     B = B_t / A_t tile (the expand), accumulated into the same TMEM tile.
// Segments are multiples of 64 rows, so a 256-row tile holds at most four
// tasks; their adapter MMAs carry the tcgen05 disable-output-lane mask of every
// other task's rows, so a row is only ever multiplied by its own task's
// weights (NaN isolation).
// Fused projections (num_slices > 1, e.g. q|k|v): every task has one adapter per
// column slice of W.  A side tile then computes the shrink of every slice in one
// pass over A: per (task group, slice pair) unit, CTA rk stages slice 2 sp + rk of
// the adapter, so one N = 128 MMA yields two slices (TMEM columns 64 s); a main
// tile runs one extension block per (task, slice overlapping the tile), the
// slice's B_t rows addressed relative to the slice start so rows outside it are
// TMA zero fill (a tile straddling two slices runs both).  The dX tiles run an
// extension block per (task, slice): Gs_s A_{t,s} contributes to every column.
// Side tiles come first in their band (or, for reductions <= 2048, before all
// main tiles) and never wait, so every dependency points to a lower tile
// index: with all CTAs resident the lowest unfinished tile always progresses
// (no deadlock).  Variants of the same kernel: has_main = 0 runs side tiles
// only, over a row-block range (mux_linear_shrink); has_side = 0 runs main
// tiles only, with Hs given by the caller (mux_linear_fwd_hs); kNarrow uses
// 256 x 128 pair tiles (outputs <= 128 columns).
//
// Roles (256 threads per CTA): warp 0 = TMA producer (both CTAs), warp 1 = MMA
// issuer (leader CTA), warp 2 = TMEM allocator, warps 4..7 = epilogue
// (TMEM -> regs -> bf16 -> swizzled smem -> TMA store).  Two 256-column TMEM
// accumulators: the epilogue of tile i overlaps the mainloop of tile i+1.
#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {

// Stage layout per CTA (all 128 B swizzled, 1024 B aligned):
//   A: kKSub k-subtiles of [128 rows x 128 B] (16 KB each)
//   B K-major (fwd): kKSub k-subtiles of [128 n-rows x 128 B]
//   B MN-major (bwd): 2 MN atoms (64 columns each) of [kBK K-rows x 128 B]
//   side-tile B per task group: [64 rows x 128 B] per k-subtile (8 KB each)
constexpr uint32_t kBox = 64 * 128;                  // 8 KB: one {64 x 128 B} TMA box
constexpr uint32_t kSubA = kBM * 128;                // 16 KB: one k-subtile of A
constexpr uint32_t kEpiBuf = 32 * 128;               // 32 rows x 64 bf16 (one TMA store box)
constexpr uint32_t kSmemMisc = 1024;
// per-row-block task groups, computed once per launch by all threads (8 B per pair row block)
constexpr int kGroupTab = 128;                       // row blocks covered (32768 rows); beyond: on the fly
constexpr uint32_t kSmemGroups = kGroupTab * 8;

// kTileN = output columns of a pair tile: 128 (narrow), 256 (standard: two 256-column TMEM
// accumulators, the epilogue of tile i overlaps the mainloop of tile i+1) or 512 (wide: one
// 512-column accumulator filled by two N = 256 MMAs per k-step; each CTA stages 256 B rows, so the
// operand feed per FLOP is 3/4 of the standard tile's, at the cost of the epilogue overlap —
// cuBLAS's own choice on these shapes, profiles/r02_cublas_kernels.csv).
// Carrier shrink (standard tiles): the shrink Hs = s_t X A_t^T (bwd: Gs = s_t dY B_t) rides on the
// first main tiles of each row block instead of a side tile (no second pass over X / dY).  Per stage
// each CTA stages kShrinkRows of the 32 stacked adapter rows of the carrier's task groups (fwd: A_t
// K-major, {64 k x 8 rows} boxes, 128 B swizzle; bwd: B_t MN-major, one {16 j x 128 n} box, 32 B
// swizzle), so one N = 32 MMA per k-step accumulates the shrink into the other accumulator's first
// columns.
constexpr int kShrinkRows = 16;                       // per CTA: MMA N = 32 stacked adapter rows
constexpr uint32_t kShrinkSub = kShrinkRows * 128;    // 2 KB per 64-deep k-subtile per CTA

template <bool kBwd, int kTileN = 256>
struct GemmLayout {
  static constexpr bool kWide = kTileN == 512;
  static constexpr bool kCarry = kTileN == 256;              // instantiations that can carry the shrink
  static constexpr int kEpiBufs = kCarry ? 1 : 2;           // TMA-store staging buffers per epilogue warp
  static constexpr int kBK = kWide ? 64 : GemmCfg<kBwd>::kBK;
  static constexpr int kKSub = kBK / 64;
  static constexpr int kStages = kWide ? 4 : GemmCfg<kBwd>::kStages;
  static constexpr int kBoxesB = kWide ? 4 : 2;             // 64-row B boxes per CTA per k-subtile
  static constexpr uint32_t kBSub = kBoxesB * kBox;         // one k-subtile of this CTA's B (K-major)
  static constexpr uint32_t kStageA = kKSub * kSubA;
  static constexpr uint32_t kStageB = kKSub * kBSub;        // this CTA's share of B
  static constexpr uint32_t kStageBytes = kStageA + kStageB;
  static constexpr uint32_t kAtomMN = kBK * 128;            // MN-major atom: kBK K-rows x 128 B
  static constexpr uint32_t kSideGrp = kKSub * kBox;        // side-tile B of one task group
  static constexpr uint32_t kSmemPipe = kStages * kStageBytes;
  static constexpr uint32_t kShrinkStage = kKSub * kShrinkSub;  // fwd 16 rows x 128 B; bwd 128 k-rows x 32 B
  static constexpr uint32_t kSmemShrink = kCarry ? kStages * kShrinkStage : 0;
  static constexpr uint32_t kSmemEpiL = 4 * kEpiBufs * kEpiBuf;
  static constexpr uint32_t kSmemBytes = kSmemPipe + kSmemShrink + kSmemEpiL + kSmemMisc + kSmemGroups + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB of dynamic shared memory per block");
};
constexpr uint32_t kTmemCols = 512;
constexpr int kGemmThreads = 256;
constexpr uint16_t kPairMask = 0x3;

// Tasks present in a 256-row pair tile, packed in registers (a dynamically indexed array here sat
// in local memory: ~3k cycles of dependent LDL/STL per tile in the producer and the MMA issuer,
// a third of an 8-k-block tile, profiles/r02_gemm_waits_tp.jsonl): group i's segment in byte i of
// seg4, its quarter mask in nibble i of hm4 (bit h set: the group owns rows [64h, 64h+64)).
struct PairGroups {
  int n;
  uint32_t seg4;
  uint32_t hm4;
  __device__ __forceinline__ int seg(int i) const { return static_cast<int>((seg4 >> (8 * i)) & 0xFFu); }
  __device__ __forceinline__ int hm(int i) const { return static_cast<int>((hm4 >> (4 * i)) & 0xFu); }
};

// Binary search over the (non-decreasing) segment offsets: the segment s with
// so[s] <= row < so[s+1], or -1.  Empty segments are skipped by construction
// (the largest s with so[s] <= row is taken).
__device__ __forceinline__ int seg_containing(const int* so, int S, int row) {
  if (S <= 0 || row < so[0] || row >= so[S]) return -1;
  int lo = 0, hi = S;  // so[lo] <= row < so[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (so[mid] <= row) lo = mid; else hi = mid;
  }
  return lo;
}

// Runs once per tile in the producer and the MMA issuer: the first quarter's
// segment by binary search, the next quarters by advancing from it (a linear
// search per quarter was ~2.5 k cycles per tile at 16 segments, which the
// producer could not hide behind short reductions).
__device__ __forceinline__ PairGroups pair_groups(const GemmParams& p, const int* so, int m) {
  PairGroups g;
  g.n = 0;
  g.seg4 = 0u;
  g.hm4 = 0u;
  const int S = p.num_segs;
  const int row0 = m * kPairRows;
  int s = seg_containing(so, S, row0);
  if (s < 0 && S > 0 && row0 < so[0]) s = 0;  // rows before the first segment: start from segment 0
  int last = -1;                              // segments are contiguous row ranges: a quarter's segment
#pragma unroll                                // is either the previous quarter's or a new group
  for (int h = 0; h < 4; ++h) {
    const int row = row0 + kRowQuarter * h;
    if (s < 0 || row >= so[S]) break;
    while (s + 1 < S && so[s + 1] <= row) ++s;
    if (!(so[s] <= row && row < so[s + 1])) continue;
    if (p.seg_rank[s] == 0) continue;
    if (s != last) {
      g.seg4 |= static_cast<uint32_t>(s) << (8 * g.n);
      ++g.n;
      last = s;
    }
    g.hm4 |= (1u << h) << (4 * (g.n - 1));
  }
  return g;
}

// Does the extension block of adapter slot `slot` (slice s) contribute to the main tile covering
// output columns [tc0, tc1)?  Forward: only where the tile overlaps the slice's columns (a tile
// straddling two slices runs both, each with the other slice's rows of B zero-filled).  Backward
// (dX): every slice, the reduction of Gs_s A_{t,s} is over ranks.  Producer and MMA issuer take
// the same decision.
template <bool kBwd>
__device__ __forceinline__ bool ext_live(const GemmParams& p, int slot, int s, int tc0, int tc1) {
  if (p.slot_rank[slot] == 0) return false;
  if (kBwd) return true;
  return p.slice_off[s] < tc1 && p.slice_off[s + 1] > tc0;
}

// disable-output-lane mask of a group owning the quarters in `hm`
__device__ __forceinline__ void lane_masks(int hm, uint32_t (&m)[8]) {
#pragma unroll
  for (int w = 0; w < 8; ++w) m[w] = ((hm >> (w >> 1)) & 1) ? 0u : ~0u;
}

struct Tile {
  int m, n;
  bool side;
  bool carrier;  // carrier mode: this main tile also computes (part of) its row block's shrink
};

// Carrier schedule (p.carry, forward): no side tiles.  Every row block's first `nc` main tiles
// (n < nc) carry its shrink — carrier j the task groups [j * gpc, (j + 1) * gpc), gpc = 32 / r_cap —
// and come first (carrier 0 of every row block, then carrier 1, ...); then the other main tiles in
// row bands as usual.  A carrier waits only for its own shrink (published by its own epilogue
// before the tile's extension blocks); every other tile depends on lower-indexed carriers.
__device__ __forceinline__ Tile tile_at_carry(int t, int num_m, int num_n, int nc, int group_m) {
  Tile r;
  r.side = false;
  if (t < num_m * nc) {
    r.n = t / num_m;
    r.m = t - r.n * num_m;
    r.carrier = true;
    return r;
  }
  t -= num_m * nc;
  const int nn = num_n - nc;
  const int per_band = group_m * nn;
  const int band = t / per_band;
  const int first_m = band * group_m;
  const int gm = min(num_m - first_m, group_m);
  const int w = t - band * per_band;
  r.m = first_m + w % gm;
  r.n = nc + w / gm;
  r.carrier = false;
  return r;
}

// Raster: bands of `group_m` pair row-blocks.  Each band is [its side tiles]
// then [its main tiles, row block fastest], so the side tiles' pass over the
// band's A rows warms L2 right before the main tiles sweep W through it, and
// every main tile still depends only on a lower-indexed side tile (group_m is
// sized on the host so a band of A rows fits L2 next to the streamed W tiles).
// Without main tiles (shrink only) the side tiles cover row blocks [side_lo, ..);
// without side tiles (Hs given by the caller) the bands hold main tiles only.
// side_first (short reductions, chosen on the host): every side tile first, then the main tiles
// band by band.  With short main tiles, a band's main tiles otherwise reach their extension
// block while that band's side tiles (same wave) are still in their epilogue, and the producer
// stalls on the flag (profiles/r01_gemm_ab_sidefirst.jsonl).
// group_n > 0 (chosen on the host for long reductions where W is the smaller operand, e.g. the
// 11008 -> 4096 down projection): bands of group_n output-column blocks instead; within a band
// row block by row block, columns fastest, so the band's W tiles (group_n * 256 columns * kred)
// stay L2-resident while A streams past them once per band; the first band carries each row
// block's side tile right before that row block's main tiles (dependencies still point down).
__device__ __forceinline__ Tile tile_at(int t, int num_m, int num_n, int group_m, bool has_main, bool has_side,
                                       int side_lo, bool side_first, int group_n) {
  Tile r;
  r.carrier = false;
  if (!has_main) {
    r.m = side_lo + t; r.n = 0; r.side = true;
    return r;
  }
  if (group_n > 0) {
    const int ns = has_side ? 1 : 0;
    const int g0 = min(group_n, num_n);
    const int first = num_m * (g0 + ns);
    if (t < first) {
      const int m = t / (g0 + ns);
      const int w = t - m * (g0 + ns);
      r.m = m; r.n = w - ns; r.side = w < ns;
      if (r.side) r.n = 0;
      return r;
    }
    t -= first;
    const int per = num_m * group_n;
    const int b = 1 + t / per;
    const int loc = t - (b - 1) * per;
    const int gnb = min(group_n, num_n - b * group_n);
    r.m = loc / gnb;
    r.n = b * group_n + (loc - r.m * gnb);
    r.side = false;
    return r;
  }
  if (has_side && side_first) {
    if (t < num_m) {
      r.m = t; r.n = 0; r.side = true;
      return r;
    }
    t -= num_m;
    has_side = false;
  }
  const int ns = has_side ? 1 : 0;
  const int per_band = group_m * (num_n + ns);
  const int band = t / per_band;
  const int first_m = band * group_m;
  const int gm = min(num_m - first_m, group_m);
  const int w = t - band * per_band;
  if (w < gm * ns) {
    r.m = first_m + w; r.n = 0; r.side = true;
    return r;
  }
  const int v = w - gm * ns;
  r.m = first_m + v % gm;
  r.n = v / gm;
  r.side = false;
  return r;
}

// ---- stream-K (p.sk): balance the main tiles' k-block units over the clusters.
// Every cluster first runs its shrink (side) tiles, round-robin as in the data-parallel schedule;
// then one contiguous range of main-tile k-block units [b[c], b[c+1]) in tile-major order
// (tile = n * num_m + m, k fastest: the clusters' ranges advance in lockstep, so the pairs working
// at the same moment cover one stretch of row blocks under every output tile and share it in L2), sized so that every cluster's side + main work is equal (a
// side tile's k-block counts sk_side_cost_x4 / 4 main k-blocks).  A range that starts inside a
// tile computes a partial accumulator (k-blocks [k0, k1) of that tile) into cluster c's slot of
// sk_part and publishes it on sk_flags[c]; the piece holding k-block 0 of a tile — at the END of
// an earlier cluster's range — runs the LoRA extension blocks, waits for the partials of every
// later cluster whose range starts inside the tile and adds them in ascending cluster order
// (deterministic).  A partial piece is the first item of its cluster's main range and never
// waits on anything, so the finalizing piece (last item of an earlier range) cannot deadlock.
__device__ void sk_compute_bounds(const GemmParams& p, int num_m, int num_n, int num_kb, int ncl, int* b) {
  const long long n_side = p.has_side ? num_m : 0;
  const long long w = (static_cast<long long>(p.sk_side_cost_x4) * num_kb + 3) / 4;
  const long long U = static_cast<long long>(num_m) * num_n * num_kb;
  const long long L = U + n_side * w;
  long long side_before = 0, prev = 0;
  b[0] = 0;
  for (int c = 1; c <= ncl; ++c) {
    const long long ns = (c - 1 < n_side) ? (n_side - 1 - (c - 1)) / ncl + 1 : 0;  // side tiles of cluster c-1
    side_before += ns * w;
    long long a = (c == ncl) ? U : (L * c) / ncl - side_before;
    a = a < prev ? prev : (a > U ? U : a);
    b[c] = static_cast<int>(a);
    prev = a;
  }
}

struct SkPiece {
  int k0, k1;   // k-block range of the piece
  bool fin;     // holds k-block 0: runs the extension blocks, adds the partials, stores the tile
  int tile;     // main tile index (n * num_m + m), stream-K only
};

// Every role walks the same item sequence: f(tile, piece).
template <typename F>
__device__ __forceinline__ void for_each_item(const GemmParams& p, int cid, int ncl, int num_m, int num_n,
                                              int side_lo, int total_tiles, int num_kb, const int* skb, int nc,
                                              F&& f) {
  if (nc > 0) {
    for (int t = cid; t < num_m * num_n; t += ncl)
      f(tile_at_carry(t, num_m, num_n, nc, p.group_m), SkPiece{0, num_kb, true, 0});
    return;
  }
  if (!p.sk) {
    for (int t = cid; t < total_tiles; t += ncl)
      f(tile_at(t, num_m, num_n, p.group_m, p.has_main != 0, p.has_side != 0, side_lo, p.side_first != 0,
                p.group_n),
        SkPiece{0, num_kb, true, 0});
    return;
  }
  const int n_side = p.has_side ? num_m : 0;
  for (int t = cid; t < n_side; t += ncl) f(Tile{t, 0, true, false}, SkPiece{0, num_kb, true, 0});
  const int end = skb[cid + 1];
  for (int u = skb[cid]; u < end;) {
    const int tile = u / num_kb;
    const int k0 = u - tile * num_kb;
    const int k1 = min(num_kb, end - tile * num_kb);
    const int n = tile / num_m;   // row block fastest: the clusters running at the same time share
    f(Tile{tile - n * num_m, n, false, false}, SkPiece{k0, k1, k0 == 0, tile});  // A rows and W tiles in L2
    u = tile * num_kb + k1;
  }
}

// Opt-in instrumentation (-DMUX_PROFILE, experiment builds only): per-role
// cycles spent waiting on each barrier, accumulated into GemmParams::dbg:
//   [0] MMA total  [1] MMA wait full  [2] MMA wait tmem-empty
//   [3] producer total [4] producer wait empty  [5] epilogue total [6] epilogue wait tmem-full
//   [7] producer per-tile setup (task lookup)  [8] producer TMA issue  [9] producer shrink-flag wait
//   [10] epilogue wait for its smem staging buffer (TMA store read)  [11] main tiles (producer 0s)
#ifdef MUX_PROFILE
#define PROF_T0(v) const long long v = clock64()
#define PROF_ADD(acc, t0) acc += clock64() - (t0)
#else
#define PROF_T0(v)
#define PROF_ADD(acc, t0)
#endif

template <bool kBwd, int kTileN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    mux_gemm_kernel(const __grid_constant__ GemmParams p) {
  using Ly = GemmLayout<kBwd, kTileN>;
  // kTileN = 128: 256 x 128 pair tiles (64 output columns per CTA) for narrow outputs, where 256-wide
  // tiles leave most CTA pairs idle (e.g. 128-column tensor-parallel shards); 512: wide tiles
  constexpr bool kWide = Ly::kWide;
  constexpr int kHalves = kTileN / 128;  // 64-row B boxes per CTA
  constexpr int kAccs = kWide ? 1 : 2;   // TMEM accumulators (512 columns in total)
  constexpr uint32_t kBSub = Ly::kBSub;
  constexpr int kBK = Ly::kBK;
  constexpr int kKSub = Ly::kKSub;
  constexpr int kStages = Ly::kStages;
  constexpr uint32_t kStageA = Ly::kStageA;
  constexpr uint32_t kStageBytes = Ly::kStageBytes;
  constexpr uint32_t kAtomMN = Ly::kAtomMN;
  constexpr uint32_t kSideGrp = Ly::kSideGrp;
  constexpr uint32_t kSmemPipe = Ly::kSmemPipe;
  constexpr bool kCarry = Ly::kCarry;
  constexpr int kEpiBufs = Ly::kEpiBufs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* pipe = smem;
  uint8_t* shrink_area = smem + kSmemPipe;  // carrier shrink B: [stage][16 rows x 128 B] per CTA
  uint8_t* epi = shrink_area + Ly::kSmemShrink;
  uint8_t* misc = epi + Ly::kSmemEpiL;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(misc);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sfull_bar = tempty_bar + 2;   // carrier: its shrink accumulator is complete
  uint64_t* sempty_bar = sfull_bar + 1;   // carrier: the epilogue has read it (8 warps of the pair)
  // the TMEM address slot sits apart from the mbarriers (which peer CTAs and the async proxy write)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(misc + 192);
  static_assert((2 * GemmLayout<kBwd, kTileN>::kStages + 6) * 8 <= 192, "mbarriers overlap the TMEM slot");
  int* so = reinterpret_cast<int*>(misc + 256);  // seg_off copy, <= 65 ints
  int* skb = reinterpret_cast<int*>(misc + 528);  // stream-K range table, <= kSkMaxClusters + 1 ints
  int* s_gmax = reinterpret_cast<int*>(misc + 1016);  // max task groups over the row blocks (carrier mode)
  uint2* gtab = reinterpret_cast<uint2*>(misc + kSmemMisc);  // [kGroupTab] {seg4, hm4 | n << 24}

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int cid = static_cast<int>(cluster_id_x());
  const int ncl = static_cast<int>(nclusters_x());

  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.map_a);
    tma_prefetch(&p.map_side);
    if (p.has_main) {  // shrink-only launches leave these maps unencoded
      tma_prefetch(&p.map_w);
      tma_prefetch(&p.map_out);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8);
    }
    mbar_init(sfull_bar, 1);
    mbar_init(sempty_bar, 8);
    *s_gmax = 0;
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_holder);
  // --- everything above overlaps the previous kernel (PDL); inputs below ---
  griddep_wait();
  griddep_launch_dependents();
  for (int i = threadIdx.x; i <= p.num_segs; i += blockDim.x) so[i] = p.seg_off[i];
  if (p.sk && threadIdx.x == 96) {  // warp 3 has no role: the stream-K range table
    const int rows = p.seg_off[p.num_segs];
    sk_compute_bounds(p, (rows + kPairRows - 1) / kPairRows, (p.nout + kTileN - 1) / kTileN,
                      (p.kred + GemmCfg<kBwd>::kBK - 1) / GemmCfg<kBwd>::kBK, ncl, skb);
  }
  const unsigned long long epoch = *reinterpret_cast<volatile unsigned long long*>(p.epoch) + 1ull;
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total_rows = so[p.num_segs];
  const int num_m = (total_rows + kPairRows - 1) / kPairRows;
  // the task groups of every pair row block, once per launch (the producer and the MMA issuer
  // would otherwise each rebuild them per tile on their critical path)
  const bool tab_ok = num_m <= kGroupTab;
  const bool carry = kCarry && p.carry && p.has_main && p.has_side;
  if (tab_ok || carry) {
    int gm = 0;
    for (int m = threadIdx.x; m < num_m; m += blockDim.x) {
      const PairGroups g = pair_groups(p, so, m);
      if (tab_ok) gtab[m] = make_uint2(g.seg4, g.hm4 | (static_cast<uint32_t>(g.n) << 24));
      gm = max(gm, g.n);
    }
    if (carry && gm > 0) atomicMax(s_gmax, gm);
  }
  __syncthreads();
  // carrier mode: nc carrier tiles per row block, each carrying gpc task groups (32 stacked rows).
  // Carriers are used only when all of them are first items of their clusters (one wave): with
  // nc > 1 a carrier's extension blocks wait for every carrier of its row block, which is
  // deadlock-free only then; and a carrier that is a cluster's second item waits for the previous
  // tile's epilogue before its shrink can use the other accumulator (measured: 84 row blocks on 74
  // pairs, carriers 0.3-3.6 % slower than side tiles, profiles/r02_carry4_envab_tp.jsonl).
  // Otherwise this launch runs side tiles (same decision in every CTA: it depends on seg_off only).
  const int gpc = carry ? kShrinkRows * 2 / p.r_cap : 1;
  int nc = carry ? max(1, (*s_gmax + gpc - 1) / gpc) : 0;
  if (num_m * nc > ncl && !(p.carry == 2 && nc == 1)) nc = 0;  // carry 2: one carrier may span waves
  auto groups_of = [&](int m) -> PairGroups {
    if (!tab_ok) return pair_groups(p, so, m);
    const uint2 e = gtab[m];
    PairGroups g;
    g.seg4 = e.x;
    g.hm4 = e.y & 0xFFFFu;
    g.n = static_cast<int>(e.y >> 24);
    return g;
  };
  const int num_n = (p.nout + kTileN - 1) / kTileN;
  const int side_lo = min(p.side_m_lo, num_m);
  const int total_tiles = p.has_main ? num_m * (num_n + (p.has_side && nc == 0 ? 1 : 0))
                                     : max(0, min(p.side_m_hi, num_m) - side_lo);
  const int num_kb = (p.kred + kBK - 1) / kBK;  // a partial last block reads TMA zero fill

#ifdef MUX_PROFILE
  long long pw_empty = 0, mw_full = 0, mw_tempty = 0, ew_tfull = 0;
  long long p_setup = 0, p_issue = 0, p_flag = 0, e_store = 0, n_tiles = 0;
  const long long t_role0 = clock64();
#endif
  if (warp == 0) {
    // =========================== TMA producer (both CTAs) ===============
    // Warp-uniform loop; one elected lane issues (operands stay in uniform
    // registers: the producer's issue rate bounds the pipeline).
    {
      int stage = 0;
      uint32_t phase = 0;
      auto advance = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      };
      const int rk = static_cast<int>(crank);
      const uint32_t pipe_u = smem_u32(pipe);
      const uint32_t full_u = smem_u32(full_bar);
      const uint32_t full_leader = mapa_shared(full_u, 0);  // stage s barrier: + 8 s
      uint32_t ag_ok = 0;  // owners whose rows have landed in the gather buffer (fused all-gather)
      for_each_item(p, cid, ncl, num_m, num_n, side_lo, total_tiles, num_kb, skb, nc, [&](const Tile& tl, const SkPiece& pc) {
        PROF_T0(ts_);
        const PairGroups g = groups_of(tl.m);
        const int row_c = tl.m * kPairRows + kBM * rk;  // this CTA's rows
        if (p.ag_world > 0) {
          const int owner = (tl.m * kPairRows) / p.ag_rows;
          if (!((ag_ok >> owner) & 1u)) {
            if (elect_one_sync()) {
              const unsigned long long* f = p.ag_flags + owner;
              if (ld_acquire_sys_u64(f) < p.ag_seq) {
                const uint64_t t0 = globaltimer_ns();
                while (ld_acquire_sys_u64(f) < p.ag_seq)
                  if (peer_wait_expired(t0, p.peer_wait_ns)) __trap();
              }
              fence_async_global();  // the rows the copy engine wrote -> this CTA's TMA reads
            }
            __syncwarp();
            ag_ok |= 1u << owner;
          }
        }
        if (tl.side) {
          // units (task group gi, slice pair sp), two per pass: CTA rk stages slice 2 sp + rk of
          // the group's adapter (a missing slice or a rank-0 slot: rows >= 64, all zero fill)
          const int S = p.num_slices;
          const int nsp = (S + 1) >> 1;
          const int nunits = g.n * nsp;
          for (int u0 = 0; u0 < nunits; u0 += 2) {
            const int nu = min(2, nunits - u0);
            int slot[2], jrow[2], coff[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int u = min(u0 + i, nunits - 1);
              const int gi = u / nsp;
              const int s = 2 * (u - gi * nsp) + rk;
              const int base = p.seg_adapter[g.seg(gi)] * S;
              slot[i] = base + (s < S ? s : 0);
              jrow[i] = (s < S && p.slot_rank[base + s] > 0) ? 0 : 64;
              coff[i] = s < S ? p.slice_off[s] : 0;
            }
            for (int kb = 0; kb < num_kb; ++kb) {
              PROF_T0(tw_);
              mbar_wait(&empty_bar[stage], phase ^ 1u);
              PROF_ADD(pw_empty, tw_);
              if (elect_one_sync()) {
                const uint32_t sa = pipe_u + stage * kStageBytes;
                const uint32_t sb = sa + kStageA;
                const uint32_t fbl = full_leader + 8u * stage;
                if (leader) mbar_arrive_expect_tx_u32(full_u + 8u * stage, 2u * (kStageA + nu * kSideGrp));
                const int k0 = kb * kBK;
#pragma unroll
                for (int s2 = 0; s2 < kKSub; ++s2) tma_load_2d_pair_u32(&p.map_a, fbl, sa + s2 * kSubA, k0 + 64 * s2, row_c);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  if (i >= nu) break;
#pragma unroll
                  for (int s2 = 0; s2 < kKSub; ++s2) {
                    const uint32_t dst = sb + i * kSideGrp + s2 * kBox;
                    if (!kBwd)  // A_{t,s} [r, K] K-major rows j
                      tma_load_2d_pair_u32(&p.map_lora_a[slot[i]], fbl, dst, k0 + 64 * s2, jrow[i]);
                    else        // B_{t,s} [n_s, r] read MN-major {64 j, 64 n}: rows outside the slice are zero fill
                      tma_load_2d_pair_u32(&p.map_lora_b[slot[i]], fbl, dst, jrow[i], k0 + 64 * s2 - coff[i]);
                  }
                }
              }
              __syncwarp();
              advance();
            }
          }
        } else {
          // this CTA's B columns: box i covers output columns bcol(i) .. +63 (standard / narrow: the
          // CTA's half of the tile; wide: the CTA's half of each 256-column MMA half)
          const int col_c = tl.n * kTileN + (kWide ? 128 : kTileN / 2) * rk;
          auto bcol = [&](int i) { return col_c + 256 * (i >> 1) + 64 * (i & 1); };
          // carrier: this CTA stages stacked adapter rows [16 rk, 16 rk + 16) of the carried groups
          // (group gl at stacked rows gl * r_cap ..): fwd two {64 k x 8 rows} boxes, bwd one
          // {16 j x 128 n} box; rows of a group this carrier does not have are not loaded (their MMA
          // columns are never read)
          constexpr int kUnits = kBwd ? 1 : 2;
          constexpr uint32_t kUnitBytes = kBwd ? Ly::kShrinkStage : 8 * 128;
          int sh_slot[2] = {0, 0}, sh_row[2] = {0, 0};
          uint32_t sh_mask = 0u, sh_bytes = 0u;  // this CTA's live units; both CTAs' bytes (leader)
          if (kCarry && tl.carrier) {
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
              for (int s8 = 0; s8 < kUnits; ++s8) {
                const int i = kShrinkRows * c2 + 8 * s8;
                const int gl = i / p.r_cap;
                const int gi = tl.n * gpc + gl;
                if (gi >= g.n) continue;
                sh_bytes += kUnitBytes;
                if (c2 == rk) {
                  sh_mask |= 1u << s8;
                  sh_slot[s8] = p.seg_adapter[g.seg(gi)];
                  sh_row[s8] = i - gl * p.r_cap;
                }
              }
          }
          PROF_ADD(p_setup, ts_);
#ifdef MUX_PROFILE
          ++n_tiles;
#endif
          for (int kb = pc.k0; kb < pc.k1; ++kb) {
            PROF_T0(tw_);
            mbar_wait(&empty_bar[stage], phase ^ 1u);
            PROF_ADD(pw_empty, tw_);
            PROF_T0(ti_);
            if (elect_one_sync()) {
              const uint32_t sa = pipe_u + stage * kStageBytes;
              const uint32_t sb = sa + kStageA;
              const uint32_t fbl = full_leader + 8u * stage;
              if (leader)
                mbar_arrive_expect_tx_u32(full_u + 8u * stage, 2u * (kStageA + kKSub * kHalves * kBox) + sh_bytes);
              const int k0 = kb * kBK;
              if (kCarry) {
                const uint32_t sh = smem_u32(shrink_area) + stage * Ly::kShrinkStage;
#pragma unroll
                for (int s8 = 0; s8 < kUnits; ++s8)
                  if ((sh_mask >> s8) & 1u) {
                    if (!kBwd)  // A_t rows j .. j + 7, k-columns k0 .. k0 + 63
                      tma_load_2d_pair_u32(&p.map_shrink[sh_slot[s8]], fbl, sh + s8 * 1024u, k0, sh_row[s8]);
                    else        // B_t columns j .. j + 15 of rows n = k0 .. k0 + 127
                      tma_load_2d_pair_u32(&p.map_shrink[sh_slot[s8]], fbl, sh, sh_row[s8], k0);
                  }
              }
#pragma unroll
              for (int s2 = 0; s2 < kKSub; ++s2) {
                tma_load_2d_pair_u32(&p.map_a, fbl, sa + s2 * kSubA, k0 + 64 * s2, row_c);
#pragma unroll
                for (int i = 0; i < kHalves; ++i) {
                  if (!kBwd)  // W [N, K] K-major rows n: k-subtile s2, rows 64i..
                    tma_load_2d_pair_u32(&p.map_w, fbl, sb + s2 * kBSub + i * kBox, k0 + 64 * s2, bcol(i));
                  else        // W viewed [k_out (MN), n (red)]: atom i, K-rows 64*s2..
                    tma_load_2d_pair_u32(&p.map_w, fbl, sb + i * kAtomMN + s2 * kBox, bcol(i), k0 + 64 * s2);
                }
              }
            }
            __syncwarp();
            PROF_ADD(p_issue, ti_);
            advance();
          }
          PROF_T0(tf_);
#ifdef MUX_DIAG_NO_FLAG
          if (false) {  // timing-only diagnostic: no wait for the shrink tile (results may race)
#else
          if (pc.fin && g.n > 0 && p.has_side) {
#endif
            // the side tile (carrier mode: every carrier) of this row block must have published
            // Hs/Gs (a caller-given Hs was written by an earlier kernel in stream order).  (Polling
            // it from the idle warp 3 ahead of time and handing it over through an mbarrier was
            // measured: no gain, profiles/r02_fok_ab_cfg2.jsonl.)
            if (elect_one_sync()) {
              const unsigned long long* flag = p.flags + tl.m;
              // row-block flags are plain counters (8 epilogue warps per shrink tile / carrier),
              // reset to 0 by the last CTA of every launch
              const unsigned long long want = 8ull * static_cast<unsigned long long>(nc > 0 ? nc : 1);
              if (ld_acquire_gpu_u64(flag) != want) {
                const uint64_t t0 = globaltimer_ns();
                while (ld_acquire_gpu_u64(flag) != want) {
                  if (globaltimer_ns() - t0 > kWatchdogNs) __trap();
                }
              }
              fence_async_global();
            }
            __syncwarp();
          }
          PROF_ADD(p_flag, tf_);
          // LoRA expand (the tile's final piece only): one extension block per (task group, slice
          // with an adapter on this tile); reduction = the slot's rank (<= 64): first k-subtile only
          const int S = p.num_slices;
          const int tc0 = tl.n * kTileN, tc1 = tc0 + kTileN;
          for (int i = 0; i < (pc.fin ? g.n : 0); ++i) {
            for (int s = 0; s < S; ++s) {
              const int slot = p.seg_adapter[g.seg(i)] * S + s;
              if (!ext_live<kBwd>(p, slot, s, tc0, tc1)) continue;
              PROF_T0(tw_);
              mbar_wait(&empty_bar[stage], phase ^ 1u);
              PROF_ADD(pw_empty, tw_);
              if (elect_one_sync()) {
                const uint32_t sa = pipe_u + stage * kStageBytes;
                const uint32_t sb = sa + kStageA;
                const uint32_t fbl = full_leader + 8u * stage;
                if (leader) mbar_arrive_expect_tx_u32(full_u + 8u * stage, 2u * (kSubA + kHalves * kBox));
                tma_load_2d_pair_u32(&p.map_side, fbl, sa, s * p.r_cap, row_c);
#pragma unroll
                for (int j = 0; j < kHalves; ++j) {
                  if (!kBwd)  // B_{t,s} [n_s, r] K-major rows n: box {64 j, 64 n}, zero fill outside the slice
                    tma_load_2d_pair_u32(&p.map_lora_b[slot], fbl, sb + j * kBox, 0, bcol(j) - p.slice_off[s]);
                  else        // A_{t,s} [r, K] viewed [k_out (MN), j (red)]: atom j, K-rows 0..63
                    tma_load_2d_pair_u32(&p.map_lora_a[slot], fbl, sb + j * kAtomMN, bcol(j), 0);
                }
              }
              __syncwarp();
              advance();
            }
          }
        }
      });
    }
  } else if (warp == 1) {
    // =========================== MMA issuer (leader CTA) ================
    // The whole warp runs the loop (warp-uniform values stay in uniform
    // registers); one elected lane issues tcgen05.mma / tcgen05.commit.
    if (leader) {
      constexpr uint32_t kIdescMain = idesc_bf16(kPairRows, kWide ? 256 : kTileN, false, kBwd);
      // wide tiles: the second N = 256 MMA reads rows 128.. of this CTA's B share and writes TMEM
      // columns 256..
      constexpr uint32_t kBHalf2 = (kBwd ? 2 * kAtomMN : 2 * kBox) >> 4;
      constexpr uint32_t kIdescSide = idesc_bf16(kPairRows, kSideN, false, kBwd);
      // B operand per CTA: K-major rows of 128 B (SBO 1024), or MN-major atoms
      // of 64 elements x 64 K-rows (LBO 8 KB between atoms, SBO 1024).
      constexpr uint32_t kBLbo = kBwd ? kAtomMN : 16;
      // start-address offset (16 B units) of k-step k (16 reduction elements)
      auto a_off = [](int k) -> uint32_t { return ((k >> 2) * kSubA + (k & 3) * 32) >> 4; };
      auto b_off = [](int k) -> uint32_t {
        return kBwd ? (k * 16 * 128) >> 4 : ((k >> 2) * kBSub + (k & 3) * 32) >> 4;
      };
      auto side_b_off = [](int k) -> uint32_t {
        return kBwd ? (k * 16 * 128) >> 4 : ((k >> 2) * kBox + (k & 3) * 32) >> 4;
      };
      constexpr uint32_t kHi = desc_hi(1024);
      const uint32_t pipe_s = smem_u32(pipe);
      const uint32_t a_lo0 = desc_lo(pipe_s, 16);
      const uint32_t b_lo0 = desc_lo(pipe_s + kStageA, kBLbo);
      constexpr uint32_t kStageStep = kStageBytes >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      bool prev_carrier = false;
      uint32_t se_phase = 0;
      // carrier shrink: M = 256, N = 32 (16 stacked adapter rows per CTA), both operands K-major
      constexpr uint32_t kIdescShrink = idesc_bf16(kPairRows, 2 * kShrinkRows, false, kBwd);
      // fwd: K-major 128 B swizzle (8-row groups 1 KB apart); bwd: MN-major 32 B swizzle, one atom of 16
      // columns, 8-row groups 256 B apart, a k-step (16 rows) = 512 B
      constexpr uint32_t kShHi = kBwd ? desc_hi_sw32(256) : desc_hi(1024);
      const uint32_t sh_lo0 = desc_lo(smem_u32(shrink_area), 16);
      auto advance = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      };
      for_each_item(p, cid, ncl, num_m, num_n, side_lo, total_tiles, num_kb, skb, nc, [&](const Tile& tl, const SkPiece& pc) {
        const PairGroups g = groups_of(tl.m);
        PROF_T0(tw_);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1u);
        if (kCarry && prev_carrier) {  // the previous carrier's shrink sat in this accumulator
          mbar_wait(sempty_bar, se_phase);
          se_phase ^= 1u;
        }
        if (kCarry && tl.carrier)  // this carrier's shrink goes to the other accumulator: wait for the
          mbar_wait(&tempty_bar[acc ^ 1], (acc ? acc_phase ^ 1u : acc_phase) ^ 1u);  // previous tile's drain
        prev_carrier = kCarry && tl.carrier;
        PROF_ADD(mw_tempty, tw_);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
        if (tl.side) {
          // units (task group, slice pair sp) as staged by the producer: slice pair sp accumulates
          // into TMEM columns [128 sp, 128 sp + 128) (slice s at 64 s), masked to the group's rows
          const int nsp = (p.num_slices + 1) >> 1;
          const int nunits = g.n * nsp;
          for (int u0 = 0; u0 < nunits; u0 += 2) {
            const int nu = min(2, nunits - u0);
            uint32_t mk[2][8];
            uint32_t dcol[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int u = min(u0 + i, nunits - 1);
              const int gi = u / nsp;
              lane_masks(i < nu ? g.hm(gi) : 0, mk[i]);
              dcol[i] = static_cast<uint32_t>(128 * (u - gi * nsp));
            }
            for (int kb = 0; kb < num_kb; ++kb) {
              PROF_T0(tw_);
              mbar_wait(&full_bar[stage], phase);
              PROF_ADD(mw_full, tw_);
              tc_fence_after();
              const uint32_t a_lo = a_lo0 + stage * kStageStep;
              const uint32_t b_lo = b_lo0 + stage * kStageStep;
              if (elect_one_sync()) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  if (i >= nu) break;
#pragma unroll
                  for (int k = 0; k < kBK / 16; ++k)
                    mma_bf16_pair(d_tmem + dcol[i], make_desc(a_lo + a_off(k), kHi),
                                  make_desc(b_lo + i * (kSideGrp >> 4) + side_b_off(k), kHi), kIdescSide,
                                  (kb | k) != 0, mk[i]);
                }
                mma_commit_pair_mc(&empty_bar[stage], kPairMask);
              }
              __syncwarp();
              advance();
            }
          }
        } else {
          if constexpr (kWide) {
            // Wide tiles: one accumulator, drained by the epilogue in two halves (tempty_bar[0] after
            // columns 0-255, tempty_bar[1] after 256-511).  The tile starts as soon as half 0 is free
            // (waited above); the second half's MMAs of the first k-blocks are held back — their
            // stages stay occupied, up to kStages - 1 of them — until half 1 has drained, so the
            // previous tile's epilogue overlaps this tile's first k-blocks.
            const uint32_t h1_bar = smem_u32(&tempty_bar[1]);
            bool h1 = false;
            int pend = 0, pst = 0, pkb = 0;
            auto h1_mmas = [&](int st, int kbb) {
              const uint32_t a2 = a_lo0 + st * kStageStep;
              const uint32_t b2 = b_lo0 + st * kStageStep + kBHalf2;
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                mma_bf16_pair_nomask(d_tmem + 256, make_desc(a2 + a_off(k), kHi), make_desc(b2 + b_off(k), kHi),
                                     kIdescMain, (kbb | k) != 0);
              mma_commit_pair_mc(&empty_bar[st], kPairMask);
            };
            auto flush = [&]() {  // half 1 is free: its held-back MMAs, oldest stage first
              for (int i = 0; i < pend; ++i) {
                int st = pst + i;
                if (st >= kStages) st -= kStages;
                if (elect_one_sync()) h1_mmas(st, pkb + i);
                __syncwarp();
              }
              pend = 0;
            };
            for (int kb = 0; kb < num_kb; ++kb) {
              PROF_T0(tw_);
              mbar_wait(&full_bar[stage], phase);
              PROF_ADD(mw_full, tw_);
              tc_fence_after();
              const uint32_t a_lo = a_lo0 + stage * kStageStep;
              const uint32_t b_lo = b_lo0 + stage * kStageStep;
              if (elect_one_sync()) {
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                  mma_bf16_pair_nomask(d_tmem, make_desc(a_lo + a_off(k), kHi), make_desc(b_lo + b_off(k), kHi),
                                       kIdescMain, (kb | k) != 0);
              }
              __syncwarp();
              if (!h1) {
                h1 = __all_sync(0xffffffffu, mbar_test_wait(h1_bar, acc_phase ^ 1u));
                if (!h1 && pend == kStages - 1) {
                  mbar_wait(&tempty_bar[1], acc_phase ^ 1u);
                  h1 = true;
                }
                if (h1) {
                  tc_fence_after();
                  flush();
                }
              }
              if (h1) {
                if (elect_one_sync()) h1_mmas(stage, kb);
                __syncwarp();
              } else {
                if (pend == 0) { pst = stage; pkb = kb; }
                ++pend;
              }
              advance();
            }
            if (!h1) {
              mbar_wait(&tempty_bar[1], acc_phase ^ 1u);
              tc_fence_after();
              flush();
            }
          } else {
          for (int kb = pc.k0; kb < pc.k1; ++kb) {
            PROF_T0(tw_);
            mbar_wait(&full_bar[stage], phase);
            PROF_ADD(mw_full, tw_);
            tc_fence_after();
            const uint32_t a_lo = a_lo0 + stage * kStageStep;
            const uint32_t b_lo = b_lo0 + stage * kStageStep;
            if (elect_one_sync()) {
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                mma_bf16_pair_nomask(d_tmem, make_desc(a_lo + a_off(k), kHi), make_desc(b_lo + b_off(k), kHi),
                                     kIdescMain, ((kb - pc.k0) | k) != 0);
              if (kCarry && tl.carrier) {  // the shrink from the same A stage into the other accumulator
                const uint32_t s_lo = sh_lo0 + stage * (Ly::kShrinkStage >> 4);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                  mma_bf16_pair_nomask(tmem_base + static_cast<uint32_t>((acc ^ 1) * kBN),
                                       make_desc(a_lo + a_off(k), kHi),
                                       make_desc(s_lo + (kBwd ? (k * 512) >> 4 : ((k & 3) * 32) >> 4), kShHi),
                                       kIdescShrink, (kb | k) != 0);
              }
              mma_commit_pair_mc(&empty_bar[stage], kPairMask);
            }
            __syncwarp();
            advance();
          }
          if (kCarry && tl.carrier) {  // shrink complete: the epilogue publishes Hs before the extension
            if (elect_one_sync()) mma_commit_pair_mc(sfull_bar, kPairMask);
            __syncwarp();
          }
          }
          // LoRA expand: the tile's final piece only, the producer's (group, live slice) blocks
          const int S = p.num_slices;
          const int tc0 = tl.n * kTileN, tc1 = tc0 + kTileN;
          for (int i = 0; i < (pc.fin ? g.n : 0); ++i) {
            uint32_t mk[8];
            lane_masks(g.hm(i), mk);
            for (int s = 0; s < S; ++s) {
              const int slot = p.seg_adapter[g.seg(i)] * S + s;
              if (!ext_live<kBwd>(p, slot, s, tc0, tc1)) continue;
              PROF_T0(tw_);
              mbar_wait(&full_bar[stage], phase);
              PROF_ADD(mw_full, tw_);
              tc_fence_after();
              const uint32_t a_lo = a_lo0 + stage * kStageStep;
              const uint32_t b_lo = b_lo0 + stage * kStageStep;
              const int nk = (p.slot_rank[slot] + 15) / 16;
              if (elect_one_sync()) {
                for (int k = 0; k < nk; ++k) {
                  mma_bf16_pair(d_tmem, make_desc(a_lo + a_off(k), kHi), make_desc(b_lo + b_off(k), kHi),
                                kIdescMain, 1u, mk);
                  if (kWide)
                    mma_bf16_pair(d_tmem + 256, make_desc(a_lo + a_off(k), kHi),
                                  make_desc(b_lo + kBHalf2 + b_off(k), kHi), kIdescMain, 1u, mk);
                }
                mma_commit_pair_mc(&empty_bar[stage], kPairMask);
              }
              __syncwarp();
              advance();
            }
          }
        }
        if (elect_one_sync()) mma_commit_pair_mc(&tfull_bar[acc], kPairMask);
        __syncwarp();
        if (++acc == kAccs) { acc = 0; acc_phase ^= 1u; }
      });
    }
  } else if (warp >= 4) {
    // =========================== epilogue (both CTAs) ===================
    const int q = warp & 3;  // TMEM lane quadrant = this CTA's rows 32q .. 32q+31
    if (p.rs_world > 0 && p.has_main) {
      // fused reduce-scatter: every destination rank must have consumed the previous call's
      // partials from its receive slot before this call overwrites them
      if (lane == 0) {
        for (int d = 0; d < p.rs_world; ++d) {
          const unsigned long long* f = p.rs_ack + d;
          if (ld_acquire_sys_u64(f) + 1ull < p.rs_seq) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_sys_u64(f) + 1ull < p.rs_seq)
              if (peer_wait_expired(t0, p.peer_wait_ns)) __trap();
          }
        }
      }
      __syncwarp();
    }
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t sf_phase = 0;
    uint8_t* bufs = epi + q * kEpiBufs * kEpiBuf;
    int buf_sel = 0;
    for_each_item(p, cid, ncl, num_m, num_n, side_lo, total_tiles, num_kb, skb, nc, [&](const Tile& tl, const SkPiece& pc) {
      const int row_w = tl.m * kPairRows + kBM * static_cast<int>(crank) + 32 * q;  // first row of this warp
      const uint32_t t_addr = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(acc * kBN);
      if (!(kCarry && tl.carrier)) {
        PROF_T0(tw_);
        mbar_wait(&tfull_bar[acc], acc_phase);
        PROF_ADD(ew_tfull, tw_);
        tc_fence_after();
      } else {
        // carrier: its shrink (other accumulator, columns [gl * r_cap, ..) for carried group gl) is
        // complete after the main k-loop; publish Hs rows of the carried groups (carrier 0 also
        // writes the zero rows of segments without an adapter) before this tile's extension blocks
        mbar_wait(sfull_bar, sf_phase);
        sf_phase ^= 1u;
        tc_fence_after();
        uint32_t v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>((acc ^ 1) * kBN), v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(sempty_bar), 0));
        const int row = row_w + lane;
        if (row < total_rows) {
          const PairGroups g = groups_of(tl.m);
          const int seg = seg_containing(so, p.num_segs, row);
          int gi = -1;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i < g.n && g.seg(i) == seg) gi = i;
          if ((gi >= 0 ? gi / gpc : 0) == tl.n) {
            const int gl = gi >= 0 ? gi - tl.n * gpc : 0;
            const int rank = gi >= 0 ? p.slot_rank[p.seg_adapter[seg]] : 0;
            const float sc = gi >= 0 ? p.slot_scale[p.seg_adapter[seg]] : 0.f;
            uint4* dst = reinterpret_cast<uint4*>(p.side_out + static_cast<size_t>(row) * p.r_cap);
#pragma unroll
            for (int j0 = 0; j0 < 32; j0 += 8) {
              if (j0 < p.r_cap) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int j = j0 + 2 * e;
                  // group gl's column j: stacked column gl * r_cap + j (gl = 1 only when r_cap = 16)
                  const uint32_t a = (gl != 0 && j < 16) ? v[16 + (j & 15)] : v[j];
                  const uint32_t b = (gl != 0 && j + 1 < 16) ? v[16 + ((j + 1) & 15)] : v[j + 1];
                  const float lo = j < rank ? __uint_as_float(a) * sc : 0.f;
                  const float hi = j + 1 < rank ? __uint_as_float(b) * sc : 0.f;
                  w[e] = pack_bf16x2(lo, hi);
                }
                dst[j0 / 8] = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
          }
        }
        fence_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) red_add_release_gpu_u64(p.flags + tl.m, 1ull);
        PROF_T0(tw2_);
        mbar_wait(&tfull_bar[acc], acc_phase);
        PROF_ADD(ew_tfull, tw2_);
        tc_fence_after();
      }
      const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty_bar[acc]), 0);
      // wide tiles: the second half of the accumulator has its own barrier (see the MMA issuer)
      const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty_bar[1]), 0);
      if (tl.side) {
        // slice sl of the shrink sits in TMEM columns [64 sl, 64 sl + 64) -> Hs/Gs columns
        // [sl * r_cap, sl * r_cap + r_cap), scaled by the row's task's s_{t,sl}
        const int row = row_w + lane;
        const int S = p.num_slices;
        const int seg = row < total_rows ? seg_containing(so, p.num_segs, row) : -1;
        const size_t ld = static_cast<size_t>(S) * p.r_cap;
        for (int sl = 0; sl < S; ++sl) {
          uint32_t v0[32], v1[32];
          tmem_ld32(t_addr + 64 * sl, v0);
          tmem_ld32(t_addr + 64 * sl + 32, v1);
          tmem_ld_wait();
          if (sl == S - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              mbar_arrive_cluster(tempty_leader);
              if (kWide) mbar_arrive_cluster(tempty_leader1);  // side tiles never touch half 1
            }
          }
          if (row < total_rows) {
            const int slot = seg >= 0 ? p.seg_adapter[seg] * S + sl : 0;
            const int rank = seg >= 0 ? p.slot_rank[slot] : 0;
            const float sc = seg >= 0 ? p.slot_scale[slot] : 0.f;
            uint4* dst = reinterpret_cast<uint4*>(p.side_out + static_cast<size_t>(row) * ld + sl * p.r_cap);
#pragma unroll
            for (int j0 = 0; j0 < 64; j0 += 8) {
              if (j0 < p.r_cap) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int j = j0 + 2 * e;
                  const uint32_t a = j < 32 ? v0[j & 31] : v1[j & 31];
                  const uint32_t b = j + 1 < 32 ? v0[(j + 1) & 31] : v1[(j + 1) & 31];
                  const float lo = j < rank ? __uint_as_float(a) * sc : 0.f;
                  const float hi = j + 1 < rank ? __uint_as_float(b) * sc : 0.f;
                  w[e] = pack_bf16x2(lo, hi);
                }
                dst[j0 / 8] = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
          }
        }
        fence_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) red_add_release_gpu_u64(p.flags + tl.m, 1ull);
      } else if (!pc.fin) {
        // stream-K partial (the first piece of this cluster's range): fp32 accumulator into this
        // cluster's slot, laid out [CTA][warp][col / 4][lane][4] so every access is coalesced
        float4* slot = reinterpret_cast<float4*>(p.sk_part + static_cast<size_t>(cid) * kSkSlotFloats +
                                                 (static_cast<size_t>(crank) * 4 + q) * (256 * 32));
#pragma unroll 1
        for (int c = 0; c < kTileN / 64; ++c) {
          uint32_t v0[32], v1[32];
          tmem_ld32(t_addr + c * 64, v0);
          tmem_ld32(t_addr + c * 64 + 32, v1);
          tmem_ld_wait();
          if (c == kTileN / 64 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader);
          }
#pragma unroll
          for (int g4 = 0; g4 < 16; ++g4) {
            const uint32_t* v = g4 < 8 ? v0 : v1;
            const int b = (g4 & 7) * 4;
            __stcg(slot + (c * 16 + g4) * 32 + lane, make_float4(__uint_as_float(v[b]), __uint_as_float(v[b + 1]),
                                                                 __uint_as_float(v[b + 2]), __uint_as_float(v[b + 3])));
          }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) flag_arrive(p.sk_flags + cid, epoch);
      } else {
        // stream-K: the later clusters whose ranges start inside this tile hold its other k-blocks
        const int t_end = (pc.tile + 1) * num_kb;
        if (p.sk) {
          if (lane == 0) {
            const unsigned long long want = (epoch << 8) | 8ull;
            for (int c2 = cid + 1; c2 < ncl && skb[c2] < t_end; ++c2) {
              if (skb[c2 + 1] == skb[c2]) continue;  // empty range: no partial
              const unsigned long long* f = p.sk_flags + c2;
              if (ld_acquire_gpu_u64(f) != want) {
                const uint64_t t0 = globaltimer_ns();
                while (ld_acquire_gpu_u64(f) != want)
                  if (globaltimer_ns() - t0 > kWatchdogNs) __trap();
              }
            }
          }
          __syncwarp();
        }
        const bool valid = row_w < total_rows;
        const int col_t = tl.n * kTileN;
#pragma unroll 1
        for (int c = 0; c < kTileN / 64; ++c) {
          uint32_t v0[32], v1[32];
          tmem_ld32(t_addr + c * 64, v0);
          tmem_ld32(t_addr + c * 64 + 32, v1);
          tmem_ld_wait();
          if (p.sk) {  // + the partials, ascending cluster order (deterministic)
            for (int c2 = cid + 1; c2 < ncl && skb[c2] < t_end; ++c2) {
              if (skb[c2 + 1] == skb[c2]) continue;
              const float4* src = reinterpret_cast<const float4*>(
                                      p.sk_part + static_cast<size_t>(c2) * kSkSlotFloats +
                                      (static_cast<size_t>(crank) * 4 + q) * (256 * 32)) + (c * 16) * 32 + lane;
#pragma unroll
              for (int g4 = 0; g4 < 16; ++g4) {
                const float4 x = __ldcg(src + g4 * 32);
                uint32_t* v = g4 < 8 ? v0 : v1;
                const int b = (g4 & 7) * 4;
                v[b] = __float_as_uint(__uint_as_float(v[b]) + x.x);
                v[b + 1] = __float_as_uint(__uint_as_float(v[b + 1]) + x.y);
                v[b + 2] = __float_as_uint(__uint_as_float(v[b + 2]) + x.z);
                v[b + 3] = __float_as_uint(__uint_as_float(v[b + 3]) + x.w);
              }
            }
          }
          if (kWide && c == kTileN / 128 - 1) {  // wide: half 0 drained, the next tile may start
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader);
          }
          if (c == kTileN / 64 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(kWide ? tempty_leader1 : tempty_leader);
          }
          uint8_t* buf = bufs + buf_sel * kEpiBuf;
          PROF_T0(tsw_);
          if (lane == 0) tma_store_wait_read<kEpiBufs - 1>();
          __syncwarp();
          PROF_ADD(e_store, tsw_);
          uint8_t* rowp = buf + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint32_t* v = ch < 4 ? v0 : v1;
            const int b = (ch & 3) * 8;
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(v[b + 0]), __uint_as_float(v[b + 1]));
            w.y = pack_bf16x2(__uint_as_float(v[b + 2]), __uint_as_float(v[b + 3]));
            w.z = pack_bf16x2(__uint_as_float(v[b + 4]), __uint_as_float(v[b + 5]));
            w.w = pack_bf16x2(__uint_as_float(v[b + 6]), __uint_as_float(v[b + 7]));
            *reinterpret_cast<uint4*>(rowp + ((ch ^ (lane & 7)) << 4)) = w;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            const int col = col_t + c * 64;
            if (valid && col < p.nout) {
              if (p.rs_world > 0) {  // the rows' owner rank receives this partial tile
                const int owner = row_w / p.rs_rows;
                tma_store_2d(&p.map_out_rs[owner], buf, col, row_w - owner * p.rs_rows);
              } else {
                tma_store_2d(&p.map_out, buf, col, row_w);
              }
            }
            tma_store_commit();
          }
          if (kEpiBufs == 2) buf_sel ^= 1;
        }
      }
      if (++acc == kAccs) { acc = 0; acc_phase ^= 1u; }
    });
    if (lane == 0) {
      tma_store_wait<0>();
      if (p.rs_world > 0) fence_async_global();  // bulk stores -> generic-proxy release below
    }
  }
#ifdef MUX_PROFILE
  {
    const long long tot = clock64() - t_role0;
    if (warp == 1 && leader && lane == 0) {
      atomicAdd(p.dbg + 0, static_cast<unsigned long long>(tot));
      atomicAdd(p.dbg + 1, static_cast<unsigned long long>(mw_full));
      atomicAdd(p.dbg + 2, static_cast<unsigned long long>(mw_tempty));
    }
    if (warp == 0 && lane == 0) {
      atomicAdd(p.dbg + 3, static_cast<unsigned long long>(tot));
      atomicAdd(p.dbg + 4, static_cast<unsigned long long>(pw_empty));
      atomicAdd(p.dbg + 7, static_cast<unsigned long long>(p_setup));
      atomicAdd(p.dbg + 8, static_cast<unsigned long long>(p_issue));
      atomicAdd(p.dbg + 9, static_cast<unsigned long long>(p_flag));
      atomicAdd(p.dbg + 11, static_cast<unsigned long long>(n_tiles));
    }
    if (warp == 4 && lane == 0) {
      atomicAdd(p.dbg + 5, static_cast<unsigned long long>(tot));
      atomicAdd(p.dbg + 6, static_cast<unsigned long long>(ew_tfull));
      atomicAdd(p.dbg + 10, static_cast<unsigned long long>(e_store));
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 0) {
    // the last CTA out advances the workspace epoch for the next launch (and, for a fused
    // reduce-scatter, tells every destination rank that this rank's partials have landed)
    if (p.rs_world > 0) __threadfence_system();
    else __threadfence();
    if (atomicAdd(p.done, 1u) == gridDim.x - 1) {
      __threadfence();  // every CTA's flag arrivals are ordered before this reset
      *p.done = 0u;
      for (int m = 0; m < num_m; ++m) p.flags[m] = 0ull;
      *reinterpret_cast<volatile unsigned long long*>(p.epoch) = epoch;
      __threadfence_system();
      for (int d = 0; d < p.rs_world; ++d) st_release_sys_u64(p.rs_ready[d], p.rs_seq);
    }
  }
}

// ---------------------------------------------------------------- launchers
template <bool kBwd, int kTileN>
cudaError_t launch_gemm_impl(const GemmParams& p, int grid, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t ce = once_per_device(configured, [] {
    return cudaFuncSetAttribute(mux_gemm_kernel<kBwd, kTileN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(GemmLayout<kBwd, kTileN>::kSmemBytes));
  });
  if (ce != cudaSuccess) return ce;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = GemmLayout<kBwd, kTileN>::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mux_gemm_kernel<kBwd, kTileN>, p);
}

// grid must be even (clusters of 2); tile_n = output columns of a pair tile (128, 256 or 512)
cudaError_t launch_gemm(const GemmParams& p, bool bwd, int tile_n, int grid, cudaStream_t stream) {
  switch (tile_n) {
    case 128: return bwd ? launch_gemm_impl<true, 128>(p, grid, stream) : launch_gemm_impl<false, 128>(p, grid, stream);
    case 512: return bwd ? launch_gemm_impl<true, 512>(p, grid, stream) : launch_gemm_impl<false, 512>(p, grid, stream);
    default: return bwd ? launch_gemm_impl<true, 256>(p, grid, stream) : launch_gemm_impl<false, 256>(p, grid, stream);
  }
}

}  // namespace mux
