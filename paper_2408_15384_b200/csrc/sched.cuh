// sched.cuh — the persistent work schedule shared by the tcgen05 and FP64 kernels.
//
// Tiles of C are the units of the paper's row/column decomposition (each
// C[i][j] an independent dot product); a persistent grid of nc clusters
// (or CTAs) walks them.
#pragma once
#include <cstdint>

namespace mmb {

// Work schedule: every cluster first takes whole tiles round-robin (W full waves,
// grouped raster), then the tiles of the last, partial wave are split stream-K
// style: their (tile, k-block) iterations are cut into ntc equal ranges, one per
// cluster, so no SM idles through a ragged last wave (C3: 3.46 waves -> 3 + an
// even tail; C4: 55.35 -> 55 + tail).  The parts of a split tile take tickets as
// they finish; every part but the last publishes its partial tile, the last adds
// them in segment order (fixed order: deterministic).  No part waits for a cluster
// that may not have started, so the grid never relies on co-residency.
struct WorkSched {
  int tiles_m, tiles_n, group_m, num_kb;
  int nc;    // clusters
  int W;     // full data-parallel waves
  int ntc;   // clusters taking part in the stream-K tail (0 = no tail)
  int land;  // tail tiles split in exact halves: the last half lands the other's slab in its idle stage ring
  int red;   // tail tiles split in exact halves, both adding into C (zeroed first) by TMA reduce-add stores
  int nhalf; // tail tiles split in N halves (whole K each): cluster c < ntc takes half c & 1 of tail tile c / 2
  int64_t TI;  // tail iterations = tail tiles * num_kb

  __device__ __forceinline__ void tile_coords(int t, int& tm, int& tn) const {
    const int per_group = group_m * tiles_n;
    const int g = t / per_group;
    const int first_m = g * group_m;
    const int gm = min(tiles_m - first_m, group_m);
    const int r = t - g * per_group;
    tm = first_m + r % gm;
    tn = r / gm;
  }
  __device__ __forceinline__ int64_t tstart(int c) const { return ((int64_t)c * TI) / ntc; }
  __device__ __forceinline__ int tail_cluster_of(int64_t it) const {
    int c = (int)((it * ntc) / TI);
    while (c + 1 < ntc && tstart(c + 1) <= it) ++c;
    while (c > 0 && tstart(c) > it) --c;
    return c;
  }
  // N half of item j of cluster c (tail mode 4), or -1 for a whole-width item
  __device__ __forceinline__ int half_of(int c, int j) const { return (nhalf && j == W && c < ntc) ? (c & 1) : -1; }
  // j-th work item of cluster c: tile t, k-blocks [kb0, kb1). Returns false past the end.
  __device__ __forceinline__ bool item(int c, int j, int& t, int& kb0, int& kb1) const {
    if (j < W) {
      t = c + j * nc;
      kb0 = 0;
      kb1 = num_kb;
      return t < tiles_m * tiles_n;
    }
    if (c >= ntc) return false;
    if (nhalf) {
      if (j != W) return false;
      t = W * nc + c / 2;
      kb0 = 0;
      kb1 = num_kb;
      return true;
    }
    int64_t it = tstart(c);
    const int64_t end = tstart(c + 1);
    for (int s = 0; it < end; ++s) {
      const int64_t tt = it / num_kb;
      const int k0 = (int)(it - tt * num_kb);
      const int64_t lim = (tt + 1) * num_kb < end ? (tt + 1) * num_kb : end;
      if (s == j - W) {
        t = W * nc + (int)tt;
        kb0 = k0;
        kb1 = (int)(lim - tt * num_kb);
        return true;
      }
      it = lim;
    }
    return false;
  }
};

// Host: a schedule over tiles_m x tiles_n tiles of num_kb k-blocks for nc clusters.
//   tail_mode 0: whole tiles only (the last wave may be partial);
//   tail_mode 1: the tiles of the last partial wave split evenly over the clusters
//                (>= min_seg k-blocks per segment, <= 4 segments per tile);
//   tail_mode 2: the tail tiles split in exact halves (needs 2*tail <= nc);
//   tail_mode 3: the same halves, both added into C by TMA reduce-add (no partial slabs);
//   tail_mode 4: the tail tiles split in N halves, each with its whole K (needs 2*tail <= nc):
//                no partial sums at all, twice the clusters on the last round.
inline WorkSched sched_build(int tiles_m, int tiles_n, int group_m, int num_kb, int nc, int tail_mode, int min_seg = 4) {
  WorkSched s;
  s.tiles_m = tiles_m;
  s.tiles_n = tiles_n;
  s.group_m = group_m < 1 ? 1 : (group_m > tiles_m ? tiles_m : group_m);
  s.num_kb = num_kb;
  s.nc = nc < 1 ? 1 : nc;
  const int64_t T = (int64_t)tiles_m * tiles_n;
  s.W = (int)(T / s.nc);
  const int64_t tail = T - (int64_t)s.W * s.nc;
  s.TI = tail * num_kb;
  s.land = 0;
  s.red = 0;
  s.nhalf = 0;
  if (tail == 0 || tail_mode == 0 || (tail_mode >= 2 && 2 * tail > s.nc)) {
    s.W = (int)((T + s.nc - 1) / s.nc);
    s.ntc = 0;
    s.TI = 0;
  } else if (tail_mode >= 2) {
    s.ntc = (int)(2 * tail);  // exact halves: two parts per tile
    s.land = tail_mode == 2;
    s.red = tail_mode == 3;
    s.nhalf = tail_mode == 4;
    if (s.nhalf) s.TI = 0;
  } else {
    int64_t ntc = s.nc < tail * 4 ? s.nc : tail * 4;
    const int64_t cap = s.TI / (min_seg < 1 ? 1 : min_seg);
    ntc = ntc < cap ? ntc : cap;
    s.ntc = (int)(ntc < 1 ? 1 : ntc);
  }
  return s;
}

}  // namespace mmb
