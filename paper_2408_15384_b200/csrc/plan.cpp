// plan.cpp — the per-rank schedule of mm_gemm_sharded as data (include/mm.h, mm_shard_plan).
//
// Pure host logic: from the collective's arguments alone it lists, for rank r of G, the local
// products, pitched copies, NCCL collectives and stream events that rank runs.  shard.cu executes
// the list with NCCL on the GPU; the test suite executes the same list over gloo on CPU with the
// oracle as the local product, so every offset, pitch, root and ordering here is checked at world
// sizes the GPU box does not have.
//
// Layouts (PAPER.md:119 row partition of the outer loop, applied across processes; PAPER.md:135
// SUMMA and 2.5D):
//   ROW_BLOCK  rank r owns rows mm_shard_range(m, G, r) of A and C; B replicated — broadcast from
//              `root` in column panels (MM_BCAST_B) double-buffered against the products of the
//              previous panel; C gathered to the root by send/recv (MM_GATHER_C) or stored by each
//              rank's product kernel straight into the root's C_full (MM_GATHER_C_FUSED).
//   SUMMA_2D   grid_rows × grid_cols; k-panels never straddle an A column block or a B row block
//              (mm_summa_panels); panel t of A broadcast along grid row from its owner column, of B
//              along grid column from its owner row, double-buffered; C_ij (+)= A_i,t · B_t,j.
//   SUMMA_25D  c layers of that grid; layer l runs panels t ≡ l (mod c) and the layers' C blocks are
//              summed onto layer 0 (MM_REPLICATE: blocks valid on layer 0 only, broadcast along depth).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mm.h"
#include "knobs.h"

namespace {

struct Range {
  int64_t start, count;
};
Range shard(int64_t total, int G, int r) {
  Range x;
  mm_shard_range(total, G, r, &x.start, &x.count);
  return x;
}
int64_t esz_in(mm_dtype t) { return (t == MM_F64 || t == MM_F64_EMU) ? 8 : (t == MM_BF16_F32 ? 2 : 1); }
int64_t esz_out(mm_dtype t) { return (t == MM_F64 || t == MM_F64_EMU) ? 8 : 4; }

// event ids
enum { EV_START = 0, EV_END = 1, EV_READY0 = 2, EV_FREE0 = 4, EV_COUNT = 6 };

struct Builder {
  std::vector<mm_plan_step> v;
  mm_plan_step& add(int op, int stream = 0) {
    mm_plan_step s;
    memset(&s, 0, sizeof s);
    s.op = op;
    s.stream = stream;
    v.push_back(s);
    return v.back();
  }
  void record(int ev, int stream) { add(MM_OP_RECORD, stream).event = ev; }
  void wait(int stream, int ev) { add(MM_OP_WAIT, stream).event = ev; }
  void copy2d(int stream, int dst, int64_t doff, int64_t dpitch, int src, int64_t soff, int64_t spitch,
              int64_t width, int64_t rows) {
    mm_plan_step& s = add(MM_OP_COPY2D, stream);
    s.dst = dst, s.dst_off = doff, s.dst_ld = dpitch, s.src = src, s.src_off = soff, s.src_ld = spitch;
    s.n = width, s.m = rows;
  }
  void gemm(int64_t m, int64_t n, int64_t p, int A, int64_t aoff, int64_t lda, int B, int64_t boff, int64_t ldb,
            int C, int64_t coff, int64_t ldc, int beta, int overlap) {
    mm_plan_step& s = add(MM_OP_GEMM, 0);
    s.m = m, s.n = n, s.p = p, s.src = A, s.src_off = aoff, s.src_ld = lda, s.src2 = B, s.src2_off = boff;
    s.src2_ld = ldb, s.dst = C, s.dst_off = coff, s.dst_ld = ldc, s.beta = beta, s.overlap = overlap;
  }
  void coll(int op, int stream, int comm, int peer, int buf, int64_t off, int64_t count) {
    mm_plan_step& s = add(op, stream);
    s.comm = comm, s.peer = peer, s.n = count;
    if (op == MM_OP_SEND) s.src = buf, s.src_off = off;
    else s.dst = buf, s.dst_off = off;
  }
};

// Default column-panel width of the B broadcast: p/8, a 16-element multiple (every panel pitch
// 16-B aligned for TMA).  MM_F64_EMU: p/2 — each panel is a separate emulated product whose
// fixed costs (the residues of the whole local A, the reconstruction) do not shrink with its width.
int64_t bcast_panel(int64_t p, int64_t panel, mm_dtype dt) {
  int64_t w = panel;
  if (w <= 0) {
    int64_t npan = dt == MM_F64_EMU ? 2 : 8;
    if (const char* e = mmb::knob("MM_BCAST_PANELS")) npan = std::max<int64_t>(1, atoll(e));  // tuning knob
    w = (p + npan - 1) / npan;
  }
  w = (w + 15) / 16 * 16;
  return std::min(w, p);
}
// Default k-panel width of SUMMA: 2048; MM_F64_EMU: 8192 (every panel's emulated product
// reconstructs the whole local C block, so fewer, wider panels)
int64_t summa_panel(int64_t panel, mm_dtype dt) {
  if (panel > 0) return panel;
  int64_t w = dt == MM_F64_EMU ? 8192 : 2048;
  if (const char* e = mmb::knob("MM_SUMMA_PANEL")) w = std::max<int64_t>(16, atoll(e));  // tuning knob
  return w;
}

void row_block(Builder& b, mm_plan_info* info, int64_t m, int64_t n, int64_t p, mm_dtype dt, unsigned flags,
               int root, int G, int r, int64_t panel) {
  const int64_t ei = esz_in(dt), eo = esz_out(dt);
  const Range mine = shard(m, G, r);
  int target = MM_BUF_C;
  int64_t toff = 0;
  if (flags & MM_GATHER_C_FUSED) {
    // GEMM -> gather as one kernel per rank: the product stores its C tiles into the root's C_full
    b.add(MM_OP_MAP_PEER).peer = root;
    target = MM_BUF_CPEER;
    toff = mine.start * p * eo;
  }
  if (flags & MM_BCAST_B) {
    const int64_t w = bcast_panel(p, panel, dt);
    const int64_t J = (p + w - 1) / w;
    info->stage_bytes[0] = info->stage_bytes[1] = n * w * ei;
    b.record(EV_START, 0);
    b.wait(1, EV_START);
    for (int64_t j = 0; j < J; ++j) {
      const int s = (int)(j & 1);
      const int stage = MM_BUF_S0 + s;
      const int64_t c0 = j * w, wj = std::min(w, p - c0);
      if (j >= 2) b.wait(1, EV_FREE0 + s);  // the product of panel j-2 has consumed this buffer
      if (r == root) b.copy2d(1, stage, 0, wj * ei, MM_BUF_B, c0 * ei, p * ei, wj * ei, n);
      b.coll(MM_OP_BCAST, 1, MM_COMM_WORLD, root, stage, 0, n * wj * ei);
      // keep "B_local holds B afterwards" on every rank (off the critical path)
      if (r != root) b.copy2d(1, MM_BUF_B, c0 * ei, p * ei, stage, 0, wj * ei, wj * ei, n);
      b.record(EV_READY0 + s, 1);
      b.wait(0, EV_READY0 + s);
      if (mine.count > 0)
        b.gemm(mine.count, n, wj, MM_BUF_A, 0, n, stage, 0, wj, target, toff + c0 * eo, p, 0, 1);
      b.record(EV_FREE0 + s, 0);
    }
    b.record(EV_END, 1);
    b.wait(0, EV_END);
  } else if (mine.count > 0) {
    b.gemm(mine.count, n, p, MM_BUF_A, 0, n, MM_BUF_B, 0, p, target, toff, p, 0, 0);
  }
  if (flags & MM_GATHER_C_FUSED) {
    // the root's C_full is complete once every rank's products have finished
    b.add(MM_OP_BARRIER).comm = MM_COMM_WORLD;
  } else if (flags & MM_GATHER_C) {
    b.add(MM_OP_GROUP_START);
    if (r == root) {
      for (int q = 0; q < G; ++q) {
        const Range rq = shard(m, G, q);
        if (rq.count == 0) continue;
        if (q == r) b.copy2d(0, MM_BUF_CFULL, rq.start * p * eo, p * eo, MM_BUF_C, 0, p * eo, p * eo, rq.count);
        else b.coll(MM_OP_RECV, 0, MM_COMM_WORLD, q, MM_BUF_CFULL, rq.start * p * eo, rq.count * p * eo);
      }
    } else if (mine.count > 0) {
      b.coll(MM_OP_SEND, 0, MM_COMM_WORLD, root, MM_BUF_C, 0, mine.count * p * eo);
    }
    b.add(MM_OP_GROUP_END);
  }
}

void summa(Builder& b, mm_plan_info* info, int64_t m, int64_t n, int64_t p, mm_dtype dt, unsigned flags, int pr,
           int pc, int layers, int r, int64_t panel) {
  const int64_t ei = esz_in(dt), eo = esz_out(dt);
  const int l = r / (pr * pc), r2 = r % (pr * pc);
  const int gi = r2 / pc, gj = r2 % pc;
  // sub-communicators: grid row (colour l·pr+gi, rank gj), grid column (colour l·pc+gj, rank gi),
  // depth (colour gi·pc+gj, rank l)
  info->color[MM_COMM_ROW] = l * pr + gi, info->key[MM_COMM_ROW] = gj;
  info->color[MM_COMM_COL] = l * pc + gj, info->key[MM_COMM_COL] = gi;
  if (layers > 1) info->color[MM_COMM_DEPTH] = gi * pc + gj, info->key[MM_COMM_DEPTH] = l;
  const Range am = shard(m, pr, gi), ak = shard(n, pc, gj);  // my A block: rows am, cols ak
  const Range bk = shard(n, pr, gi), bn = shard(p, pc, gj);  // my B block: rows bk, cols bn
  if (layers > 1 && (flags & MM_REPLICATE)) {
    // the blocks are valid on layer 0 only: replicate them along the depth first
    b.add(MM_OP_GROUP_START);
    if (am.count > 0 && ak.count > 0) b.coll(MM_OP_BCAST, 0, MM_COMM_DEPTH, 0, MM_BUF_A, 0, am.count * ak.count * ei);
    if (bk.count > 0 && bn.count > 0) b.coll(MM_OP_BCAST, 0, MM_COMM_DEPTH, 0, MM_BUF_B, 0, bk.count * bn.count * ei);
    b.add(MM_OP_GROUP_END);
  }
  const int64_t w = summa_panel(panel, dt);
  const int np = mm_summa_panels(n, pr, pc, w, 0, nullptr, nullptr, nullptr, nullptr);
  std::vector<int64_t> k0(np), kw(np);
  std::vector<int> ao(np), bo(np);
  mm_summa_panels(n, pr, pc, w, np, k0.data(), kw.data(), ao.data(), bo.data());
  // two buffer sets {A panel (am × w) in S0/S2, B panel (w × bn) in S1/S3}
  info->stage_bytes[0] = info->stage_bytes[2] = std::max<int64_t>(am.count, 1) * w * ei;
  info->stage_bytes[1] = info->stage_bytes[3] = w * std::max<int64_t>(bn.count, 1) * ei;
  b.record(EV_START, 0);
  b.wait(1, EV_START);
  int done = 0;  // panels this layer has accumulated
  for (int t = l; t < np; t += layers) {
    const int s = (t / layers) & 1;
    const int Ap = MM_BUF_S0 + 2 * s, Bp = MM_BUF_S1 + 2 * s;
    if (done >= 2) b.wait(1, EV_FREE0 + s);
    // owners stage their panel (A: a column slice, pitched; B: whole rows of the block)
    if (gj == ao[t] && am.count > 0)
      b.copy2d(1, Ap, 0, kw[t] * ei, MM_BUF_A, (k0[t] - ak.start) * ei, ak.count * ei, kw[t] * ei, am.count);
    if (gi == bo[t] && bn.count > 0)
      b.copy2d(1, Bp, 0, kw[t] * bn.count * ei, MM_BUF_B, (k0[t] - bk.start) * bn.count * ei, kw[t] * bn.count * ei,
               kw[t] * bn.count * ei, 1);
    b.add(MM_OP_GROUP_START, 1);
    if (am.count > 0) b.coll(MM_OP_BCAST, 1, MM_COMM_ROW, ao[t], Ap, 0, am.count * kw[t] * ei);
    if (bn.count > 0) b.coll(MM_OP_BCAST, 1, MM_COMM_COL, bo[t], Bp, 0, kw[t] * bn.count * ei);
    b.add(MM_OP_GROUP_END, 1);
    b.record(EV_READY0 + s, 1);
    b.wait(0, EV_READY0 + s);
    if (am.count > 0 && bn.count > 0)
      b.gemm(am.count, kw[t], bn.count, Ap, 0, kw[t], Bp, 0, bn.count, MM_BUF_C, 0, bn.count, done > 0 ? 1 : 0, 1);
    b.record(EV_FREE0 + s, 0);
    ++done;
  }
  // the caller's stream must not run ahead of the last communication
  b.record(EV_END, 1);
  b.wait(0, EV_END);
  if (layers > 1 && am.count > 0 && bn.count > 0) {
    // a layer that received no panel contributes zeros; then sum the layers onto layer 0
    if (done == 0) b.coll(MM_OP_MEMSET0, 0, 0, 0, MM_BUF_C, 0, am.count * bn.count * eo);
    b.coll(MM_OP_REDUCE_SUM, 0, MM_COMM_DEPTH, 0, MM_BUF_C, 0, am.count * bn.count);
  }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) void mm_shard_range(int64_t total, int G, int r, int64_t* start,
                                                           int64_t* count) {
  int64_t s = 0, c = 0;
  if (G >= 1 && r >= 0 && r < G && total > 0) {
    const int64_t q = (total + G - 1) / G;  // ⌈total/G⌉
    s = std::min<int64_t>((int64_t)r * q, total);
    c = std::min<int64_t>(q, total - s);
  }
  if (start) *start = s;
  if (count) *count = c;
}

__attribute__((visibility("default"))) int mm_summa_panels(int64_t n, int grid_rows, int grid_cols, int64_t panel,
                                                           int cap, int64_t* k0, int64_t* kw, int* a_col,
                                                           int* b_row) {
  if (n < 1 || grid_rows < 1 || grid_cols < 1 || panel < 1) return 0;
  // boundaries = union of A's column-block and B's row-block boundaries along k
  std::vector<int64_t> cuts = {0, n};
  for (int j = 0; j < grid_cols; ++j) cuts.push_back(shard(n, grid_cols, j).start);
  for (int i = 0; i < grid_rows; ++i) cuts.push_back(shard(n, grid_rows, i).start);
  std::sort(cuts.begin(), cuts.end());
  cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
  int np = 0;
  for (size_t c = 0; c + 1 < cuts.size(); ++c) {
    for (int64_t k = cuts[c]; k < cuts[c + 1]; k += panel) {
      const int64_t w = std::min<int64_t>(panel, cuts[c + 1] - k);
      if (np < cap) {
        if (k0) k0[np] = k;
        if (kw) kw[np] = w;
        int oa = 0, ob = 0;
        for (int j = 0; j < grid_cols; ++j) {
          Range rr = shard(n, grid_cols, j);
          if (k >= rr.start && k < rr.start + rr.count) oa = j;
        }
        for (int i = 0; i < grid_rows; ++i) {
          Range rr = shard(n, grid_rows, i);
          if (k >= rr.start && k < rr.start + rr.count) ob = i;
        }
        if (a_col) a_col[np] = oa;
        if (b_row) b_row[np] = ob;
      }
      ++np;
    }
  }
  return np;
}

__attribute__((visibility("default"))) mm_status mm_shard_plan(int64_t m, int64_t n, int64_t p, mm_dtype dtype,
                                                               mm_layout layout, int grid_rows, int grid_cols,
                                                               unsigned flags, int root, int G, int r,
                                                               int64_t panel, mm_plan_step* steps, int cap,
                                                               mm_plan_info* info) {
  if (!info) return MM_ERR_USAGE;
  memset(info, 0, sizeof *info);
  for (int c = 0; c < 4; ++c) info->color[c] = info->key[c] = -1;
  info->color[MM_COMM_WORLD] = 0;
  info->key[MM_COMM_WORLD] = r;
  if (dtype != MM_F64 && dtype != MM_BF16_F32 && dtype != MM_S8_S32 && dtype != MM_F64_EMU) return MM_ERR_USAGE;
  if (m < 1 || n < 1 || p < 1 || G < 1 || r < 0 || r >= G || cap < 0 || (cap > 0 && !steps)) return MM_ERR_USAGE;
  Builder b;
  if (layout == MM_ROW_BLOCK) {
    if (root < 0 || root >= G) return MM_ERR_USAGE;
    if (flags & ~(unsigned)(MM_BCAST_B | MM_GATHER_C | MM_GATHER_C_FUSED | MM_C_WINDOW)) return MM_ERR_USAGE;
    if ((flags & MM_GATHER_C) && (flags & MM_GATHER_C_FUSED)) return MM_ERR_USAGE;
    if ((flags & MM_C_WINDOW) && !(flags & MM_GATHER_C_FUSED)) return MM_ERR_USAGE;  // (executor detail only)
    row_block(b, info, m, n, p, dtype, flags, root, G, r, panel);
  } else if (layout == MM_SUMMA_2D || layout == MM_SUMMA_25D) {
    // panels accumulate with beta = 1 (the FP64 kernel and the FP64 emulation's reconstruction)
    if (dtype != MM_F64 && dtype != MM_F64_EMU) return MM_ERR_UNSUPPORTED;
    if (grid_rows < 1 || grid_cols < 1) return MM_ERR_USAGE;
    const int g2 = grid_rows * grid_cols;
    if (layout == MM_SUMMA_2D && (g2 != G || flags)) return MM_ERR_USAGE;
    if (layout == MM_SUMMA_25D && (G % g2 != 0 || (flags & ~(unsigned)MM_REPLICATE))) return MM_ERR_USAGE;
    summa(b, info, m, n, p, dtype, flags, grid_rows, grid_cols, G / g2, r, panel);
  } else {
    return MM_ERR_USAGE;
  }
  info->steps = (int32_t)b.v.size();
  info->events = EV_COUNT;
  for (int i = 0; i < cap && i < (int)b.v.size(); ++i) steps[i] = b.v[i];
  return MM_OK;
}

}  // extern "C"
