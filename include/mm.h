/*
 * mm.h — C-ABI of the B200-native dense product C = A·B.
 *
 * The operation (§III, displayed equation):
 *     C[i][j] = Σ_{k=1..n} A[i][k] · B[k][j],   A is m×n, B is n×p, C is m×p,
 * i.e. each element is the dot product of row i of A and column j of B
 * (PAPER.md:62-74), for all i ≤ m, j ≤ p.
 *
 * Layout: every matrix is dense ROW-MAJOR ("C ... stores data in row-major
 * order"): element (i,j) of an r×c matrix lives at i*c + j, so
 * the leading dimensions are n (A), p (B) and p (C).  No transposes, no α/β.
 *
 * Types (mm_dtype, input → output):
 *   MM_F64      double   × double   → double   (the paper's precision)
 *   MM_BF16_F32 bfloat16 × bfloat16 → float    (FP32 accumulate; BASELINE.json config 3)
 *   MM_F64_EMU  double   × double   → double   (the same binary64 product computed on the INT8
 *                                               tensor cores (Ozaki scheme, second kind): rows of A
 *                                               / columns of B scaled by powers of two to integers
 *                                               of β ≥ 53 bits, their residues modulo N = 14..16
 *                                               coprime moduli ≤ 256 multiplied as N exact
 *                                               INT8·INT8→INT32 products, the integer product
 *                                               rebuilt by Chinese remaindering (Garner) and
 *                                               rounded once to binary64; exact for integer
 *                                               inputs, ~1e-17..1e-16 normalised error on U[-1,1)
 *                                               inputs; finite inputs only (an Inf / NaN is
 *                                               reported by mm_sync_check, MM_ERR_RUNTIME, C
 *                                               undefined); n < 131072 (n·2^14 <
 *                                               2^31 per INT32 sum); device scratch ≈
 *                                               N·(m·n + n·p + m·p) bytes
 *                                               (mm_workspace_size); every layout of
 *                                               mm_gemm_sharded, its local products emulated)
 *   MM_S8_S32   int8     × int8     → int32    (INT32 accumulate, exact while
 *                                               n·128² < 2^31; BASELINE.json config 2)
 *
 * Ownership: the caller owns A, B, C, the optional workspace and the stream.
 * The context owns only device properties, a device error word and the
 * small internal buffers it allocates for padding / host staging.
 *
 * Asynchrony: device-pointer calls enqueue on `stream` and return; C is valid
 * once the stream reaches that point.  A and B must not change before then.
 * Launch-time errors are returned; in-kernel errors (a pipeline wait that
 * timed out) are latched in the context's device error word and reported by
 * mm_sync_check().
 *
 * Errors: every call returns an mm_status; on failure mm_last_error(ctx)
 * names the offending argument (shapes included).  Status codes 0/1/2 mirror
 * SPEC.md:498 (0 ok, 1 runtime failure, 2 usage error).
 *
 * Thread safety: one context per host thread at a time; distinct contexts are
 * independent.  No global state besides lazily resolved driver/NCCL symbols.
 */
#ifndef MM_B200_H
#define MM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { MM_F64 = 0, MM_BF16_F32 = 1, MM_S8_S32 = 2, MM_F64_EMU = 3 } mm_dtype;

typedef enum {
  MM_OK = 0,
  MM_ERR_RUNTIME = 1,     /* CUDA / NCCL failure, or a device-side pipeline timeout */
  MM_ERR_USAGE = 2,       /* bad argument: dims < 1, NULL pointer, bad enum, overlap of C with A/B */
  MM_ERR_UNSUPPORTED = 3, /* no sm_100a device, or sizes beyond TMA / int64 limits */
  MM_ERR_WORKSPACE = 4    /* an internal allocation failed */
} mm_status;

typedef struct mm_ctx mm_ctx;

/* Create a context bound to CUDA `device` (must be sm_100).  `workspace` is an
 * optional caller-owned device buffer (may be NULL / 0 bytes); it is used for
 * the padding path before the context allocates its own.  *out receives the
 * context.  Errors: MM_ERR_USAGE (out NULL), MM_ERR_UNSUPPORTED (not sm_100),
 * MM_ERR_RUNTIME (CUDA failure). */
mm_status mm_create(int device, void* workspace, size_t workspace_bytes, mm_ctx** out);

/* Free the context and its internal buffers (never the caller's). NULL is a no-op. */
void mm_destroy(mm_ctx* ctx);

/* C := A·B on the device.  A (m×n), B (n×p), C (m×p) are device pointers,
 * row-major, element types per `dtype`.  m, n, p ≥ 1.  Any base alignment and
 * any m, n, p are accepted: operands whose base or row pitch is not a
 * multiple of 16 bytes are first copied into a zero-padded buffer (coalesced
 * 16-byte path), otherwise the kernels read them in place through TMA.
 * `stream` is a cudaStream_t (NULL = legacy default stream). */
mm_status mm_gemm(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype,
                  const void* A, const void* B, void* C, void* stream);

/* Same product with HOST operands: A, B, C are host pointers (pinned memory
 * gives full PCIe bandwidth; pageable works).  Copies A and B to the device,
 * computes, copies C back, in row blocks so that the host↔device copies of
 * one block overlap the product of the previous one (the paper's row
 * partition, applied to the PCIe link).  Synchronous: returns
 * after C is written on the host. */
mm_status mm_gemm_host(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype,
                       const void* A, const void* B, void* C, void* stream);

/* Synchronize `stream` and report any device-side error latched since the
 * last call (MM_ERR_RUNTIME with a message), then clear it. */
mm_status mm_sync_check(mm_ctx* ctx, void* stream);

const char* mm_status_string(mm_status s);
const char* mm_last_error(const mm_ctx* ctx);

/* ------------------------------------------------------------------ sharded
 * Multi-GPU products, one process per GPU (§III-B2
 * "Processes"; SUMMA named at PAPER.md:135).  Collective: every rank calls
 * with identical (m, n, p, dtype, layout, grid, flags, root).
 *
 * MM_ROW_BLOCK: C is split by row blocks of A (the paper's row partition of
 *   the outer loop, across processes).  Rank r owns rows
 *   [row0, row0+rows) from mm_shard_range(m, G, r, ...) of A and C; B is
 *   replicated.  A_local is (rows × n), C_local is (rows × p).
 *   flags: MM_BCAST_B — B is valid only on `root` and is broadcast first
 *          (B_local must be an n×p buffer on every rank);
 *          MM_GATHER_C — after the product, the full m×p C is assembled on
 *          `root` into C_full (ignored elsewhere) by NCCL send/recv;
 *          MM_GATHER_C_FUSED — the same result without a separate gather:
 *          every rank's product kernel stores its C tiles straight into the
 *          root's C_full over NVLink (peer memory, CUDA IPC mapping of the
 *          root's allocation exchanged through the communicator), so the
 *          transfer overlaps the math tile by tile; C_local is not written
 *          (may be NULL).  Ends with a communicator-wide barrier so C_full is
 *          complete on `root` when the call's stream work finishes.
 *          MM_C_WINDOW (with MM_GATHER_C_FUSED): the peer mapping is NCCL's
 *          instead — every rank passes, as C_full, its own buffer from
 *          mm_window_alloc at the same offset (symmetric memory), and the root's
 *          address comes from the window (ncclGetPeerPointer, NCCL's LSA/NVLink
 *          mapping) with no handle exchange.
 * MM_SUMMA_2D: ranks form a grid_rows × grid_cols grid (G = grid_rows*grid_cols),
 *   rank r ↔ (r / grid_cols, r % grid_cols).  Rank (i,j) owns block (i,j)
 *   of A (row block i of m, column block j of n), of B (row block i of n,
 *   column block j of p) and of C (row block i of m, column block j of p),
 *   blocks by mm_shard_range on each axis.  k-panels of A are broadcast along
 *   grid rows and of B along grid columns; local products accumulate.
 * MM_SUMMA_25D: 2.5D: G = grid_rows·grid_cols·c ranks form c
 *   layers of that grid, rank r ↔ (l, i, j) with r = l·grid_rows·grid_cols +
 *   i·grid_cols + j.  Every layer holds the same blocks (flag MM_REPLICATE:
 *   only layer 0's are valid and are broadcast along the depth first); layer l
 *   runs the SUMMA k-panels t ≡ l (mod c), and the layers' C blocks are summed
 *   onto layer 0 (NCCL reduce); other layers' C_local hold partial sums.
 *   SUMMA layouts are implemented for MM_F64 and MM_F64_EMU (they accumulate with β = 1).
 *
 * Mismatched arguments across ranks are a usage error: the diagnostic build (and the release
 * library with MM_CHECK_COLLECTIVE=1, at the cost of one all-reduce and a stream synchronisation)
 * checks them with an all-reduce of their hash and returns MM_ERR_USAGE on every rank.
 *
 * nccl_comm is an ncclComm_t spanning exactly the G ranks (e.g. torch's
 * ProcessGroupNCCL._comm_ptr()).  The library resolves NCCL symbols at run
 * time from the libnccl.so.2 already loaded in the process.
 */
typedef enum { MM_ROW_BLOCK = 0, MM_SUMMA_2D = 1, MM_SUMMA_25D = 2 } mm_layout;
enum { MM_BCAST_B = 1u, MM_GATHER_C = 2u, MM_GATHER_C_FUSED = 4u, MM_REPLICATE = 8u, MM_C_WINDOW = 16u };

mm_status mm_gemm_sharded(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype,
                          mm_layout layout, int grid_rows, int grid_cols,
                          const void* A_local, void* B_local, void* C_local, void* C_full,
                          unsigned flags, int root, void* nccl_comm, void* stream);

/* CUDA-IPC export / open of device memory (the peer mapping behind MM_GATHER_C_FUSED, exposed
 * so a handle can travel by any channel).  mm_ipc_export fills *out with a handle to the
 * allocation holding dev_ptr plus dev_ptr's offset in it (MM_ERR_USAGE if dev_ptr is not device
 * memory).  mm_ipc_open, in ANOTHER process, maps it (cached per context; unmapped by mm_destroy)
 * and returns the address of dev_ptr in this process; products may then store into it (TMA stores
 * through the mapping — over NVLink when it is a peer GPU's memory).  MM_ERR_RUNTIME if the
 * handle cannot be opened (e.g. an allocation of this same process). */
typedef struct { unsigned char bytes[72]; } mm_ipc_handle;
mm_status mm_ipc_export(mm_ctx* ctx, const void* dev_ptr, mm_ipc_handle* out);
mm_status mm_ipc_open(mm_ctx* ctx, const mm_ipc_handle* handle, void** dev_ptr);

/* NCCL symmetric memory for MM_GATHER_C_FUSED | MM_C_WINDOW (PAPER.md:135/146 —
 * communication between the processes of a node).  Collective over nccl_comm (every rank, same
 * `bytes`): allocates `bytes` with ncclMemAlloc (cuMem VMM memory NCCL can map into its peers)
 * and registers it as a window (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC); *ptr receives
 * this rank's buffer.  The context records (buffer, window, communicator); the caller frees it
 * with mm_window_free (collective, same order on every rank) before mm_destroy.
 * MM_ERR_UNSUPPORTED if the loaded NCCL has no window API; MM_ERR_RUNTIME on NCCL failure. */
mm_status mm_window_alloc(mm_ctx* ctx, void* nccl_comm, size_t bytes, void** ptr);
mm_status mm_window_free(mm_ctx* ctx, void* ptr);

/* Contiguous block partition of `total` items over G parts:
 * part r gets [start, start+count); the first parts get ⌈total/G⌉, the
 * last non-empty part is short, surplus parts (G > total) are empty. */
void mm_shard_range(int64_t total, int G, int r, int64_t* start, int64_t* count);

/* SUMMA k-panel schedule for an n-long contraction over a grid_rows × grid_cols
 * grid with target panel width `panel`: panel t covers k in [k0[t], k0[t]+kw[t]),
 * never straddles a column block of A (owner a_col[t]) nor a row block of B
 * (owner b_row[t]).  Returns the number of panels, writing at most `cap`.
 * Pure host logic (tested without a GPU). */
int mm_summa_panels(int64_t n, int grid_rows, int grid_cols, int64_t panel, int cap,
                    int64_t* k0, int64_t* kw, int* a_col, int* b_row);

/* ------------------------------------------------------------------ sharded schedule as data
 * mm_gemm_sharded runs a per-rank PLAN: a list of steps (local products, pitched copies, NCCL
 * collectives, stream events) that mm_shard_plan computes from the collective's arguments alone
 * (pure host logic, no device, no communicator).  The same plan can be executed by another runtime
 * (the test suite runs it over torch.distributed/gloo on CPU with the oracle as the local product,
 * at world sizes 2-8), so the partition, offsets, pitches, roots and ordering that the GPU path
 * uses are checked on any machine.  The rules are the ones documented for mm_gemm_sharded above
 * (PAPER.md:119 row partition; PAPER.md:135 SUMMA / 2.5D).
 *
 * Buffers (mm_plan_buf): the caller's A_local, B_local, C_local, C_full (root only), the root's
 * C_full as mapped into this rank (CPEER, fused gather), and staging buffers S0..S3 of
 * info.stage_bytes[i] bytes owned by the executor.  Offsets are in bytes.
 * Streams: 0 = the caller's (compute) stream, 1 = the executor's communication stream.
 * Communicators (mm_plan_comm): WORLD, and the ROW / COL / DEPTH sub-communicators obtained by
 * splitting WORLD with info.color[c] / info.key[c] (ncclCommSplit semantics: ranks with equal
 * colour form one communicator, ordered by key); `peer` is a rank inside the step's communicator.
 *
 *   MM_OP_GEMM        C[dst]+dst_off (ld dst_ld elements) (+)= A[src]+src_off (ld src_ld) ·
 *                     B[src2]+src2_off (ld src2_ld); m×n · n×p; beta 0 overwrite, 1 accumulate;
 *                     overlap = 1: communication runs concurrently (the product leaves SMs free).
 *   MM_OP_COPY2D      m rows of n bytes: dst+dst_off (pitch dst_ld bytes) <- src+src_off (pitch src_ld).
 *   MM_OP_BCAST       n bytes at dst+dst_off, from `peer` to all ranks of `comm` (in place).
 *   MM_OP_SEND/RECV   n bytes at src+src_off to / dst+dst_off from `peer` of `comm`.
 *   MM_OP_GROUP_START / MM_OP_GROUP_END   bracket sends/receives issued together.
 *   MM_OP_REDUCE_SUM  n elements (FP64) at dst+dst_off summed onto `peer` of `comm` (in place).
 *   MM_OP_MEMSET0     n bytes at dst+dst_off set to zero.
 *   MM_OP_BARRIER     all ranks of `comm` (device-side: an all-reduce of one word).
 *   MM_OP_MAP_PEER    collective on WORLD: every rank obtains CPEER = `peer`'s C_full.
 *   MM_OP_RECORD      record event `event` on `stream`;  MM_OP_WAIT: `stream` waits for `event`.
 */
typedef enum {
  MM_OP_GEMM = 1, MM_OP_COPY2D = 2, MM_OP_BCAST = 3, MM_OP_SEND = 4, MM_OP_RECV = 5, MM_OP_GROUP_START = 6,
  MM_OP_GROUP_END = 7, MM_OP_REDUCE_SUM = 8, MM_OP_MEMSET0 = 9, MM_OP_BARRIER = 10, MM_OP_MAP_PEER = 11,
  MM_OP_RECORD = 12, MM_OP_WAIT = 13
} mm_plan_op;
typedef enum {
  MM_BUF_NONE = 0, MM_BUF_A = 1, MM_BUF_B = 2, MM_BUF_C = 3, MM_BUF_CFULL = 4, MM_BUF_CPEER = 5,
  MM_BUF_S0 = 6, MM_BUF_S1 = 7, MM_BUF_S2 = 8, MM_BUF_S3 = 9
} mm_plan_buf;
typedef enum { MM_COMM_WORLD = 0, MM_COMM_ROW = 1, MM_COMM_COL = 2, MM_COMM_DEPTH = 3 } mm_plan_comm;

typedef struct {
  int32_t op, stream, comm, peer;       /* mm_plan_op; 0/1; mm_plan_comm; rank inside comm */
  int32_t dst, src, src2, beta;         /* mm_plan_buf ids (GEMM: C = dst, A = src, B = src2) */
  int64_t dst_off, src_off, src2_off;   /* byte offsets into those buffers */
  int64_t dst_ld, src_ld, src2_ld;      /* GEMM: leading dimensions in elements; COPY2D: pitches in bytes */
  int64_t m, n, p;                      /* GEMM: dims; COPY2D: rows = m, row bytes = n; others: n = count */
  int32_t event, overlap;               /* RECORD/WAIT: event id; GEMM: 1 = overlapped with communication */
} mm_plan_step;

typedef struct {
  int32_t steps;           /* steps in the plan (may exceed the cap passed in) */
  int32_t events;          /* event ids used: [0, events) */
  int32_t color[4];        /* per mm_plan_comm: split colour of this rank (-1: communicator unused) */
  int32_t key[4];          /* per mm_plan_comm: rank of this rank inside that communicator */
  int64_t stage_bytes[4];  /* staging buffers S0..S3 the executor provides */
} mm_plan_info;

/* The plan rank r of G executes for mm_gemm_sharded(m, n, p, dtype, layout, grid_rows, grid_cols,
 * flags, root).  `panel`: column-panel width of the B broadcast (row-block) or k-panel width (SUMMA);
 * 0 = the library default (p/8 and 2048; MM_F64_EMU: p/2 and 8192, each emulated panel product
 * having fixed costs).  Writes at most `cap` steps to `steps` (may be NULL with cap 0) and the
 * plan's metadata to *info (required).  Returns MM_ERR_USAGE for invalid arguments (the same checks
 * as mm_gemm_sharded: dims >= 1, 0 <= r < G, root in range, grid consistent with G, flags valid for
 * the layout; SUMMA layouts for MM_F64 and MM_F64_EMU only).  Pure host logic. */
mm_status mm_shard_plan(int64_t m, int64_t n, int64_t p, mm_dtype dtype, mm_layout layout, int grid_rows,
                        int grid_cols, unsigned flags, int root, int G, int r, int64_t panel,
                        mm_plan_step* steps, int cap, mm_plan_info* info);

/* Upper bound, in bytes, of the device memory a context allocates internally for one call with
 * these arguments: the zero-padded operand copies of the edge path (counted as if
 * neither A nor B had a 16-byte pitch), the split-tail partial tiles and tickets, and, for G > 1,
 * the panel staging buffers of the sharded layouts (the largest over all ranks, and for the SUMMA
 * layouts over every grid that G factors into).  Buffers are allocated lazily, grow only, and are
 * freed by mm_destroy; a mm_create `workspace` of at least the padding part is used instead of an
 * internal padding buffer.  Pure host logic: the bound assumes at most 160 SMs.  0 for invalid
 * arguments. */
size_t mm_workspace_size(int64_t m, int64_t n, int64_t p, mm_dtype dtype, mm_layout layout, int G);

/* MM_F64_EMU plan for inner dimension n (pure host logic): writes the moduli used (the first
 * *count of the fixed list, largest first, pairwise coprime, each ≤ 256) to `moduli` (room for 16;
 * may be NULL) and the scaling width β to *beta: the fewest moduli with
 * n·2^(2β) ≤ Π m_l / 2 − 1 and β ≥ 53, β as large as that product allows (≤ 60).
 * MM_ERR_USAGE for n < 1, null count/beta; MM_ERR_UNSUPPORTED for n ≥ 131072 (INT32 sums). */
mm_status mm_f64_emu_plan(int64_t n, int* moduli, int* count, int* beta);

/* Clock meter (measurement): enable = 1 makes every product kernel of this context record, per
 * CTA, its SM cycle count (clock64) and elapsed nanoseconds (globaltimer) between entry and exit
 * (four stores per CTA; results unchanged).  enable = 0 synchronises the device, stops recording and
 * returns in *mhz the effective SM clock of the most recent launch: Σ cycles / Σ ns over its CTAs
 * (0 if nothing was recorded).  MM_ERR_WORKSPACE if the 128-KiB record buffer cannot be allocated. */
mm_status mm_clock_meter(mm_ctx* ctx, int enable, double* mhz);

/* Number of kernels this context has launched so far (product, padding and
 * fix-up kernels; NCCL's own kernels are not counted). */
uint64_t mm_launches(const mm_ctx* ctx);

/* Library/version info: "mm_b200 <version> sm_100a". */
const char* mm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MM_B200_H */
