/*
 * uhmv.h -- C ABI of the B200-native uniform-H matrix-vector product (sm_100a).
 *
 * The reference (uhm-kit, pure Python) has no FFI: its boundary is the Python callable
 *   matvec_uh(u, v, workers=1, adjoint=False, stats=None)
 *     /root/reference/pkg/src/uhm_kit/uniform.py:476-556
 * plus UniformHMatrix.matvec (uniform.py:116-117).  This library replaces the body of that
 * callable; the Python layer (paper_2405_15573_b200/matvec.py) keeps its signature, argument
 * meaning and error behaviour and binds these entry points with ctypes.
 *
 * Ownership: every device buffer named in uhmv_desc is allocated and kept alive by the caller
 * (PyTorch tensors in the Python layer).  The plan never frees them; it only owns launch
 * configuration.  All entry points return 0 on success and a negative code on failure; the text
 * of the last failure of the calling thread is available from uhmv_last_error().
 *
 * Concurrency: plans that share device state (the same ticket buffer -- a plan and its multi-RHS
 * plan) form a group whose launches never overlap.  Every enqueueing entry point holds the
 * group's host mutex while it enqueues and records a group event after the launch; a call on a
 * different stream than the group's previous launch first waits for that event.  So any mix of
 * host threads and streams calling one plan gives the results of some serial order.  Inside a
 * stream capture the event ordering is skipped (replay the captured graph on one stream at a
 * time).
 */
#ifndef UHMV_H
#define UHMV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UHMV_ABI_VERSION 13
#define UHMV_MAX_PHASES 8

/* Execution modes of uhmv_execute. */
#define UHMV_MODE_PHASED 0 /* one launch per phase (P1+NEAR, RED, U, Z, FAR)          */
#define UHMV_MODE_FUSED 1  /* one persistent launch, register-streaming op engine         */
#define UHMV_MODE_BULK 2   /* one persistent launch, warp-specialised bulk-copy (TMA) op
                              engine: producer lane streams arena pieces with cp.async.bulk
                              into an mbarrier stage ring ahead of dependency waits      */

/* Error codes. */
#define UHMV_OK 0
#define UHMV_EINVAL (-1)
#define UHMV_ECUDA (-2)
#define UHMV_ENOMEM (-3)

/* One op program (forward or adjoint) -- device pointers to the tables built by the packer
 * (paper_2405_15573_b200/packer.py).  ops: n_ops x 16 int32; segs: n_segs x 8 int64;
 * runs: n_runs x 5 int64; waits: n_waits x 2 int32; sigs: int32; fused_order: n_ops int32. */
typedef struct uhmv_program {
    int32_t n_ops;
    const int32_t* ops;
    const int64_t* segs;
    const int64_t* runs;
    const int32_t* waits;
    const int32_t* sigs;
    const int32_t* fused_order;
    const int64_t* pieces; /* n_pieces x 8 int64 (bulk engine) */
    int32_t n_phases;
    int32_t phase_lo[UHMV_MAX_PHASES];
    int32_t phase_hi[UHMV_MAX_PHASES];
    int32_t in_max;     /* largest gathered input vector of any op (complex elements)  */
    int32_t out_max;    /* largest output vector of any op (complex elements)          */
    int32_t n_counters; /* dependency counters used by the fused mode                  */
    int32_t xin_max;    /* largest work-buffer input of any op (bulk engine)           */
    int32_t zero_output; /* zero w before the launch (0 for the post-exchange program of a
                            multi-GPU rank, which adds into w)                          */
    int32_t stage_elems; /* complex128 elements per shared-memory stage (bulk engine)  */
    const int64_t* mr_segs;   /* multi-RHS segments, n x 8 int64 (one input source each);
                                 mode field: low byte mode, bit 8 first writer of its outputs */
    const int32_t* mr_ranges; /* n_ops x 3 int32: mr_segs range of every op + flags
                                 (bit 0: zero the op's work outputs first)                   */
    int32_t n_tmaps;          /* distinct leading dimensions of the arena matrices the
                                 multi-RHS segments read (mr_segs mode field bits 16..)      */
    const int64_t* tmap_lds;  /* HOST array of n_tmaps leading dimensions (complex elements) */
    void* tmaps;              /* DEVICE buffer, 2 * n_tmaps * 128 bytes, 64-B aligned, that
                                 uhmv_plan_create fills with TMA tensor maps over the arena
                                 (per ld: a 16 x 16 and a 16 x 80 complex box)              */
    int32_t flags;            /* UHMV_PROG_SYM: symmetric single-triangle program
                                 (paper_2405_15573_b200/packer_sym.py; T-mode and alias
                                 pieces): bulk engine only                                  */
} uhmv_program;

#define UHMV_PROG_SYM 1
#define UHMV_PROG_WORDER 4 /* ordered output (packer w_order): the NEAR ops of an output leaf STORE
                              their rows of w, its FAR ops wait for them and add (plain read-modify-
                              write): uhmv_execute runs no memset and no atomics.  The multi-RHS
                              engines always add atomically into a W they zero first.             */
#define UHMV_PROG_XWIN 2 /* windowed-input ops (H-format FAR, packer_h OP_XWIN): the bulk engine runs
                            them with uhmv_bulk_xwin_kernel; no peer / host-I/O programs          */

/* A packed uniform H-matrix.  Replaces the UniformHMatrix dicts (uniform.py:90-117). */
typedef struct uhmv_desc {
    int32_t abi_version;      /* = UHMV_ABI_VERSION */
    int32_t device;           /* CUDA device ordinal */
    int64_t n_rows, n_cols;   /* operator shape (bct.shape, clustering.py:196-198) */
    const void* arena;        /* complex128 bases, coupling and dense slabs (read-only) */
    int64_t arena_len;        /* arena elements; the allocation extends max(tmap_lds)
                                 elements further (TMA rows of the last ld may overhang) */
    void* work;               /* complex128 scratch: partials, y, staging u, z */
    int64_t work_len;
    uint32_t* counters;       /* >= max(n_counters) zero-initialised uint32 */
    unsigned long long* ticket; /* one zero-initialised uint64 (fused dispatch) */
    uint32_t* exit_count;     /* one zero-initialised uint32 (fused self-reset) */
    void* x_scratch;          /* complex128 device buffers used by uhmv_matvec_host, */
    void* w_scratch;          /* each >= max(n_rows, n_cols) elements (may be NULL)  */
    uhmv_program fwd;
    uhmv_program adj;
} uhmv_desc;

typedef struct uhmv_plan uhmv_plan;

/* ABI version compiled into the library. */
int uhmv_abi_version(void);

/* Validate a descriptor and prepare launch configuration (occupancy, shared memory).
 * Replaces: nothing in the reference -- the reference walks dicts on every call
 * (uniform.py:505-548); packing happens once per operator. */
int uhmv_plan_create(const uhmv_desc* desc, uhmv_plan** out);

/* w = A x (adjoint=0) or w = A^H x (adjoint=1); x, w device complex128 in tree order.
 * Replaces: matvec_uh body, uniform.py:496-556 (phase 1 :509-520, phase 2 :524-556).
 * stream: a cudaStream_t (NULL = legacy default stream).  Asynchronous. */
int uhmv_execute(uhmv_plan* plan, const void* x, void* w, int adjoint, int mode, void* stream);

/* Phased execution of phases [phase_lo, phase_hi) only (multi-GPU: the Python layer
 * inserts the NCCL all-gather of y/u between the halves).  Asynchronous. */
int uhmv_execute_phases(uhmv_plan* plan, const void* x, void* w, int adjoint, int phase_lo,
                        int phase_hi, void* stream);

/* End-to-end call with HOST buffers: H2D copy of x, execute, D2H copy of w, stream sync.
 * x_host / w_host: complex128 (interleaved re,im doubles), length n_in / n_out.
 * With pinned (page-locked) buffers the whole call is captured once per direction and buffer
 * pair into a CUDA graph and replayed (UHMV_HOST_GRAPH=0 disables), and -- after
 * uhmv_plan_set_io -- runs as one host-I/O launch instead of copy / launch / copy.
 * Replaces: the whole matvec_uh call as a caller sees it (uniform.py:476-556). */
int uhmv_matvec_host(uhmv_plan* plan, const void* x_host, void* w_host, int adjoint, int mode,
                     void* stream);

/* 1 if `host` points into page-locked (pinned, device-mapped) host memory, else 0. */
int uhmv_host_pinned(const void* host);

/* Which path pinned uhmv_matvec_host calls of one direction take once host-I/O programs are
 * attached: 1 the host-I/O launch (default), 0 H2D copy / launch / D2H copy.  A captured graph is
 * kept per path, so switching (e.g. while measuring both) replays instead of recapturing. */
int uhmv_plan_set_host_path(uhmv_plan* plan, int adjoint, int path);

/* Path the last uhmv_matvec_host of a direction took: 1 host-I/O launch, 0 copy path with pinned
 * buffers, -1 pageable buffers (always the copy path), or a negative error code. */
int uhmv_plan_last_host_path(const uhmv_plan* plan, int adjoint);

/* Attach the host-I/O variant of the plan's programs (packer io_programs(); counters: a
 * zeroed uint32 buffer of max(n_counters) of the two).  Afterwards uhmv_matvec_host with
 * PINNED host buffers runs ONE bulk launch whose P1 ops read x over PCIe (publishing it to
 * the device copy the NEAR ops read) and whose NEAR / FAR ops copy every finished output leaf
 * to w_host as soon as its last contribution lands: the transfers overlap the kernel instead
 * of bracketing it.  Pageable buffers keep the copy / launch / copy path.  A direction whose
 * program has n_ops = 0 keeps the copy path; fwd = adj = NULL detaches. */
int uhmv_plan_set_io(uhmv_plan* plan, const uhmv_program* fwd, const uhmv_program* adj, uint32_t* counters);

/* Multi-RHS product on FP64 tensor cores (DMMA): W = A X or A^H X, X (n_in x nrhs), W
 * (n_out x nrhs) and work_mr (work_len x nrhs) device complex128, row-major, nrhs a
 * multiple of 16.  Replaces the reference's column loop over matvec_uh (uniform.py:493-494
 * rejects 2-D input).  Asynchronous. */
int uhmv_execute_mrhs(uhmv_plan* plan, const void* x, void* w, void* work_mr, int nrhs,
                      int adjoint, void* stream);

/* Multi-RHS with HOST buffers, pipelined: X_host (n_in x nrhs) and W_host (n_out x nrhs)
 * row-major complex128 (pinned for overlap); the nrhs columns go in chunks of `chunk` (a
 * multiple of 16 dividing nrhs): the H2D copy of chunk c+1, the DMMA product of chunk c and
 * the D2H copy of chunk c-1 run concurrently on three streams.  X_dev / W_dev: device buffers
 * of 2 x n x chunk complex128 (double buffers); work_mr: work_len x chunk.  Synchronous.
 * Replaces: the reference's column loop over matvec_uh for a block of right-hand sides. */
int uhmv_matmat_host(uhmv_plan* plan, const void* X_host, void* W_host, int nrhs, void* X_dev, void* W_dev,
                     void* work_mr, int chunk, int adjoint, void* stream);

/* One rank of a peer-exchange partition (packer pack(peer=True)), as mapped in the calling
 * process: its own buffers, or a peer's NVLink-mapped ones (CUDA IPC / symmetric memory). */
typedef struct uhmv_peer_rank {
    void* work;          /* complex128 work buffer of 2 x work_len elements: epoch e uses half e & 1 */
    int64_t work_len;    /* that rank's program work length (uhmv_desc.work_len of its plan)     */
    uint32_t* counters;  /* >= n_counters uint32, zero before epoch 1 (monotonic afterwards)       */
    uint32_t* done;      /* world uint32, zero before epoch 1: done[q] = last epoch rank q finished */
} uhmv_peer_rank;

/* Multi-GPU matvec with the y/u exchange fused into the kernel: ONE launch per rank, whose
 * producer ops store this rank's y_t / u_t into every rank's work buffer over NVLink and
 * signal the peers' dependency counters (system-scope release); Z ops wait on them.  Replaces
 * the launch A / NCCL all-gather / launch B sequence of the partitioned path.
 * plans[0..nplans): the plans of ranks rank0 .. rank0+nplans-1 (nplans = 1 on a real multi-GPU
 * rank; nplans = world emulates the whole partition in one launch on one GPU, each rank on
 * its share of the SMs).  ranks[0..world): every rank's buffers.  w[i]: rank rank0+i's output
 * (zeroed here; ranks write disjoint rows, so the emulation may pass one vector for all).
 * epoch: 1, 2, ... consecutive per partition.  Asynchronous. */
int uhmv_execute_peer(uhmv_plan* const* plans, int nplans, int rank0, int world,
                      const uhmv_peer_rank* ranks, const void* x, void* const* w, int adjoint,
                      uint32_t epoch, void* stream);

/* Diagnostics of uhmv_execute_peer: a peer wait polls 2^spin_log2 times (default 28, ~10 s)
 * before trapping; host_mapped (pinned, device-visible, 512 uint32, zeroed, or NULL) receives
 * [0] the number of timed-out waits and, from [8], up to 63 records of 8 uint32: {rank,
 * counter (or 0x80000000 | peer for a done flag), value, need, epoch, block, 1, 0}. */
int uhmv_peer_set_diag(void* host_mapped, int spin_log2);

/* Launch geometry chosen for a mode (grid CTAs, dynamic shared memory bytes, threads per CTA,
 * shared-memory stages of the bulk engine). */
int uhmv_plan_info(const uhmv_plan* plan, int adjoint, int mode, int* grid, int* smem_bytes,
                   int* threads_per_cta, int* stages);

/* Diagnostics: per-CTA cycle counters of the bulk engine ([grid][8] uint64 device buffer, or
 * NULL to disable): consumer waiting for data / dependencies / computing / op overhead,
 * producer waiting for a free stage / an op slot, ops, pieces. */
int uhmv_plan_set_profile(uhmv_plan* plan, void* counters);

/* Diagnostics: op timeline of the profiled bulk engine (with uhmv_plan_set_profile on):
 * trace is a [n_ops][4] uint64 device buffer receiving {start, dependencies met, end, CTA} per
 * op, times from %globaltimer in ns (NULL disables). */
int uhmv_plan_set_trace(uhmv_plan* plan, void* trace);

/* Diagnostics: measured FP64 tensor-core (DMMA m16n8k16) throughput of the device, TFLOP/s
 * (the roofline denominator of the multi-RHS product; MEASURED_PEAKS.json has no FP64 entry). */
int uhmv_dmma_peak(int device, double* tflops);

int uhmv_plan_destroy(uhmv_plan* plan);

/* Thread-local text of the last failure ("" if none). */
const char* uhmv_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* UHMV_H */
