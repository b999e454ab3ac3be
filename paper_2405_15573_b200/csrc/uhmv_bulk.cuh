// uhmv_bulk.cuh -- warp-specialised bulk-copy engine for the uniform-H op programs (sm_100a).
//
// Same op semantics as the register kernel in uhmv.cu, different data path.  Every arena slab an
// op streams is cut on the host into "pieces" (row ranges, packer._pieces) packed into 16-KiB
// shared-memory stages.  Per CTA:
//
//   producer warp  claims ops from the fused ticket order (one ticket ahead), prefetches each
//                  op's header, run table and compressed piece descriptors into an op slot in
//                  shared memory (one coalesced round trip), publishes the slot, then streams the
//                  op's pieces with cp.async.bulk (TMA engine, SASS UBLKCP) into an mbarrier-
//                  guarded stage ring.  It never waits for an op's dependencies -- arena data
//                  depends on nothing -- so HBM streaming runs ahead across ops.
//   4 consumer     wait for the op's dependency counters (ld.acquire.gpu), gather the op's input
//   warps          vector into shared memory (one batched round trip), compute the GEMV pieces
//                  out of the stage ring accumulating each segment group in registers, reduce
//                  once per group, scatter the outputs (st.cg / fp64 red.add) and signal
//                  (red.release.gpu).
//
//   N group: out[o] += sum_j T[r,j] in[j]   row o owned by row-group o % 16 (8 lanes per row,
//            128 contiguous smem bytes per row-group load), register slot o / 16.
//   H group: out[j] += sum_r conj(T[r,j]) in[r]   column j owned by a P-lane group (rows split
//            over the P lanes), register slot j / nJ.
//   S group: out[j] += sum_r W[r,j] over the partial vectors, read directly (ld.cg) from work.
// Every output entry has exactly one owner thread and a fixed summation order: results are
// bit-reproducible run to run.

#pragma once

namespace bulk {

// consumer warps per CTA and the register cap (build-time experiments: -DUHMV_CWARPS=8
// -DUHMV_BULK_REGS=112 with UHMV_BULK_CTAS=2 runs 16 consumer warps per SM instead of 12)
#ifndef UHMV_CWARPS
#define UHMV_CWARPS 4
#endif
#ifndef UHMV_BULK_REGS
#define UHMV_BULK_REGS 128
#endif
#ifndef UHMV_NACC1
#define UHMV_NACC1 1
#endif
#ifdef UHMV_DIAGNOSTICS
constexpr bool kDiag = true;
#else
constexpr bool kDiag = false;  // release builds: the skip-waits / skip-compute switches are compiled out
#endif
constexpr int kConsumerWarps = UHMV_CWARPS;
constexpr int kConsumers = kConsumerWarps * 32;  // 128
constexpr int kThreads = kConsumers + 32;        // + one producer warp

constexpr int kOpSlots = 2;
constexpr int kMaxRanks = 8;      // peer-exchange programs: ranks of one NVLink domain
constexpr int kOpPeer = 16;       // op field 12 flag (packer.OP_PEER)
constexpr int kRunPeer = 4;       // out-run flag (packer.RUN_PEER)
// host-I/O programs (packer OP_XHOST / OP_XWAIT / OP_DRAIN, uhmv_matvec_host with pinned buffers)
constexpr int kOpXHost = 32;  // P1: gather x from the host buffer, publish it to device x
constexpr int kOpXWait = 64;  // NEAR: the producer waits for the op's x windows in device x
constexpr int kOpDrain = 128; // NEAR/FAR: the last op of an output leaf copies w[leaf] to the host
// symmetric single-triangle programs (packer_sym OP_DUAL): the op's N pieces and their alias
// T / H pieces write disjoint output ranges (own part vs mirror slots), so they need no barrier
// between them, N rows go straight to outv, and a T group's register accumulators live across
// the interleaved N pieces until the next T group (one flush per mirrored block, not per stage)
constexpr int kOpDual = 512;
// windowed-input ops (packer_h FAR, OP_XWIN): the op's N pieces read a gathered input far
// longer than shared memory allows at 3 CTAs/SM; it is gathered window by window (hdr[15]
// elements, hdr[0] in total) in piece order, one consumer barrier pair per window
constexpr int kOpXWin = 1024;
constexpr int kLanesPerRow = 8;
constexpr int kRowGroups = kConsumers / kLanesPerRow;  // 16
constexpr bool kPow2 = (kConsumers & (kConsumers - 1)) == 0;
// owner index v mod m (v may be negative): a mask for the power-of-2 consumer counts
template <int M>
__device__ __forceinline__ int wrapc(int v) {
    if constexpr ((M & (M - 1)) == 0) {
        return v & (M - 1);
    } else {
        const int r = v % M;
        return r < 0 ? r + M : r;
    }
}
__device__ __forceinline__ int wrap_nj(int v, int nJ) {  // nJ = kConsumers / P, P in {1, 2, 4}
    if constexpr (kPow2) {
        return v & (nJ - 1);
    } else {
        const int r = v % nJ;
        return r < 0 ? r + nJ : r;
    }
}
constexpr int kPieceFields = 8;
constexpr int kSlots = 4;         // register accumulator slots per thread
constexpr int kSlotRuns = 48;     // run descriptors cached per op slot
constexpr int kSlotPieces = 128;  // piece descriptors cached per op slot
constexpr int kGatherBatch = 8;   // loads in flight per thread in the gather
constexpr int64_t kPiBegin = 1ll << 24, kPiEnd = 1ll << 25, kPiDirect = 1ll << 26,
                  kPiXStage = 1ll << 28, kPiAlias = 1ll << 29;
constexpr int kModeT = 4;  // out[j] += sum_r M[r,j] in[r] (no conjugation; symmetric variant)

// compressed consumer-side piece descriptor (int4):
//   x = rows << 16 | cols, y = in_off (alias pieces: in_off | smem row stride << 16), z = out_off,
//   w = smem_off | mode << 16 | begin << 20 | end << 21 | direct << 22 | xstage << 23 | alias << 24
// An alias piece (packer_sym) copies nothing: it re-reads a column sub-block of the rows the
// N piece before it staged, as a T / H product (one HBM read, the product and its mirror).
constexpr int kCBegin = 1 << 20, kCEnd = 1 << 21, kCDirect = 1 << 22, kCXStage = 1 << 23,
              kCAlias = 1 << 24;

struct OpSlot {
    int hdr[16];
    int64_t roff[kSlotRuns];
    int rlen[kSlotRuns];
    int rdst[kSlotRuns];
    int rbf[kSlotRuns];  // buf | flags << 8
    int4 pc[kSlotPieces];
    int op;
    int pad[3];
};

struct Params {
    const double2* arena;
    double2* work;
    const double2* x;
    double2* w;
    const int32_t* ops;
    const int64_t* pieces;
    const int64_t* runs;
    const int32_t* waits;
    const int32_t* sigs;
    const int32_t* fused_order;
    int32_t op_count;
    int32_t nstage;
    int32_t stage_bytes;  // 16 x program.stage_elems
    uint32_t* counters;
    unsigned long long* ticket;
    uint32_t* exit_count;
    int32_t n_counters;
    int32_t xin_max;
    int32_t out_max;
    int32_t skip_waits;        // diagnostics: ignore dependencies (results are wrong)
    int32_t dbg;               // diagnostics: 1 skip compute, 2 skip gather/scatter (wrong results)
    unsigned long long* prof;  // optional [grid][64] cycle counters, else null
    // ---- peer-exchange programs only (PEER kernels, packer pack(peer=True)) ----
    int32_t rank, world;
    uint32_t epoch;     // 1, 2, ...: counters are monotonic, a wait for n arrivals needs n x epoch
    int32_t n_ctas;     // CTAs running this rank's program (the self-reset's exit count)
    double2* peer_work[kMaxRanks];       // every rank's work buffer, this epoch's half ([rank] = work)
    uint32_t* peer_counters[kMaxRanks];  // every rank's dependency counters
    uint32_t* peer_done[kMaxRanks];      // every rank's done-epoch array (world uint32 each)
    uint32_t* done;                      // this rank's done-epoch array: done[q] = last epoch q finished
    uint32_t* diag;     // optional host-mapped record of a timed-out wait (rank, what, value, need)
    const double2* x_host;  // host-I/O programs: device-visible pointers of the pinned host x / w
    double2* w_host;
    unsigned long long* trace;  // diagnostics (PROF kernels): per op {start, deps ready, end, cta} ns
    int32_t spin_log2;  // bounded spin of the peer waits: 2^spin_log2 polls, then trap
};

// One launch running the programs of several ranks (peer-exchange emulation of a multi-GPU
// partition on one GPU: CTAs [r*G/n, (r+1)*G/n) run rank r).  A real multi-GPU rank launches it
// with n = 1 and its peers' NVLink-mapped pointers.
struct PeerLaunch {
    Params r[kMaxRanks];
    int32_t nranks;
};

// prof layout per CTA (64 x u64): [kind * 8 + c] for op kinds 0..6 with c = 0 consumer waiting
// for stage data, 1 dependency wait, 2 compute, 3 op prologue/epilogue, 4 pieces, 5 ops;
// [56] producer waiting for a free stage, [57] producer waiting for a free op slot,
// [58 + w] consumer warp w waiting for stage data (all kinds).

struct Layout {
    int stage_off, xin_off, out_off, slot_off, bar_off, prof_off, total;
};

__host__ __device__ inline Layout layout(int nstage, int stage_bytes, int xin_max, int out_max) {
    Layout L;
    L.stage_off = 0;
    L.xin_off = nstage * stage_bytes;
    L.out_off = L.xin_off + ((xin_max * 16 + 127) & ~127);
    L.slot_off = L.out_off + ((out_max * 16 + 127) & ~127);
    L.bar_off = L.slot_off + kOpSlots * (int)sizeof(OpSlot);
    L.prof_off = L.bar_off + (2 * nstage + 2 * kOpSlots) * 8 + 16;
    L.total = L.prof_off + 64 * 8;
    return L;
}

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
            su32(b)),
        "r"(bytes)
        : "memory");
}
// Blocking wait: with a suspend-time hint the warp sleeps in hardware until the phase
// completes instead of re-issuing try_wait (spinning warps stole issue slots from consumers).
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(su32(b)),
        "r"(parity), "r"(0x989680)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_add(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// system scope (peer-exchange programs: counters and flags another GPU writes over NVLink)
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_relaxed_add_sys(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Bounded spin of the peer-exchange waits: a peer that never arrives (a dead rank) traps the
// kernel after ~20 s instead of hanging the GPU.
template <bool PEER>
__device__ __forceinline__ void wait_count(const uint32_t* c, uint32_t need, const Params& p, uint32_t what) {
    if (!PEER) {
        while (ld_acquire(c) < need) __nanosleep(20);
        return;
    }
    long long spins = 0;
    uint32_t v;
    while ((int32_t)((v = ld_acquire_sys(c)) - need) < 0) {  // wrap-safe: counters grow monotonically
        __nanosleep(32);
        if (++spins > (1ll << p.spin_log2)) {
            if (p.diag) {  // record (up to 63 waits), then give the others time to record too
                const uint32_t i = atomicAdd(p.diag, 1u);
                if (i < 63) {
                    uint32_t* rec = p.diag + 8 + 8 * i;
                    rec[0] = (uint32_t)p.rank;
                    rec[1] = what;
                    rec[2] = v;
                    rec[3] = need;
                    rec[4] = p.epoch;
                    rec[5] = blockIdx.x;
                    rec[6] = 1;
                }
                __threadfence_system();
                for (int k = 0; k < 4096; ++k) __nanosleep(1000000);
            }
            __trap();
        }
    }
}
// Signal counters sigs[b..e) once every prior write of the CTA (ordered before the caller by
// a bar.sync) is visible: ONE release fence, then relaxed adds (a release pattern each).
__device__ __forceinline__ void signal_counters(uint32_t* counters, const int32_t* sigs, int b, int e) {
    if (e - b == 1) {
        red_release_add(counters + __ldg(sigs + b), 1u);
        return;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    for (int i = b; i < e; ++i) red_relaxed_add(counters + __ldg(sigs + i), 1u);
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

__device__ __forceinline__ int4 compress_piece(int64_t rows, int64_t cols, int64_t mode,
                                               int64_t in_off, int64_t out_off, int64_t info) {
    int4 c;
    c.x = (int)((rows << 16) | cols);
    c.y = (info & kPiAlias) ? (int)(in_off | (((info >> 32) & 0xFFFF) << 16)) : (int)in_off;
    c.z = (int)out_off;
    c.w = (int)((info & 0xFFFF) | (mode << 16) | ((info & kPiBegin) ? kCBegin : 0) |
                ((info & kPiEnd) ? kCEnd : 0) | ((info & kPiDirect) ? kCDirect : 0) |
                ((info & kPiXStage) ? kCXStage : 0) | ((info & kPiAlias) ? kCAlias : 0));
    return c;
}

// Lanes per output column of an H/S piece: columns go round-robin over 128/P thread groups
// in up to kSlots passes; the P lanes of a column (32/P apart in a warp) split its rows and
// are reduced by shuffles at the flush.  (P = 4 up to 128 columns measured slower.)
__device__ __forceinline__ int h_lanes(int cols) { return cols <= 32 ? 4 : (cols <= 64 ? 2 : 1); }

template <bool PROF, bool IO>
__device__ __forceinline__ void producer(const Params& p, unsigned char* stages, uint64_t* full,
                                         uint64_t* empty, uint64_t* opfull, uint64_t* opempty,
                                         OpSlot* slots) {
    const int lane = threadIdx.x & 31;
    uint64_t policy, policy_keep;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy_keep));
    int stage = 0;
    uint32_t sphase = 0;
    int q = 0;
    uint32_t qphase = 0;
    unsigned long long c_empty = 0, c_slot = 0;
    const bool prof = PROF && lane == 0;
    unsigned long long t_next = 0;
    if (lane == 0) t_next = atomicAdd(p.ticket, 1ull);
    t_next = __shfl_sync(0xffffffffu, t_next, 0);
    for (;;) {
        const int op = (t_next < (unsigned long long)p.op_count) ? __ldg(p.fused_order + t_next) : -1;
        int hv = 0;
        if (op >= 0) {
            if (lane < 16) hv = __ldg(p.ops + (int64_t)op * 16 + lane);
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(p.ticket, 1ull);  // next op, overlapped with this one
            t_next = __shfl_sync(0xffffffffu, t, 0);
        }
        const int in_b = __shfl_sync(0xffffffffu, hv, 2);
        const int out_e = __shfl_sync(0xffffffffu, hv, 7);
        const int pc_b = __shfl_sync(0xffffffffu, hv, 13);
        const int pc_e = __shfl_sync(0xffffffffu, hv, 14);
        const long long tq = prof ? clock64() : 0;
        mbar_wait(&opempty[q], qphase ^ 1u);
        if (prof) c_slot += clock64() - tq;
        // fill the op slot: header, run table, first kSlotPieces compressed piece descriptors
        OpSlot* S = slots + q;
        if (lane < 16) S->hdr[lane] = hv;
        if (lane == 0) S->op = op;
        const int n_runs = op >= 0 ? out_e - in_b : 0;
        for (int r = lane; r < n_runs && r < kSlotRuns; r += 32) {
            const int64_t* rd = p.runs + (int64_t)(in_b + r) * kRunFields;
            S->roff[r] = __ldg(rd + 1);
            S->rlen[r] = (int)__ldg(rd + 2);
            S->rdst[r] = (int)__ldg(rd + 3);
            S->rbf[r] = (int)(__ldg(rd + 0) | (__ldg(rd + 4) << 8));
        }
        const int n_pc = op >= 0 ? pc_e - pc_b : 0;
        for (int i = lane; i < n_pc && i < kSlotPieces; i += 32) {
            const int64_t* d = p.pieces + (int64_t)(pc_b + i) * kPieceFields;
            S->pc[i] = compress_piece(__ldg(d + 2), __ldg(d + 3), __ldg(d + 4), __ldg(d + 5),
                                      __ldg(d + 6), __ldg(d + 7));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&opfull[q]);  // release: the slot writes above are visible
        if (IO && op >= 0 && (__shfl_sync(0xffffffffu, hv, 12) & kOpXWait)) {
            // host-I/O NEAR op: its x windows are published to device x by P1 ops (generic
            // stores); wait for them, then order the bulk copies (async proxy) after the acquire
            const int wb = __shfl_sync(0xffffffffu, hv, 8), we = __shfl_sync(0xffffffffu, hv, 9);
            for (int i = wb + lane; i < we; i += 32) {
                const int c = __ldg(p.waits + 2 * i);
                const uint32_t need = (uint32_t)__ldg(p.waits + 2 * i + 1);
                while (ld_acquire(p.counters + c) < need) __nanosleep(32);
            }
            __syncwarp();
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        if (++q == kOpSlots) {
            q = 0;
            qphase ^= 1u;
        }
        if (op < 0) {
            if (prof) {
                p.prof[(size_t)blockIdx.x * 64 + 56] = c_empty;
                p.prof[(size_t)blockIdx.x * 64 + 57] = c_slot;
            }
            break;
        }
        for (int base = pc_b; base < pc_e; base += 32) {
            const int nb = min(32, pc_e - base);
            int64_t f0 = 0, f1 = 0, f7 = kPiDirect, f5 = 0;
            int rc = 0, md = 0;
            if (lane < nb) {
                const int64_t* d = p.pieces + (int64_t)(base + lane) * kPieceFields;
                f0 = __ldg(d + 0);
                f1 = __ldg(d + 1);
                rc = (int)((__ldg(d + 2) << 16) | __ldg(d + 3));
                md = (int)__ldg(d + 4);
                f5 = __ldg(d + 5);
                f7 = __ldg(d + 7);
            }
            for (int k = 0; k < nb; ++k) {
                const int64_t info = __shfl_sync(0xffffffffu, f7, k);
                if (info & kPiDirect) continue;
                const int64_t m_off = __shfl_sync(0xffffffffu, f0, k);
                const int64_t ld = __shfl_sync(0xffffffffu, f1, k);
                const int rcv = __shfl_sync(0xffffffffu, rc, k);
                const int rows = rcv >> 16, cols = rcv & 0xFFFF;
                const int pmode = __shfl_sync(0xffffffffu, md, k);
                const int64_t xo = __shfl_sync(0xffffffffu, f5, k);
                if (info & kPiBegin) {
                    const long long te = prof ? clock64() : 0;
                    mbar_wait(&empty[stage], sphase ^ 1u);
                    if (prof) c_empty += clock64() - te;
                    if (lane == 0)
                        mbar_arrive_expect_tx(&full[stage], (uint32_t)(((info >> 32) & 0xFFFFFF) * 16));
                }
                if (lane == 0 && !(info & kPiAlias)) {  // (alias pieces re-read staged rows)
                    unsigned char* dst =
                        stages + (size_t)stage * p.stage_bytes + (size_t)(info & 0xFFFFFF) * 16;
                    const double2* src = p.arena + m_off;
                    if (ld == cols) {
                        bulk_g2s(dst, src, (uint32_t)rows * cols * 16, &full[stage], policy);
                    } else {
                        for (int r = 0; r < rows; ++r)
                            bulk_g2s(dst + (size_t)r * cols * 16, src + (int64_t)r * ld,
                                     (uint32_t)cols * 16, &full[stage], policy);
                    }
                    if (info & kPiXStage) {  // the piece's x window, right behind its rows
                        const int w = (pmode == kModeN || pmode == kModeNW) ? cols : rows;
                        bulk_g2s(dst + (size_t)rows * cols * 16, p.x + xo, (uint32_t)w * 16,
                                 &full[stage], policy_keep);
                    }
                }
                if (info & kPiEnd) {
                    if (++stage == p.nstage) {
                        stage = 0;
                        sphase ^= 1u;
                    }
                }
            }
        }
    }
}

struct RunRef {
    int64_t off;
    int len, dst, bf;
};

__device__ __forceinline__ RunRef get_run(const Params& p, const OpSlot* S, int base, int r) {
    RunRef R;
    if (r < kSlotRuns) {
        R.off = S->roff[r];
        R.len = S->rlen[r];
        R.dst = S->rdst[r];
        R.bf = S->rbf[r];
    } else {
        const int64_t* rd = p.runs + (int64_t)(base + r) * kRunFields;
        R.off = __ldg(rd + 1);
        R.len = (int)__ldg(rd + 2);
        R.dst = (int)__ldg(rd + 3);
        R.bf = (int)(__ldg(rd + 0) | (__ldg(rd + 4) << 8));
    }
    return R;
}

// run containing vector position pos among runs [lo, hi) (sorted by dst, contiguous cover)
__device__ __forceinline__ int find_run(const Params& p, const OpSlot* S, int base, int lo, int hi,
                                        int pos) {
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        const int d = (mid < kSlotRuns) ? S->rdst[mid] : (int)__ldg(p.runs + (int64_t)(base + mid) * kRunFields + 3);
        if (d <= pos) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int4 get_piece(const Params& p, const OpSlot* S, int pc_b, int i) {
    if (i < kSlotPieces) return S->pc[i];
    const int64_t* d = p.pieces + (int64_t)(pc_b + i) * kPieceFields;
    return compress_piece(__ldg(d + 2), __ldg(d + 3), __ldg(d + 4), __ldg(d + 5), __ldg(d + 6),
                          __ldg(d + 7));
}

template <bool PROF, bool PEER, bool IO, bool SYM, bool XWIN = false>
__device__ __forceinline__ void consumer(const Params& p, unsigned char* stages, double2* xin,
                                         double2* outv, uint64_t* full, uint64_t* empty,
                                         uint64_t* opfull, uint64_t* opempty, OpSlot* slots,
                                         unsigned long long* sprof) {
    const int tid = threadIdx.x;  // 0..127
    const int lane = tid & 31;
    const int g = tid & (kLanesPerRow - 1);
    const int rg = tid / kLanesPerRow;
    const unsigned gmask = 0xffu << (lane & ~(kLanesPerRow - 1));
    int stage = 0;
    uint32_t sphase = 0;
    int q = 0;
    uint32_t qphase = 0;
    const bool prof = PROF && tid == 0;
    unsigned long long* pr = prof ? sprof : nullptr;
    for (;;) {
        long long t0 = prof ? clock64() : 0;
        mbar_wait(&opfull[q], qphase);
        const OpSlot* S = slots + q;
        const int op = S->op;
        if (op < 0) {
            if (prof)
                for (int i = 0; i < 56; ++i) p.prof[(size_t)blockIdx.x * 64 + i] = sprof[i];
            __syncwarp();
            if (PROF && lane == 0) p.prof[(size_t)blockIdx.x * 64 + 58 + ((tid >> 5) & 3)] = sprof[58 + ((tid >> 5) & 3)];
            break;
        }
        if (PROF && tid == 0 && p.trace) {
            p.trace[(size_t)op * 4 + 0] = globaltimer_ns();
            p.trace[(size_t)op * 4 + 3] = blockIdx.x;
        }
        const int n_out = S->hdr[1];
        const int in_b = S->hdr[2], in_e = S->hdr[3];
        const int out_e = S->hdr[7];
        const int pc_b = S->hdr[13], pc_e = S->hdr[14];
        const int kind = S->hdr[12] & 7;
        const bool peer_op = PEER && (S->hdr[12] & kOpPeer);  // (read while the slot is held)
        const bool xhost = IO && (S->hdr[12] & kOpXHost) != 0;
        const bool drain_op = IO && (S->hdr[12] & kOpDrain) != 0;
        const bool dual = SYM && (S->hdr[12] & kOpDual) != 0;
        const int n_in_runs = in_e - in_b;
        const int n_runs = out_e - in_b;
        if (!(kDiag && p.skip_waits)) {  // every consumer thread polls one dependency counter in parallel
            const int wb = S->hdr[8], we = S->hdr[9];
            for (int i = wb + tid; i < we; i += kConsumers) {
                const int c = __ldg(p.waits + 2 * i);
                const uint32_t need = (uint32_t)__ldg(p.waits + 2 * i + 1);
                wait_count<PEER>(p.counters + c, PEER ? need * p.epoch : need, p, (uint32_t)c);
            }
            // peer data of epoch e lands in the peers' work half e & 1, which peer q last read
            // in epoch e - 2: wait until q has finished it (almost always long done)
            if (peer_op && tid < p.world && tid != p.rank && p.epoch > 2)
                wait_count<true>(p.done + tid, p.epoch - 2, p, 0x80000000u | tid);
        }
        consumer_sync();
        if (prof) {
            const long long t1 = clock64();
            pr[kind * 8 + 1] += t1 - t0;
            t0 = t1;
            pr[kind * 8 + 5] += 1;
            if (p.trace) p.trace[(size_t)op * 4 + 1] = globaltimer_ns();
        }
        // gather the input vector: all loads of a batch issued before any smem store
        const int n_in = (kDiag && (p.dbg & 2)) ? 0 : S->hdr[15];  // work inputs only (x rides in stages)
        const bool xwin = XWIN && (S->hdr[12] & kOpXWin) != 0;
        const int n_in_all = xwin ? S->hdr[0] : n_in;  // windowed: hdr[15] is the window length
        int xw_lo = 0;
        auto gather = [&](int lo, int hi) {  // positions [lo, hi) of the input -> xin[pos - lo]
            for (int base = lo; base < hi; base += kGatherBatch * kConsumers) {
                double2 v[kGatherBatch];
#pragma unroll
                for (int k = 0; k < kGatherBatch; ++k) {
                    const int pos = base + tid + k * kConsumers;
                    if (pos < hi) {
                        const RunRef R = get_run(p, S, in_b, find_run(p, S, in_b, 0, n_in_runs, pos));
                        const int64_t src = R.off + (pos - R.dst);
                        if ((R.bf & 0xFF) != kBufX) v[k] = __ldcg(p.work + src);
                        else v[k] = xhost ? __ldcg(p.x_host + src) : __ldg(p.x + src);  // host: over PCIe
                    }
                }
#pragma unroll
                for (int k = 0; k < kGatherBatch; ++k) {
                    const int pos = base + tid + k * kConsumers;
                    if (pos < hi) {
                        xin[pos - lo] = v[k];
                        // host-I/O P1 op: its one input run is x[a:b] -- publish it for the NEAR ops
                        if (xhost) __stcg(const_cast<double2*>(p.x) + S->roff[0] + pos, v[k]);
                    }
                }
            }
        };
        gather(0, xwin ? min(n_in, n_in_all) : n_in);
        for (int i = tid; i < n_out; i += kConsumers) outv[i] = make_double2(0.0, 0.0);
        consumer_sync();

        double accr[kSlots], acci[kSlots];
        const bool nreg = n_out <= kSlots * kRowGroups && !dual;
        // single-slot N ops (every NEAR op; n_out <= 16): row group rg owns output row rg in every
        // piece, so the four accumulation chains of its row live in accr / acci[0..3] across the
        // whole N group -- no per-row zeroing, fold or slot select (the narrow 40-column dense rows
        // of configs 1-2 spent most of their instructions there)
        const bool nacc1 = UHMV_NACC1 && n_out <= kRowGroups && !dual;
        int g_mode = -1, g_out = 0, g_cols = 0;
        auto flush = [&]() {
            if (g_mode == kModeN) {
                if (nacc1) {
                    double ar = (accr[0] + accr[1]) + (accr[2] + accr[3]);
                    double ai = (acci[0] + acci[1]) + (acci[2] + acci[3]);
#pragma unroll
                    for (int o = 1; o < kLanesPerRow; o <<= 1) {
                        ar += __shfl_xor_sync(0xffffffffu, ar, o);
                        ai += __shfl_xor_sync(0xffffffffu, ai, o);
                    }
                    if (g == 0 && rg < n_out) {
                        double2 v = outv[rg];
                        v.x += ar;
                        v.y += ai;
                        outv[rg] = v;
                    }
                } else if (nreg) {
#pragma unroll
                    for (int k = 0; k < kSlots; ++k) {
                        if (k * kRowGroups >= n_out) break;
                        double ar = accr[k], ai = acci[k];
#pragma unroll
                        for (int o = 1; o < kLanesPerRow; o <<= 1) {
                            ar += __shfl_xor_sync(0xffffffffu, ar, o);
                            ai += __shfl_xor_sync(0xffffffffu, ai, o);
                        }
                        const int o = k * kRowGroups + rg;
                        if (g == 0 && o < n_out) {
                            double2 v = outv[o];
                            v.x += ar;
                            v.y += ai;
                            outv[o] = v;
                        }
                    }
                }
            } else if (g_mode == kModeH || g_mode == kModeS || (SYM && g_mode == kModeT)) {  // (NW: outv directly)
                const int P = h_lanes(g_cols);
                const int nJ = kConsumers / P;
                const int cw = 32 / P;  // columns per warp: lane = column + cw * row offset
                const int pp = lane / cw;
                const int j0 = wrap_nj((tid >> 5) * cw + (lane & (cw - 1)) - g_out, nJ);
#pragma unroll
                for (int k = 0; k < kSlots; ++k) {
                    if (k * nJ >= g_cols) break;
                    double ar = accr[k], ai = acci[k];
                    for (int o = cw; o < 32; o <<= 1) {
                        ar += __shfl_xor_sync(0xffffffffu, ar, o);
                        ai += __shfl_xor_sync(0xffffffffu, ai, o);
                    }
                    const int j = j0 + k * nJ;
                    if (pp == 0 && j < g_cols) {
                        double2 v = outv[g_out + j];
                        v.x += ar;
                        v.y += ai;
                        outv[g_out + j] = v;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kSlots; ++k) accr[k] = acci[k] = 0.0;
        };
        if (prof) {
            const long long t1 = clock64();
            pr[kind * 8 + 3] += t1 - t0;
            t0 = t1;
        }
        for (int i = 0; i < pc_e - pc_b; ++i) {
            const int4 c = get_piece(p, S, pc_b, i);
            const int c_end = c.w & kCEnd;
            const int rows = c.x >> 16, cols = c.x & 0xFFFF;
            const bool alias = SYM && (c.w & kCAlias) != 0;
            const int in_off = alias ? (c.y & 0xFFFF) : c.y, out_off = c.z;
            const int rs = alias ? (c.y >> 16) : cols;  // smem row stride of the tile
            const int mode = (c.w >> 16) & 0xF;
            const bool direct = (c.w & kCDirect) != 0;
            if (dual) {
                if (mode != kModeN && mode != kModeNW && (g_mode != mode || g_out != out_off || g_cols != cols)) {
                    flush();  // the previous mirrored block's T / H group (disjoint outputs: no barrier)
                    g_mode = mode;
                    g_out = out_off;
                    g_cols = cols;
                }
            } else if ((mode == kModeN || mode == kModeNW) ? (g_mode != mode)
                                                    : (g_mode != mode || g_out != out_off || g_cols != cols)) {
                // row-group (N), warp (NW) and column (H/S) owners differ: order their outv adds
                const bool to_other = g_mode >= 0 && g_mode != mode &&
                                      (g_mode == kModeN || g_mode == kModeNW || mode == kModeN || mode == kModeNW);
                flush();
                if (to_other) consumer_sync();
                g_mode = mode;
                g_out = out_off;
                g_cols = cols;
            }
            if (XWIN && xwin && !(c.w & kCXStage) && (mode == kModeN || mode == kModeNW) &&
                (in_off < xw_lo || in_off + cols > xw_lo + n_in)) {
                consumer_sync();  // every warp is done with the previous window
                gather(in_off, min(n_in_all, in_off + n_in));
                xw_lo = in_off;
                consumer_sync();
            }
            const double2* tile = nullptr;
            if (!direct) {
                if (c.w & kCBegin) {
                    if (prof) {
                        const long long t1 = clock64();
                        pr[kind * 8 + 2] += t1 - t0;
                        t0 = t1;
                    }
                    long long tw = PROF ? clock64() : 0;
                    mbar_wait(&full[stage], sphase);
                    if (PROF && lane == 0) sprof[58 + ((tid >> 5) & 3)] += clock64() - tw;  // every warp
                    if (prof) {
                        const long long t1 = clock64();
                        pr[kind * 8 + 0] += t1 - t0;
                        t0 = t1;
                    }
                }
                tile = reinterpret_cast<const double2*>(stages + (size_t)stage * p.stage_bytes) +
                       (c.w & 0xFFFF);
            }
            if (prof) pr[kind * 8 + 4] += 1;
            if (kDiag && (p.dbg & 1)) {
                // diagnostics: no compute
            } else if (mode == kModeN && nacc1) {
                const double2* xv = (c.w & kCXStage) ? tile + rows * cols : xin + (in_off - xw_lo);
                const int r = wrapc<kRowGroups>(rg - out_off);  // this row group's row, if < rows
                if (r < rows) {
                    const double2* T = tile + r * cols + g;
                    const double2* X = xv + g;
#pragma unroll 2
                    for (int k = cols >> 5; k > 0; --k) {
                        const double2 t0 = T[0], x0 = X[0], t1 = T[8], x1 = X[8];
                        const double2 t2 = T[16], x2 = X[16], t3 = T[24], x3 = X[24];
                        cmac(accr[0], acci[0], t0, x0);
                        cmac(accr[1], acci[1], t1, x1);
                        cmac(accr[2], acci[2], t2, x2);
                        cmac(accr[3], acci[3], t3, x3);
                        T += 32;
                        X += 32;
                    }
                    const int tail = cols & 31;  // warp-uniform: branch over the unused lane groups
                    if (tail) {
                        if (g < tail) cmac(accr[0], acci[0], T[0], X[0]);
                        if (tail > 8) {
                            if (g + 8 < tail) cmac(accr[1], acci[1], T[8], X[8]);
                            if (tail > 16) {
                                if (g + 16 < tail) cmac(accr[2], acci[2], T[16], X[16]);
                                if (tail > 24 && g + 24 < tail) cmac(accr[3], acci[3], T[24], X[24]);
                            }
                        }
                    }
                }
            } else if (mode == kModeN) {
                const double2* xv = (c.w & kCXStage) ? tile + rows * cols : xin + (in_off - xw_lo);
                const int r0 = wrapc<kRowGroups>(rg - out_off);  // first row of this row group
                for (int r = r0; r < rows; r += kRowGroups) {
                    const double2* T = tile + r * cols + g;
                    const double2* X = xv + g;
                    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
                    double cr = 0.0, ci = 0.0, dr = 0.0, di = 0.0;
                    // full 32-column blocks: every lane of the row group has four elements,
                    // unpredicated (cols is warp-uniform per piece); then the ragged tail
                    const int nfull = cols >> 5;
                    for (int k = 0; k < nfull; ++k) {
                        const double2 t0 = T[0], x0 = X[0], t1 = T[8], x1 = X[8];
                        const double2 t2 = T[16], x2 = X[16], t3 = T[24], x3 = X[24];
                        cmac(ar, ai, t0, x0);
                        cmac(br, bi, t1, x1);
                        cmac(cr, ci, t2, x2);
                        cmac(dr, di, t3, x3);
                        T += 32;
                        X += 32;
                    }
                    const int tail = cols & 31;
                    if (g < tail) cmac(ar, ai, T[0], X[0]);
                    if (g + 8 < tail) cmac(br, bi, T[8], X[8]);
                    if (g + 16 < tail) cmac(cr, ci, T[16], X[16]);
                    if (g + 24 < tail) cmac(dr, di, T[24], X[24]);
                    ar += br + (cr + dr);
                    ai += bi + (ci + di);
                    const int o = out_off + r;
                    if (nreg) {
                        const int k = (unsigned)o / kRowGroups;
                        if (k == 0) {
                            accr[0] += ar;
                            acci[0] += ai;
                        } else {
#pragma unroll
                            for (int s = 1; s < kSlots; ++s)
                                if (s == k) {
                                    accr[s] += ar;
                                    acci[s] += ai;
                                }
                        }
                    } else {  // wide N op: reduce and add per row
#pragma unroll
                        for (int s = 1; s < kLanesPerRow; s <<= 1) {
                            ar += __shfl_xor_sync(gmask, ar, s);
                            ai += __shfl_xor_sync(gmask, ai, s);
                        }
                        if (g == 0) {
                            double2 v = outv[o];
                            v.x += ar;
                            v.y += ai;
                            outv[o] = v;
                        }
                    }
                }
            } else if (mode == kModeNW) {
                // wide rows (few per piece): warp per row, 32 lanes x 16 B, reduced across the
                // warp; row o belongs to warp o mod 4 in every piece (deterministic outv adds)
                const double2* xv = (c.w & kCXStage) ? tile + rows * cols : xin + (in_off - xw_lo);
                const int w = tid >> 5;
                for (int r = wrapc<kConsumerWarps>(w - out_off); r < rows; r += kConsumerWarps) {
                    const double2* T = tile + r * cols + lane;
                    const double2* X = xv + lane;
                    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
                    double cr = 0.0, ci = 0.0, dr = 0.0, di = 0.0;
                    const int nfull = cols >> 7;
                    for (int k = 0; k < nfull; ++k) {
                        const double2 t0 = T[0], x0 = X[0], t1 = T[32], x1 = X[32];
                        const double2 t2 = T[64], x2 = X[64], t3 = T[96], x3 = X[96];
                        cmac(ar, ai, t0, x0);
                        cmac(br, bi, t1, x1);
                        cmac(cr, ci, t2, x2);
                        cmac(dr, di, t3, x3);
                        T += 128;
                        X += 128;
                    }
                    const int tail = cols & 127;
                    if (lane < tail) cmac(ar, ai, T[0], X[0]);
                    if (lane + 32 < tail) cmac(br, bi, T[32], X[32]);
                    if (lane + 64 < tail) cmac(cr, ci, T[64], X[64]);
                    if (lane + 96 < tail) cmac(dr, di, T[96], X[96]);
                    ar += br + (cr + dr);
                    ai += bi + (ci + di);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        ar += __shfl_xor_sync(0xffffffffu, ar, o);
                        ai += __shfl_xor_sync(0xffffffffu, ai, o);
                    }
                    if (lane == 0) {
                        double2 v = outv[out_off + r];
                        v.x += ar;
                        v.y += ai;
                        outv[out_off + r] = v;
                    }
                }
            } else {
                const int P = h_lanes(cols);
                const int nJ = kConsumers / P;
                // a quarter-warp reads 8 consecutive columns of one row (conflict-free 16-B
                // loads); the P lanes of a column sit cw apart in the warp
                const int cw = 32 / P;
                const int pp = lane / cw;
                const int j0 = wrap_nj((tid >> 5) * cw + (lane & (cw - 1)) - out_off, nJ);
                int64_t dm = 0, dld = 0;
                if (direct) {
                    const int64_t* d = p.pieces + (int64_t)(pc_b + i) * kPieceFields;
                    dm = __ldg(d + 0);
                    dld = __ldg(d + 1);
                }
#pragma unroll
                for (int k = 0; k < kSlots; ++k) {
                    if (k * nJ >= cols) break;
                    const int j = j0 + k * nJ;
                    if (j >= cols) continue;
                    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
                    if (mode == kModeS) {
                        const double2* W = p.work + dm + j;
#pragma unroll 4
                        for (int r = pp; r < rows; r += P) {
                            const double2 m = __ldcg(W + (int64_t)r * dld);
                            ar += m.x;
                            ai += m.y;
                        }
                    } else if (SYM && mode == kModeT) {  // transpose without conjugation (packer_sym)
                        const double2* xv = (c.w & kCXStage) ? tile + rows * cols : xin + in_off;
                        int r = pp;
                        for (; r + P < rows; r += 2 * P) {
                            cmac(ar, ai, tile[r * rs + j], xv[r]);
                            cmac(br, bi, tile[(r + P) * rs + j], xv[r + P]);
                        }
                        if (r < rows) cmac(ar, ai, tile[r * rs + j], xv[r]);
                    } else {
                        const double2* xv = (c.w & kCXStage) ? tile + rows * cols : xin + in_off;
                        int r = pp;
                        for (; r + P < rows; r += 2 * P) {  // two independent chains
                            cmac_conj(ar, ai, tile[r * rs + j], xv[r]);
                            cmac_conj(br, bi, tile[(r + P) * rs + j], xv[r + P]);
                        }
                        if (r < rows) cmac_conj(ar, ai, tile[r * rs + j], xv[r]);
                    }
                    accr[k] += ar + br;
                    acci[k] += ai + bi;
                }
            }
            if (!direct && c_end) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
                if (++stage == p.nstage) {
                    stage = 0;
                    sphase ^= 1u;
                }
            }
        }
        flush();
        consumer_sync();
        if (prof) {
            const long long t1 = clock64();
            pr[kind * 8 + 2] += t1 - t0;
            t0 = t1;
        }
        // scatter the output vector
        for (int pos = tid; pos < ((kDiag && (p.dbg & 2)) ? 0 : n_out); pos += kConsumers) {
            const RunRef R = get_run(p, S, in_b, find_run(p, S, in_b, n_in_runs, n_runs, pos));
            const int buf = R.bf & 0xFF, flags = R.bf >> 8;
            double2* dp = (buf == kBufW ? p.w : p.work) + R.off + (pos - R.dst);
            const double2 v = outv[pos];
            if (PEER && (flags & kRunPeer)) {  // y/u of this rank: every rank gets a copy
                const int64_t o = R.off + (pos - R.dst);
                for (int q = 0; q < p.world; ++q) __stcg(p.peer_work[q] + o, v);
            } else if (flags & 2) {  // fp64 red.add into the pre-zeroed output (<= 2 addends per entry)
                red_add_f64(&dp->x, v.x);
                red_add_f64(&dp->y, v.y);
            } else if (flags & 1) {
                const double2 o = __ldcg(dp);
                __stcg(dp, make_double2(v.x + o.x, v.y + o.y));
            } else {
                __stcg(dp, v);
            }
        }
        const int sb = S->hdr[10], se = S->hdr[11];
        consumer_sync();  // all outputs issued; the slot is no longer read
        if (lane == 0) mbar_arrive(&opempty[q]);
        if (tid == 0 && !(kDiag && p.skip_waits) && se > sb) {
            if (peer_op) {  // (the slot may already hold another op: flag read at op start)
                // the CTA's local and peer stores precede the system-scope fence through the
                // bar.sync above; then one relaxed add per counter and rank
                asm volatile("fence.acq_rel.sys;" ::: "memory");
                for (int i = sb; i < se; ++i) {
                    const int c = __ldg(p.sigs + i);
                    for (int q = 0; q < p.world; ++q) red_relaxed_add_sys(p.peer_counters[q] + c, 1u);
                }
            } else {
                // red.release.gpu orders every output store of the CTA before the signal: the
                // stores happen-before this thread's release through the bar.sync above
                // (release cumulativity), so no separate fence is needed
                signal_counters(p.counters, p.sigs, sb, se);
            }
        }
        if (drain_op) {
            // host-I/O: count this op's contribution to its output leaf; the last one copies the
            // finished w[leaf] to the host buffer (PCIe writes overlap the rest of the kernel)
            int* dflag = reinterpret_cast<int*>(opempty + kOpSlots) + 1;
            const int64_t* dr = p.runs + (int64_t)(in_b + n_runs) * kRunFields;
            if (tid == 0) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");  // this CTA's w adds first
                const uint32_t old = atomicAdd(p.counters + (int)__ldg(dr + 3), 1u);
                const int last = (old + 1u == (uint32_t)__ldg(dr + 4));
                if (last) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // every CTA's w adds
                *dflag = last;
            }
            consumer_sync();
            if (*dflag) {
                const int64_t lo = __ldg(dr + 1), len = __ldg(dr + 2);
                for (int64_t i = tid; i < len; i += kConsumers) __stcg(p.w_host + lo + i, __ldcg(p.w + lo + i));
            }
        }
        if (++q == kOpSlots) {
            q = 0;
            qphase ^= 1u;
        }
        if (prof) {
            pr[kind * 8 + 3] += clock64() - t0;
            if (p.trace) p.trace[(size_t)op * 4 + 2] = globaltimer_ns();
        }
    }
}

template <bool PROF, bool PEER, bool IO = false, bool SYM = false, bool XWIN = false>
__device__ __forceinline__ void run_cta(const Params& p, int cta, int n_ctas) {
    extern __shared__ __align__(128) unsigned char smem[];
    const Layout L = layout(p.nstage, p.stage_bytes, p.xin_max, p.out_max);
    unsigned char* stages = smem + L.stage_off;
    double2* xin = reinterpret_cast<double2*>(smem + L.xin_off);
    double2* outv = reinterpret_cast<double2*>(smem + L.out_off);
    OpSlot* slots = reinterpret_cast<OpSlot*>(smem + L.slot_off);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + p.nstage;
    uint64_t* opfull = empty + p.nstage;
    uint64_t* opempty = opfull + kOpSlots;
    int* flag = reinterpret_cast<int*>(opempty + kOpSlots);
    unsigned long long* sprof = reinterpret_cast<unsigned long long*>(smem + L.prof_off);
    if (threadIdx.x < 64) sprof[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.nstage; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        for (int s = 0; s < kOpSlots; ++s) {
            mbar_init(&opfull[s], 1);
            mbar_init(&opempty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp == kConsumerWarps) {
        producer<PROF, IO>(p, stages, full, empty, opfull, opempty, slots);
    } else {
        consumer<PROF, PEER, IO, SYM, XWIN>(p, stages, xin, outv, full, empty, opfull, opempty, slots, sprof);
    }
    __syncthreads();
    // self-reset: the last CTA out zeroes the counters and the ticket for the next launch
    // (peer programs keep their counters: monotonic, every wait scaled by the epoch)
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(p.exit_count, 1u);
        flag[0] = (prev == (uint32_t)n_ctas - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag[0]) {
        __threadfence();
        if (!PEER)
            for (int i = threadIdx.x; i < p.n_counters; i += kThreads) p.counters[i] = 0u;
        if (threadIdx.x == 0) {
            *p.ticket = 0ull;
            *p.exit_count = 0u;
        }
        __threadfence();
        if (PEER && threadIdx.x == 0) {
            // every CTA of this rank is done with the epoch's work half: tell every rank
            __threadfence_system();
            for (int q = 0; q < p.world; ++q) st_release_sys(p.peer_done[q] + p.rank, p.epoch);
        }
    }
    (void)cta;
}

template <bool PROF>
__global__ void __maxnreg__(UHMV_BULK_REGS) uhmv_bulk_kernel(const Params p) {
    run_cta<PROF, false>(p, blockIdx.x, gridDim.x);
}

// Symmetric single-triangle programs (packer_sym, UHMV_PROG_SYM): T-mode and alias pieces.
template <bool PROF>
__global__ void __maxnreg__(UHMV_BULK_REGS) uhmv_bulk_sym_kernel(const Params p) {
    run_cta<PROF, false, false, true>(p, blockIdx.x, gridDim.x);
}

// Programs with windowed-input ops (packer_h FAR, UHMV_PROG_XWIN): the H format at 3 CTAs/SM.
template <bool PROF>
__global__ void __maxnreg__(UHMV_BULK_REGS) uhmv_bulk_xwin_kernel(const Params p) {
    run_cta<PROF, false, false, false, true>(p, blockIdx.x, gridDim.x);
}

// Host-I/O programs (uhmv_matvec_host with pinned buffers): x gathered over PCIe by the P1
// ops, finished output leaves drained to the host by their last NEAR / FAR op.
__global__ void __maxnreg__(UHMV_BULK_REGS) uhmv_bulk_io_kernel(const Params p) {
    run_cta<false, false, true>(p, blockIdx.x, gridDim.x);
}

// Peer-exchange programs: L.nranks ranks share the grid (n = 1 on a real multi-GPU rank).
__global__ void __maxnreg__(UHMV_BULK_REGS) uhmv_bulk_peer_kernel(const __grid_constant__ PeerLaunch L) {
    const int n = L.nranks;
    const int r = (int)(((long long)blockIdx.x * n) / gridDim.x);
    const int lo = (int)(((long long)r * gridDim.x + n - 1) / n);
    const int hi = (int)(((long long)(r + 1) * gridDim.x + n - 1) / n);
    run_cta<false, true>(L.r[r], blockIdx.x - lo, hi - lo);
}

}  // namespace bulk
