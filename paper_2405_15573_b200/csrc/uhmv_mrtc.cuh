// uhmv_mrtc.cuh -- multi-RHS uniform-H product, shared-memory-staged FP64 tensor-core engine.
//
// Same op programs, fused ticket order and dependency counters as the single-RHS engines; every
// segment group is a small complex GEMM  OUT (nout x R) += op(T) (nout x K) * IN (K x R)  on
// DMMA (mma.sync.aligned.m16n8k16.row.col.f64) through the complex -> real embedding:
//
//   D (2R' x n) += A' (2R' x 2K) * B' (2K x n),  A' = embedded IN^T,  B' = T read as reals.
//
// Warp specialisation (one CTA of 8 consumer warps + 1 producer warp per SM):
//   * the producer warp claims ops, polls their dependency counters (ld.acquire.gpu), then
//     streams every K-chunk of every segment -- KC = 16 complex inputs: the matching T slab
//     (N: nout rows x KC, H: KC rows x nout) as 2-D TMA tensor boxes (one map pair per leading
//     dimension over the whole arena, cp.async.bulk.tensor) and the IN block (KC rows x 64
//     RHS, contiguous) as one cp.async.bulk -- into a 6-deep shared-memory ring completing on
//     mbarriers: 2-6 copy instructions per 16 KFLOP/lane stage;
//   * for every group pass the producer also publishes a PASS descriptor in a shared-memory
//     ring (what to do, how many stages, the destination of every output row, atomic flags),
//     so the consumers never read the op tables, never search output runs and never meet at
//     a barrier inside an op; op boundaries travel through the same ring;
//   * the consumer warps own a fixed (16-RHS, n-tile) share of the output block, accumulate
//     the whole segment group in registers (up to 2 x 5 DMMA tiles per warp) and flush it once
//     (fp64 atomics into w -- at most two addends per entry, so order-independent -- a store
//     for the first group on a work output range, read-add-write for a later one).
//
// Fragment mapping.  The mma k index (16 reals = 8 complex) and the RHS rows are permuted so
// that every lane reads whole complex numbers with 16-B shared loads and no selects:
//   lane (g = lane>>2, t = lane&3); logical mma k = t + 4j  <->  physical real k = 4t + j,
//   i.e. complex inputs 2t and 2t+1 of the k-step; A rows m = g + 8d hold RHS g, part d.
//   A (N: {re,-im; im,re}, H: {re,im; im,-re}) from z0 = IN[2t][g], z1 = IN[2t+1][g];
//   B = T[n][2t], T[n][2t+1] (N) or T[2t][n], T[2t+1][n] (H) with n = g;
//   D: v = e + 2d -> out[2t+e][g], part d: every lane flushes whole complex outputs.
// Shared-memory row pitches (in complex) are the TMA box widths -- IN rpn, T_N 16, T_H 80 --
// so some loads take 2-4 bank wavefronts; at one DMMA per 32 clk per SM sub-partition the
// shared-memory pipe stays far below its limit (ncu: ~10%).

#pragma once

namespace mrtc {

constexpr int kCW = 8;                  // consumer warps
constexpr int kCT = kCW * 32;           // consumer threads
constexpr int kThreads = kCT + 32;      // + producer warp
constexpr int kRP = 64;                 // complex RHS per pass
constexpr int kNP = 80;                 // outputs per pass
constexpr int kKC = 16;                 // complex inputs per stage
constexpr int kNST = 6;                 // ring depth
constexpr int kMaxNT = 5;               // n-tiles per warp
constexpr int kLdTN = kKC;              // N slab [nout][16] (TMA boxes of 16 rows x 16 complex)
constexpr int kLdTH = kNP;              // H slab [16][80]   (one TMA box of 16 rows x 80 complex)
constexpr int kTElems = (kNP * kLdTN > kKC * kLdTH) ? kNP * kLdTN : kKC * kLdTH;
constexpr int kIElems = kKC * kRP;      // IN block [16][rpn] (one bulk copy when rpn == R)
constexpr int kStageElems = kTElems + kIElems;  // complex
constexpr int kPassSlots = 4;           // pass-descriptor ring depth
constexpr int kSmemStages = kNST * kStageElems * 16;

// One unit of consumer work, published by the producer (see the header comment).
enum PassType : int32_t { kPassExit = 0, kPassGemm = 1, kPassSum = 2, kPassEndOp = 3, kPassZero = 4 };
struct __align__(16) Pass {
    int32_t type, op, kind, hm;
    int32_t first;  // flush stores (first group on these outputs) instead of read-add-write
    int32_t sync;   // meet at a consumer barrier before the flush (outputs of an earlier group)
    int32_t rp, rpn, np, nst;  // RHS pass, outputs of the pass, ring stages it consumes
    int32_t s_rows, s_j0;      // kPassSum: partial vectors and first column
    int64_t s_moff, s_ld;      // kPassSum: partial block (work element offset, row stride)
    uint32_t atom[(kNP + 31) / 32];  // bit n: output n is in w (fp64 atomics)
    double2* out[kNP];         // destination of output n, RHS 0 (row stride nrhs)
};
constexpr int kSmemBytes = kSmemStages + kPassSlots * (int)sizeof(Pass) + kNST * 4 +
                           (2 * kNST + 2 * kPassSlots) * 8 + 32 + 48 * 8;

using mrhs::Params;
using bulk::mbar_arrive;
using bulk::mbar_arrive_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::su32;

__device__ __forceinline__ void cons_sync() {
    asm volatile("bar.sync 2, %0;" ::"n"(kCT) : "memory");
}

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}

__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}

struct SegD {
    int64_t m_off, ld, in_abs;
    int rows, cols, mode, in_buf, out_off;
    int first;  // first group writing these outputs: the flush stores (packer.MR_FIRST)
    int tmap;   // index of the TMA map pair of this segment's leading dimension
};

__device__ __forceinline__ SegD seg_at(const Params& p, int i) {
    const int64_t* d = p.mr_segs + (int64_t)i * 8;
    SegD s;
    s.m_off = __ldg(d + 0);
    s.ld = __ldg(d + 1);
    s.rows = (int)__ldg(d + 2);
    s.cols = (int)__ldg(d + 3);
    const int mf = (int)__ldg(d + 4);
    s.mode = mf & 0xFF;
    s.first = (mf >> 8) & 1;
    s.tmap = mf >> 16;
    s.in_buf = (int)__ldg(d + 5);
    s.in_abs = __ldg(d + 6);
    s.out_off = (int)__ldg(d + 7);
    return s;
}
__device__ __forceinline__ int seg_nout(const SegD& s) { return s.mode == kModeN ? s.rows : s.cols; }
__device__ __forceinline__ int seg_k(const SegD& s) { return s.mode == kModeN ? s.cols : s.rows; }

// end of the segment group starting at s (same mode and outputs)
__device__ __forceinline__ int group_end(const Params& p, int s, int se, const SegD& s0) {
    const int nout = seg_nout(s0);
    int e = s + 1;
    while (e < se) {
        const SegD sn = seg_at(p, e);
        if (sn.mode != s0.mode || sn.first != s0.first || sn.out_off != s0.out_off || seg_nout(sn) != nout)
            break;
        ++e;
    }
    return e;
}

// End of the run of N segments starting at si that are consecutive column ranges of ONE
// arena matrix (the packer cuts F_s / Y_t at the boundaries of their input runs); the
// producer streams such a run as one K range so 16-wide chunks are not padded per piece.
// *K receives the run's total width.
__device__ __forceinline__ int merged_end(const Params& p, int si, int e, int* K) {
    const SegD a = seg_at(p, si);
    int k = seg_k(a), sj = si + 1;
    if (a.mode == kModeN) {
        while (sj < e) {
            const SegD b = seg_at(p, sj);
            if (b.ld != a.ld || b.rows != a.rows || b.m_off != a.m_off + k) break;
            k += b.cols;
            ++sj;
        }
    }
    *K = k;
    return sj;
}

// Diagnostics (PROF): per-CTA cycle counters, summed by DeviceOperator.profile_mr --
//   [0] producer waiting for a free stage   [1] producer waiting on dependencies
//   [2] producer issuing (stages + pass descriptors)   [3] producer ticket
//   [8 + 4*kind + {0 wait data, 1 mma, 2 flush, 3 S reduction}]  consumer warp 0
//   [40] consumer warp 0 waiting for a pass descriptor

// Producer side of the pass ring: claim slot, fill it (all lanes), publish.
struct PassRing {
    Pass* slots;
    uint64_t* full;
    uint64_t* empty;
    int q;
    uint32_t phase;
    __device__ __forceinline__ Pass* claim() {
        mbar_wait(&empty[q], phase ^ 1u);
        return slots + q;
    }
    __device__ __forceinline__ void publish(int lane) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[q]);  // release: the lanes' slot writes precede it
        if (++q == kPassSlots) {
            q = 0;
            phase ^= 1u;
        }
    }
};

// destination table of outputs [o0, o0 + np) of an op (binary search over its out runs)
__device__ __forceinline__ void fill_outputs(const Params& p, Pass* ps, int out_b, int out_e, int o0, int np,
                                             int lane) {
    for (int w = lane; w < (kNP + 31) / 32; w += 32) ps->atom[w] = 0u;
    __syncwarp();
    for (int n = lane; n < np; n += 32) {
        bool at;
        ps->out[n] = mrhs::out_ptr(p, out_b, out_e, o0 + n, &at);
        if (at) atomicOr(&ps->atom[n >> 5], 1u << (n & 31));
    }
}

template <bool PROF>
__device__ void producer(const Params& p, double2* stages, int* s_kv, uint64_t* full, uint64_t* empty,
                         PassRing ring, unsigned long long* pr) {
    const int lane = threadIdx.x & 31;
    const int R = p.nrhs;
    uint32_t stage = 0, sphase = 0;
    for (;;) {
        long long t0 = PROF ? clock64() : 0;
        int op = -1;
        if (lane == 0) {
            const unsigned long long tk = atomicAdd(p.ticket, 1ull);
            op = (tk < (unsigned long long)p.op_count) ? __ldg(p.fused_order + tk) : -1;
        }
        op = __shfl_sync(0xffffffffu, op, 0);
        if (PROF && lane == 0) {
            const long long t1 = clock64();
            pr[3] += t1 - t0;
            t0 = t1;
        }
        if (op < 0) {
            Pass* ps = ring.claim();
            if (lane == 0) ps->type = kPassExit;
            ring.publish(lane);
            break;
        }
        const int32_t* hp = p.ops + (int64_t)op * kOpFields;
        {
            const int wb = __ldg(hp + 8), we = __ldg(hp + 9);
            for (int i = wb + lane; i < we; i += 32) {
                const int c = __ldg(p.waits + 2 * i);
                const uint32_t need = (uint32_t)__ldg(p.waits + 2 * i + 1);
                while (ld_acquire(p.counters + c) < need) __nanosleep(32);
            }
            __syncwarp();
            // work inputs written by other CTAs (generic proxy) are read below by the TMA
            // engine; the consumers' work reads (S passes) are ordered by the pass ring
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        if (PROF && lane == 0) {
            const long long t1 = clock64();
            pr[1] += t1 - t0;
            t0 = t1;
        }
        const int out_b = __ldg(hp + 6), out_e = __ldg(hp + 7);
        const int kind = __ldg(hp + 12);
        if (__ldg(p.mr_ranges + 3 * op + 2) & 1) {  // packer.MR_ZERO (no such op at configs 1-4)
            Pass* ps = ring.claim();
            if (lane == 0) {
                ps->type = kPassZero;
                ps->op = op;
                ps->kind = kind;
            }
            ring.publish(lane);
        }
        const int sb = __ldg(p.mr_ranges + 3 * op), se = __ldg(p.mr_ranges + 3 * op + 1);
        int s = sb;
        bool prior = false;  // an earlier group of this op was flushed
        while (s < se) {
            const SegD s0 = seg_at(p, s);
            const int e = group_end(p, s, se, s0);
            const int nout = seg_nout(s0);
            const bool need_sync = prior && !s0.first;  // adds onto an earlier group's outputs
            prior = true;
            if (s0.mode == kModeS) {
                for (int n0 = 0; n0 < nout; n0 += kNP) {
                    for (int si = s; si < e; ++si) {
                        const SegD sg = seg_at(p, si);
                        Pass* ps = ring.claim();
                        if (lane == 0) {
                            ps->type = kPassSum;
                            ps->op = op;
                            ps->kind = kind;
                            ps->first = s0.first && si == s;
                            ps->sync = need_sync && si == s && n0 == 0;
                            ps->np = min(kNP, nout - n0);
                            ps->s_rows = sg.rows;
                            ps->s_j0 = n0;
                            ps->s_moff = sg.m_off;
                            ps->s_ld = sg.ld;
                        }
                        fill_outputs(p, ps, out_b, out_e, s0.out_off + n0, min(kNP, nout - n0), lane);
                        ring.publish(lane);
                    }
                }
                s = e;
                continue;
            }
            const bool hm = s0.mode == kModeH;
            int nst = 0;  // stages of one pass: every K-chunk of every merged segment of the group
            for (int si = s; si < e;) {
                int K = 0;
                si = merged_end(p, si, e, &K);
                nst += (K + kKC - 1) / kKC;
            }
            for (int rp = 0; rp < R; rp += kRP) {
                const int rpn = min(kRP, R - rp);
                for (int n0 = 0; n0 < nout; n0 += kNP) {
                    const int np = min(kNP, nout - n0);
                    Pass* ps = ring.claim();
                    if (lane == 0) {
                        ps->type = kPassGemm;
                        ps->op = op;
                        ps->kind = kind;
                        ps->hm = hm;
                        ps->first = s0.first;
                        ps->sync = need_sync && rp == 0 && n0 == 0;
                        ps->rp = rp;
                        ps->rpn = rpn;
                        ps->np = np;
                        ps->nst = nst;
                    }
                    fill_outputs(p, ps, out_b, out_e, s0.out_off + n0, np, lane);
                    ring.publish(lane);
                    for (int si = s; si < e;) {
                        int K = 0;
                        const int sj = merged_end(p, si, e, &K);  // segments [si, sj): one T matrix
                        const SegD sg = seg_at(p, si);
                        // TMA coordinates: the segment starts at (row, col) = divmod(m_off, ld)
                        const int y0 = (int)(sg.m_off / sg.ld), x0 = (int)(sg.m_off % sg.ld);
                        const CUtensorMap* map = p.tmaps + 2 * sg.tmap + (hm ? 1 : 0);
                        const int nbox = hm ? 1 : (np + kKC - 1) / kKC;
                        int sub = si, sub_k = 0;  // input sub-segment holding column k0
                        for (int k0 = 0; k0 < K; k0 += kKC) {
                            const int kv = min(kKC, K - k0);
                            long long tw = PROF ? clock64() : 0;
                            mbar_wait(&empty[stage], sphase ^ 1u);
                            if (PROF && lane == 0) pr[0] += clock64() - tw;
                            double2* st = stages + (int64_t)stage * kStageElems;
                            double2* ti = st + kTElems;
                            // TMA boxes land whole (zero-filled past the row end); rows past kv
                            // are masked by the consumers
                            const uint32_t bytes = (uint32_t)(nbox * kKC * (hm ? kNP : kKC) + kv * rpn) * 16u;
                            if (lane == 0) {
                                s_kv[stage] = kv;  // published by the arrive (release)
                                mbar_arrive_expect_tx(&full[stage], bytes);
                            }
                            __syncwarp();
                            if (!hm) {  // T rows n0 + 16b.., columns k0..k0+16
                                if (lane < nbox)
                                    tma2d(st + lane * kKC * kLdTN, map, 2 * (x0 + k0), y0 + n0 + kKC * lane, &full[stage]);
                            } else if (lane == 0) {  // T rows k0..k0+16, columns n0..n0+80
                                tma2d(st, map, 2 * (x0 + n0), y0 + k0, &full[stage]);
                            }
                            // IN rows k0..k0+kv, possibly from several input runs (one per
                            // merged sub-segment, e.g. the u_b vectors of F_s)
                            for (int k = 0; k < kv;) {
                                while (k0 + k >= sub_k + seg_k(seg_at(p, sub))) {
                                    sub_k += seg_k(seg_at(p, sub));
                                    ++sub;
                                }
                                const SegD sb2 = seg_at(p, sub);
                                const int take = min(kv - k, sub_k + seg_k(sb2) - (k0 + k));
                                const double2* IN = (sb2.in_buf == kBufX ? p.x : p.work) +
                                                    (sb2.in_abs + (k0 + k - sub_k)) * (int64_t)R + rp;
                                if (rpn == R) {  // contiguous rows: one copy
                                    if (lane == 31) g2s(ti + k * rpn, IN, (uint32_t)(take * R) * 16u, &full[stage]);
                                } else {
                                    for (int kk = lane; kk < take; kk += 32)
                                        g2s(ti + (k + kk) * rpn, IN + (int64_t)kk * R, rpn * 16u, &full[stage]);
                                }
                                k += take;
                            }
                            if (++stage == kNST) {
                                stage = 0;
                                sphase ^= 1u;
                            }
                        }
                        si = sj;
                    }
                }
            }
            s = e;
        }
        Pass* ps = ring.claim();
        if (lane == 0) {
            ps->type = kPassEndOp;
            ps->op = op;
            ps->kind = kind;
        }
        ring.publish(lane);
        if (PROF && lane == 0) pr[2] += clock64() - t0;
    }
}

// One ring stage (KC = 16 complex inputs = two mma k-steps) of a warp's tiles.  Both k-steps'
// A fragments are loaded up front; FULL: every input of the stage is valid (no masking).
template <bool HM, bool FULL>
__device__ __forceinline__ void stage_mma(double (&acc)[2][kMaxNT][4], const double2* st,
                                          const double2* ti, int ldi, int kv, int ns, int nsplit,
                                          int ntiles, int g, int t) {
    const double2 zero = make_double2(0.0, 0.0);
    double afr[2][2][8];
    bool val[2][2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
        const int kc = ks * 8 + 2 * t;  // this lane's complex inputs kc, kc+1
        val[ks][0] = FULL || kc < kv;
        val[ks][1] = FULL || kc + 1 < kv;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const double2 z0 = val[ks][0] ? ti[kc * ldi + mt * 8] : zero;
            const double2 z1 = val[ks][1] ? ti[(kc + 1) * ldi + mt * 8] : zero;
            double* a = afr[ks][mt];
            if (!HM) {  // {re,-im; im,re}
                a[0] = z0.x; a[1] = z0.y; a[2] = -z0.y; a[3] = z0.x;
                a[4] = z1.x; a[5] = z1.y; a[6] = -z1.y; a[7] = z1.x;
            } else {  // {re,im; im,-re}
                a[0] = z0.x; a[1] = z0.y; a[2] = z0.y; a[3] = -z0.x;
                a[4] = z1.x; a[5] = z1.y; a[6] = z1.y; a[7] = -z1.x;
            }
        }
    }
    const bool two = FULL || kv > 8;
#pragma unroll
    for (int j = 0; j < kMaxNT; ++j) {
        const int nt = ns + j * nsplit;
        if (nt >= ntiles) break;
        const int n = nt * 8 + g;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            if (ks == 1 && !two) break;
            const int kc = ks * 8 + 2 * t;
            double2 b0, b1;
            if (!HM) {
                b0 = st[n * kLdTN + kc];
                b1 = st[n * kLdTN + kc + 1];
            } else {
                b0 = st[kc * kLdTH + n];
                b1 = st[(kc + 1) * kLdTH + n];
            }
            if (!val[ks][0]) b0 = zero;
            if (!val[ks][1]) b1 = zero;
            const double bfr[4] = {b0.x, b0.y, b1.x, b1.y};
            mrhs::dmma(acc[0][j], afr[ks][0], bfr);
            mrhs::dmma(acc[1][j], afr[ks][1], bfr);
        }
    }
}

template <bool PROF>
__device__ void consumer(const Params& p, double2* stages, const int* s_kv, uint64_t* full, uint64_t* empty,
                         Pass* slots, uint64_t* pfull, uint64_t* pempty, unsigned long long* pr) {
    const int ctid = threadIdx.x;  // 0 .. kCT-1
    const int lane = ctid & 31, cw = ctid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int R = p.nrhs;
    uint32_t stage = 0, sphase = 0, qphase = 0;
    int q = 0;
    const bool rec = PROF && ctid == 0;
    for (;;) {
        long long t0 = PROF ? clock64() : 0;
        mbar_wait(&pfull[q], qphase);
        const Pass* ps = slots + q;
        const int type = ps->type;
        if (rec) pr[40] += clock64() - t0;
        if (type == kPassExit) break;
        unsigned long long* pk = pr + 8 + 4 * (PROF ? ps->kind : 0);
        if (type == kPassEndOp) {
            cons_sync();  // every flush of the op issued
            if (ctid == 0) {
                const int32_t* hp = p.ops + (int64_t)ps->op * kOpFields;
                const int gb = __ldg(hp + 10), ge = __ldg(hp + 11);
                if (ge > gb)  // release cumulativity orders the CTA's flushes (bar.sync above)
                    bulk::signal_counters(p.counters, p.sigs, gb, ge);
            }
        } else if (type == kPassZero) {
            const int32_t* hp = p.ops + (int64_t)ps->op * kOpFields;
            for (int r = __ldg(hp + 6); r < __ldg(hp + 7); ++r) {
                const int64_t* rd = p.runs + (int64_t)r * kRunFields;
                if (__ldg(rd + 4) & 2) continue;
                double2* dp = p.work + __ldg(rd + 1) * (int64_t)R;
                const int64_t n = (int64_t)__ldg(rd + 2) * R;
                for (int64_t i = ctid; i < n; i += kCT) __stcg(dp + i, make_double2(0.0, 0.0));
            }
            cons_sync();
        } else if (type == kPassSum) {
            // partial-vector reduction: out[j][r] = sum_k W[k][j0 + j][r] (work, L2 reads)
            if (PROF) t0 = clock64();
            if (ps->sync) cons_sync();
            const int np = ps->np, rows = ps->s_rows;
            const int64_t stride = ps->s_ld * (int64_t)R;
            const double2* base = p.work + (ps->s_moff + ps->s_j0) * (int64_t)R;
            const int64_t tot = (int64_t)np * R;
            for (int64_t qq = ctid; qq < tot; qq += kCT) {
                const int j = (int)(qq / R), r = (int)(qq % R);
                const double2* src = base + (int64_t)j * R + r;
                double2 acc = make_double2(0.0, 0.0);
                int k = 0;
                for (; k + 8 <= rows; k += 8) {  // eight loads in flight, summed in order
                    double2 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (k + u) * stride);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        acc.x += v[u].x;
                        acc.y += v[u].y;
                    }
                }
                for (; k < rows; ++k) {
                    const double2 v = __ldcg(src + k * stride);
                    acc.x += v.x;
                    acc.y += v.y;
                }
                double2* dp = ps->out[j] + r;
                if ((ps->atom[j >> 5] >> (j & 31)) & 1u) {
                    red_add_f64(&dp->x, acc.x);
                    red_add_f64(&dp->y, acc.y);
                } else if (ps->first) {
                    __stcg(dp, acc);
                } else {
                    const double2 o = __ldcg(dp);
                    __stcg(dp, make_double2(o.x + acc.x, o.y + acc.y));
                }
            }
            if (rec) pk[3] += clock64() - t0;
        } else {  // kPassGemm
            const bool hm = ps->hm != 0;
            const int rpn = ps->rpn, rp = ps->rp, np = ps->np, nst = ps->nst;
            const int n_mg = rpn / 16;
            const int nsplit = kCW / n_mg;
            const bool active = cw < n_mg * nsplit;
            const int mg = cw % n_mg, ns = cw / n_mg;
            const int ntiles = (np + 7) >> 3;
            double acc[2][kMaxNT][4];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < kMaxNT; ++b)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[a][b][v] = 0.0;
            for (int c = 0; c < nst; ++c) {
                if (PROF) t0 = clock64();
                mbar_wait(&full[stage], sphase);
                const int kv = s_kv[stage];
                if (rec) {
                    const long long t1 = clock64();
                    pk[0] += t1 - t0;
                    t0 = t1;
                }
                if (active) {
                    const double2* st = stages + (int64_t)stage * kStageElems;
                    const double2* ti = st + kTElems + mg * 16 + g;
                    if (kv == kKC) {
                        if (hm) stage_mma<true, true>(acc, st, ti, rpn, kv, ns, nsplit, ntiles, g, t);
                        else stage_mma<false, true>(acc, st, ti, rpn, kv, ns, nsplit, ntiles, g, t);
                    } else {
                        if (hm) stage_mma<true, false>(acc, st, ti, rpn, kv, ns, nsplit, ntiles, g, t);
                        else stage_mma<false, false>(acc, st, ti, rpn, kv, ns, nsplit, ntiles, g, t);
                    }
                }
                __syncwarp();
                if (rec) pk[1] += clock64() - t0;
                if (lane == 0) mbar_arrive(&empty[stage]);
                if (++stage == kNST) {
                    stage = 0;
                    sphase ^= 1u;
                }
            }
            if (PROF) t0 = clock64();
            if (ps->sync) cons_sync();  // an earlier group's flush of these outputs is complete
            if (active) {  // flush: lane holds out[2t+e][g] for its tiles (re d=0, im d=1)
#pragma unroll
                for (int j = 0; j < kMaxNT; ++j) {
                    const int nt = ns + j * nsplit;
                    if (nt >= ntiles) break;
#pragma unroll
                    for (int ee = 0; ee < 2; ++ee) {
                        const int n = nt * 8 + 2 * t + ee;
                        if (n >= np) continue;
                        double2* base = ps->out[n] + rp + mg * 16 + g;
                        const bool at = (ps->atom[n >> 5] >> (n & 31)) & 1u;
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt) {
                            double2* dp = base + mt * 8;
                            const double re = acc[mt][j][ee], im = acc[mt][j][2 + ee];
                            if (at) {
                                red_add_f64(&dp->x, re);
                                red_add_f64(&dp->y, im);
                            } else if (ps->first) {
                                __stcg(dp, make_double2(re, im));
                            } else {
                                const double2 o = __ldcg(dp);
                                __stcg(dp, make_double2(o.x + re, o.y + im));
                            }
                        }
                    }
                }
            }
            if (rec) pk[2] += clock64() - t0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[q]);  // this warp is done with the descriptor
        if (++q == kPassSlots) {
            q = 0;
            qphase ^= 1u;
        }
    }
}

template <bool PROF>
__global__ void __launch_bounds__(kThreads, 1) uhmv_mrtc_kernel(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    double2* stages = reinterpret_cast<double2*>(smem);
    Pass* slots = reinterpret_cast<Pass*>(smem + kSmemStages);
    int* s_kv = reinterpret_cast<int*>(slots + kPassSlots);
    uint64_t* full = reinterpret_cast<uint64_t*>(s_kv + ((kNST + 1) & ~1));
    uint64_t* empty = full + kNST;
    uint64_t* pfull = empty + kNST;
    uint64_t* pempty = pfull + kPassSlots;
    int* flag = reinterpret_cast<int*>(pempty + kPassSlots);
    unsigned long long* sprof = reinterpret_cast<unsigned long long*>(flag + 2);  // 8-aligned
    if (PROF && threadIdx.x < 48) sprof[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCW);
        }
        for (int s = 0; s < kPassSlots; ++s) {
            mbar_init(&pfull[s], 1);
            mbar_init(&pempty[s], kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if ((threadIdx.x >> 5) == kCW) {
        PassRing ring{slots, pfull, pempty, 0, 0u};
        producer<PROF>(p, stages, s_kv, full, empty, ring, sprof);
    } else {
        consumer<PROF>(p, stages, s_kv, full, empty, slots, pfull, pempty, sprof);
    }
    __syncthreads();
    if (PROF && threadIdx.x < 48) p.prof[(int64_t)blockIdx.x * 64 + threadIdx.x] = sprof[threadIdx.x];
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(p.exit_count, 1u);
        flag[0] = (prev == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (flag[0]) {
        __threadfence();
        for (int i = threadIdx.x; i < p.n_counters; i += kThreads) p.counters[i] = 0u;
        if (threadIdx.x == 0) {
            *p.ticket = 0ull;
            *p.exit_count = 0u;
        }
        __threadfence();
    }
}

}  // namespace mrtc
