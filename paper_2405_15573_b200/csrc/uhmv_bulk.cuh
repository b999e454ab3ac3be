// uhmv_bulk.cuh -- warp-specialised bulk-copy engine for the uniform-H op programs (sm_100a).
//
// Same op semantics as the register kernel in uhmv.cu, different data path: every arena slab
// an op streams is cut on the host into "pieces" (row ranges, packer._pieces) packed into
// 16-KiB shared-memory stages.  One producer lane per CTA claims ops from the fused ticket
// order, publishes them to the consumer warps through an op-slot ring, and streams their
// pieces with cp.async.bulk (the TMA engine, SASS UBLKCP) into an mbarrier-guarded stage
// ring -- WITHOUT waiting for the op's dependencies: arena data never depends on anything, so
// HBM streaming runs ahead across ops while the consumers wait for y/u/z.  Four consumer warps
// gather the op's work-buffer inputs, compute the GEMV pieces out of shared memory, and write
// the op's outputs.  Bytes in flight per SM are set by the ring (stages x 16 KiB x CTAs/SM),
// not by registers or warp count.
//
//   N piece: out[r] += sum_j T[r,j] in[j]     8 lanes per row (128 B of smem per row-group
//            load, conflict-free), rows owned by row-group (out_off+r) % 16 -> no atomics.
//   H piece: out[j] += sum_r conj(T[r,j]) in[r]   column j owned by thread (out_off+j) % 128.
//   S piece: out[j] += sum_r W[r,j] read directly (ld.cg) from the work buffer (partials).
// "in" is the op's shared-memory gather of y/u/z, or x read in place (ld.global.nc, L1/L2).

#pragma once

namespace bulk {

constexpr int kConsumerWarps = 4;
constexpr int kConsumers = kConsumerWarps * 32;  // 128
constexpr int kThreads = kConsumers + 32;        // + one producer warp
constexpr int kStageElems = 1024;                // = packer.STAGE_ELEMS (16 KiB of complex128)
constexpr int kStageBytes = kStageElems * 16;
constexpr int kOpSlots = 4;
constexpr int kLanesPerRow = 8;
constexpr int kRowGroups = kConsumers / kLanesPerRow;  // 16
constexpr int kPieceFields = 8;
constexpr int64_t kPiBegin = 1ll << 24, kPiEnd = 1ll << 25, kPiDirect = 1ll << 26,
                  kPiXGlobal = 1ll << 27;

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
    uint32_t* counters;
    unsigned long long* ticket;
    uint32_t* exit_count;
    int32_t n_counters;
    int32_t xin_max;
    int32_t out_max;
    int32_t skip_waits;  // phased launches: dependencies are ordered by the stream
    unsigned long long* prof;  // optional [grid][8] cycle counters (UHMV_PROFILE), else null
};

// prof slots: 0 consumer wait for data, 1 consumer dependency wait, 2 consumer compute,
// 3 consumer op overhead (gather/scatter/barriers), 4 producer wait for a free stage,
// 5 producer wait for an op slot, 6 ops, 7 pieces

constexpr int kDescCache = 64;  // piece descriptors cached in shared memory per batch
constexpr int kSlots = 8;       // register accumulator slots per thread (segment groups)

struct Layout {
    int stage_off, xin_off, out_off, desc_off, bar_off, slot_off, total;
};

__host__ __device__ inline Layout layout(int nstage, int xin_max, int out_max) {
    Layout L;
    L.stage_off = 0;
    L.xin_off = nstage * kStageBytes;
    L.out_off = L.xin_off + ((xin_max * 16 + 127) & ~127);
    L.desc_off = L.out_off + ((out_max * 16 + 127) & ~127);
    L.bar_off = L.desc_off + kDescCache * kPieceFields * 8;
    L.slot_off = L.bar_off + (2 * nstage + 2 * kOpSlots) * 8;
    L.total = L.slot_off + 16 * 4;
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
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(su32(b)),
        "r"(parity)
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
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// Whole producer warp runs this loop in lock-step; lane 0 issues barriers and copies, the 32
// lanes fetch piece descriptors 32 at a time (one coalesced round trip per batch instead of one
// per piece), and the next ticket is claimed while the current op's pieces are issued.
__device__ __forceinline__ void producer(const Params& p, unsigned char* stages, uint64_t* full,
                                         uint64_t* empty, uint64_t* opfull, uint64_t* opempty,
                                         int* slots) {
    const int lane = threadIdx.x & 31;
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int stage = 0;
    uint32_t sphase = 0;
    int q = 0;
    uint32_t qphase = 0;
    unsigned long long c_empty = 0, c_slot = 0;
    const bool prof = p.prof != nullptr && lane == 0;
    unsigned long long t_next = 0;
    if (lane == 0) t_next = atomicAdd(p.ticket, 1ull);
    t_next = __shfl_sync(0xffffffffu, t_next, 0);
    for (;;) {
        const int op = (t_next < (unsigned long long)p.op_count) ? __ldg(p.fused_order + t_next) : -1;
        int pc_b = 0, pc_e = 0;
        if (op >= 0) {
            pc_b = __ldg(p.ops + (int64_t)op * 16 + 13);
            pc_e = __ldg(p.ops + (int64_t)op * 16 + 14);
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(p.ticket, 1ull);  // next op, overlapped with this one
            t_next = __shfl_sync(0xffffffffu, t, 0);
        }
        long long tq = prof ? clock64() : 0;
        mbar_wait(&opempty[q], qphase ^ 1u);
        if (prof) c_slot += clock64() - tq;
        if (lane == 0) {
            slots[q] = op;
            mbar_arrive(&opfull[q]);
        }
        if (++q == kOpSlots) {
            q = 0;
            qphase ^= 1u;
        }
        if (op < 0) {
            if (prof) {
                p.prof[(size_t)blockIdx.x * 8 + 4] = c_empty;
                p.prof[(size_t)blockIdx.x * 8 + 5] = c_slot;
            }
            break;
        }
        for (int base = pc_b; base < pc_e; base += 32) {
            const int nb = min(32, pc_e - base);
            int64_t f0 = 0, f1 = 0, f7 = kPiDirect;
            int rc = 0;
            if (lane < nb) {
                const int64_t* d = p.pieces + (int64_t)(base + lane) * kPieceFields;
                f0 = __ldg(d + 0);
                f1 = __ldg(d + 1);
                rc = (int)((__ldg(d + 2) << 16) | __ldg(d + 3));  // rows <= 2^15, cols <= 2^16
                f7 = __ldg(d + 7);
            }
            for (int k = 0; k < nb; ++k) {
                const int64_t info = __shfl_sync(0xffffffffu, f7, k);
                if (info & kPiDirect) continue;
                const int64_t m_off = __shfl_sync(0xffffffffu, f0, k);
                const int64_t ld = __shfl_sync(0xffffffffu, f1, k);
                const int rcv = __shfl_sync(0xffffffffu, rc, k);
                const int rows = rcv >> 16, cols = rcv & 0xFFFF;
                if (info & kPiBegin) {
                    const long long te = prof ? clock64() : 0;
                    mbar_wait(&empty[stage], sphase ^ 1u);
                    if (prof) c_empty += clock64() - te;
                    if (lane == 0)
                        mbar_arrive_expect_tx(&full[stage], (uint32_t)(((info >> 32) & 0xFFFFFF) * 16));
                }
                if (lane == 0) {
                    unsigned char* dst =
                        stages + (size_t)stage * kStageBytes + (size_t)(info & 0xFFFFFF) * 16;
                    const double2* src = p.arena + m_off;
                    if (ld == cols) {
                        bulk_g2s(dst, src, (uint32_t)rows * cols * 16, &full[stage], policy);
                    } else {
                        for (int r = 0; r < rows; ++r)
                            bulk_g2s(dst + (size_t)r * cols * 16, src + (int64_t)r * ld,
                                     (uint32_t)cols * 16, &full[stage], policy);
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

__device__ __forceinline__ void consumer(const Params& p, unsigned char* stages, double2* xin,
                                         double2* outv, int64_t* pdesc, uint64_t* full,
                                         uint64_t* empty, uint64_t* opfull, uint64_t* opempty,
                                         int* slots) {
    const int tid = threadIdx.x;  // 0..127
    const int lane = tid & 31;
    const int g = tid & (kLanesPerRow - 1);
    const int rg = tid / kLanesPerRow;
    const unsigned gmask = 0xffu << (lane & ~(kLanesPerRow - 1));
    int stage = 0;
    uint32_t sphase = 0;
    int q = 0;
    uint32_t qphase = 0;
    const bool prof = p.prof != nullptr && tid == 0;
    unsigned long long c_data = 0, c_dep = 0, c_comp = 0, c_ovh = 0, n_ops = 0, n_pcs = 0;
    for (;;) {
        long long t0 = prof ? clock64() : 0;
        mbar_wait(&opfull[q], qphase);
        const int op = slots[q];
        __syncwarp();
        if (lane == 0) mbar_arrive(&opempty[q]);
        if (++q == kOpSlots) {
            q = 0;
            qphase ^= 1u;
        }
        if (op < 0) {
            if (prof) {
                unsigned long long* pr = p.prof + (size_t)blockIdx.x * 8;
                pr[0] = c_data;
                pr[1] = c_dep;
                pr[2] = c_comp;
                pr[3] = c_ovh;
                pr[6] = n_ops;
                pr[7] = n_pcs;
            }
            break;
        }
        const int32_t* hp = p.ops + (int64_t)op * 16;
        const int n_out = __ldg(hp + 1);
        const int in_b = __ldg(hp + 2), in_e = __ldg(hp + 3);
        const int out_b = __ldg(hp + 6), out_e = __ldg(hp + 7);
        const int pc_b = __ldg(hp + 13), pc_e = __ldg(hp + 14);
        if (prof) {
            const long long t1 = clock64();
            c_ovh += t1 - t0;
            t0 = t1;
            ++n_ops;
        }
        if (tid == 0 && !p.skip_waits) {
            const int wb = __ldg(hp + 8), we = __ldg(hp + 9);
            for (int i = wb; i < we; ++i) {
                const int c = __ldg(p.waits + 2 * i);
                const uint32_t need = (uint32_t)__ldg(p.waits + 2 * i + 1);
                while (ld_acquire(p.counters + c) < need) __nanosleep(20);
            }
        }
        consumer_sync();
        if (prof) {
            const long long t1 = clock64();
            c_dep += t1 - t0;
            t0 = t1;
        }
        // gather the op's input vector: x windows (read-only) and y/u/z (coherent ld.cg)
        for (int r = in_b; r < in_e; ++r) {
            const int64_t* rd = p.runs + (int64_t)r * kRunFields;
            const int buf = (int)__ldg(rd + 0);
            const int64_t off = __ldg(rd + 1);
            const int len = (int)__ldg(rd + 2);
            const int dst = (int)__ldg(rd + 3);
            if (buf == kBufX) {
                for (int i = tid; i < len; i += kConsumers) xin[dst + i] = __ldg(p.x + off + i);
            } else {
                for (int i = tid; i < len; i += kConsumers) xin[dst + i] = __ldcg(p.work + off + i);
            }
        }
        for (int i = tid; i < n_out; i += kConsumers) outv[i] = make_double2(0.0, 0.0);
        {
            const int nb = min(kDescCache, pc_e - pc_b) * kPieceFields;
            for (int i = tid; i < nb; i += kConsumers) pdesc[i] = __ldg(p.pieces + (int64_t)pc_b * kPieceFields + i);
        }
        consumer_sync();
        // Segment groups accumulate in registers across all their pieces and are reduced once:
        //   N group (all N pieces of the op): output row o is owned by row-group o % 16, register
        //     slot o / 16 (n_out <= 128), partial over the lane's columns j = g (mod 8);
        //   H/S group (pieces of one segment): output column j owned by lane group (j mod nJ),
        //     slot = j / nJ, partial over the lane's rows r = pp (mod P).
        double accr[kSlots], acci[kSlots];
#pragma unroll
        for (int k = 0; k < kSlots; ++k) accr[k] = acci[k] = 0.0;
        const bool nreg = n_out <= kSlots * kRowGroups;
        int g_mode = -1, g_out = 0, g_cols = 0;
        auto flush = [&]() {
            if (g_mode == kModeN) {
                if (nreg) {
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
            } else if (g_mode >= 0) {
                const int P = g_cols <= 32 ? 4 : (g_cols <= 64 ? 2 : 1);
                const int nJ = kConsumers / P;
                const int pp = tid % P;
                int j0 = (tid / P - (g_out % nJ)) % nJ;
                if (j0 < 0) j0 += nJ;
#pragma unroll
                for (int k = 0; k < kSlots; ++k) {
                    if (k * nJ >= g_cols) break;
                    double ar = accr[k], ai = acci[k];
                    for (int o = 1; o < P; o <<= 1) {
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
        for (int pc = pc_b; pc < pc_e; ++pc) {
            const int slot = (pc - pc_b) & (kDescCache - 1);
            if (slot == 0 && pc > pc_b) {  // refill the descriptor cache (ops with > 64 pieces)
                consumer_sync();
                const int nb = min(kDescCache, pc_e - pc) * kPieceFields;
                for (int i = tid; i < nb; i += kConsumers) pdesc[i] = __ldg(p.pieces + (int64_t)pc * kPieceFields + i);
                consumer_sync();
            }
            const int64_t* d = pdesc + slot * kPieceFields;
            const int64_t info = d[7];
            const int rows = (int)d[2];
            const int cols = (int)d[3];
            const int mode = (int)d[4];
            const int in_off = (int)d[5];
            const int out_off = (int)d[6];
            const bool direct = (info & kPiDirect) != 0;
            // group change?
            if (mode == kModeN ? (g_mode != kModeN)
                               : (g_mode != mode || g_out != out_off || g_cols != cols)) {
                const bool to_h = (g_mode == kModeN) && mode != kModeN;
                flush();
                if (to_h) consumer_sync();  // N owners and H owners differ: order their outv adds
                g_mode = mode;
                g_out = out_off;
                g_cols = cols;
            }
            const double2* tile = nullptr;
            if (prof) {
                const long long t1 = clock64();
                c_ovh += t1 - t0;
                t0 = t1;
                ++n_pcs;
            }
            if (!direct) {
                if (info & kPiBegin) mbar_wait(&full[stage], sphase);
                if (prof) {
                    const long long t1 = clock64();
                    c_data += t1 - t0;
                    t0 = t1;
                }
                tile = reinterpret_cast<const double2*>(stages + (size_t)stage * kStageBytes) +
                       (info & 0xFFFFFF);
            }
            if (mode == kModeN) {
                const double2* xv = xin + in_off;
                int r0 = (rg - (out_off % kRowGroups)) % kRowGroups;
                if (r0 < 0) r0 += kRowGroups;
                for (int r = r0; r < rows; r += kRowGroups) {
                    const double2* T = tile + r * cols;
                    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
                    int j = g;
                    for (; j + kLanesPerRow < cols; j += 2 * kLanesPerRow) {  // two chains
                        cmac(ar, ai, T[j], xv[j]);
                        cmac(br, bi, T[j + kLanesPerRow], xv[j + kLanesPerRow]);
                    }
                    if (j < cols) cmac(ar, ai, T[j], xv[j]);
                    ar += br;
                    ai += bi;
                    const int o = out_off + r;
                    if (nreg) {
                        const int k = o / kRowGroups;
#pragma unroll
                        for (int q = 0; q < kSlots; ++q)
                            if (q == k) {
                                accr[q] += ar;
                                acci[q] += ai;
                            }
                    } else {  // wide N op: reduce and add per row
#pragma unroll
                        for (int s2 = 1; s2 < kLanesPerRow; s2 <<= 1) {
                            ar += __shfl_xor_sync(gmask, ar, s2);
                            ai += __shfl_xor_sync(gmask, ai, s2);
                        }
                        if (g == 0) {
                            double2 v = outv[o];
                            v.x += ar;
                            v.y += ai;
                            outv[o] = v;
                        }
                    }
                }
            } else {
                const int P = cols <= 32 ? 4 : (cols <= 64 ? 2 : 1);
                const int nJ = kConsumers / P;
                const int pp = tid % P;
                int j0 = (tid / P - (out_off % nJ)) % nJ;
                if (j0 < 0) j0 += nJ;
#pragma unroll
                for (int k = 0; k < kSlots; ++k) {
                    if (k * nJ >= cols) break;
                    const int j = j0 + k * nJ;
                    if (j >= cols) continue;
                    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
                    if (mode == kModeS) {
                        const int64_t ld = d[1];
                        const double2* W = p.work + d[0] + j;
#pragma unroll 4
                        for (int r = pp; r < rows; r += P) {
                            const double2 m = __ldcg(W + (int64_t)r * ld);
                            ar += m.x;
                            ai += m.y;
                        }
                    } else {
                        const double2* xv = xin + in_off;
                        int r = pp;
                        for (; r + P < rows; r += 2 * P) {  // two independent chains
                            cmac_conj(ar, ai, tile[r * cols + j], xv[r]);
                            cmac_conj(br, bi, tile[(r + P) * cols + j], xv[r + P]);
                        }
                        if (r < rows) cmac_conj(ar, ai, tile[r * cols + j], xv[r]);
                    }
                    accr[k] += ar + br;
                    acci[k] += ai + bi;
                }
            }
            if (prof) {
                const long long t1 = clock64();
                c_comp += t1 - t0;
                t0 = t1;
            }
            if (!direct && (info & kPiEnd)) {
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
        for (int r = out_b; r < out_e; ++r) {
            const int64_t* rd = p.runs + (int64_t)r * kRunFields;
            const int buf = (int)__ldg(rd + 0);
            const int64_t off = __ldg(rd + 1);
            const int len = (int)__ldg(rd + 2);
            const int dst = (int)__ldg(rd + 3);
            const int flags = (int)__ldg(rd + 4);
            const int add = flags & 1;
            double2* dp = (buf == kBufW ? p.w : p.work) + off;
            if (flags & 2) {  // fp64 red.add into the pre-zeroed output (<= 2 addends per entry)
                for (int i = tid; i < len; i += kConsumers) {
                    const double2 v = outv[dst + i];
                    atomicAdd(&dp[i].x, v.x);
                    atomicAdd(&dp[i].y, v.y);
                }
                continue;
            }
            for (int i = tid; i < len; i += kConsumers) {
                double2 v = outv[dst + i];
                if (add) {
                    const double2 o = __ldcg(dp + i);
                    v.x += o.x;
                    v.y += o.y;
                }
                __stcg(dp + i, v);
            }
        }
        if (prof) c_ovh += clock64() - t0;
        if (!p.skip_waits) {
            consumer_sync();
            if (tid == 0) {
                const int sb = __ldg(hp + 10), se = __ldg(hp + 11);
                if (se > sb) {
                    __threadfence();
                    for (int i = sb; i < se; ++i) atomicAdd(p.counters + __ldg(p.sigs + i), 1u);
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) uhmv_bulk_kernel(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const Layout L = layout(p.nstage, p.xin_max, p.out_max);
    unsigned char* stages = smem + L.stage_off;
    double2* xin = reinterpret_cast<double2*>(smem + L.xin_off);
    double2* outv = reinterpret_cast<double2*>(smem + L.out_off);
    int64_t* pdesc = reinterpret_cast<int64_t*>(smem + L.desc_off);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + p.nstage;
    uint64_t* opfull = empty + p.nstage;
    uint64_t* opempty = opfull + kOpSlots;
    int* slots = reinterpret_cast<int*>(smem + L.slot_off);
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
        producer(p, stages, full, empty, opfull, opempty, slots);
    } else {
        consumer(p, stages, xin, outv, pdesc, full, empty, opfull, opempty, slots);
    }
    __syncthreads();
    // self-reset: the last CTA out zeroes the counters and the ticket for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(p.exit_count, 1u);
        slots[8] = (prev == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (slots[8]) {
        __threadfence();
        for (int i = threadIdx.x; i < p.n_counters; i += kThreads) p.counters[i] = 0u;
        if (threadIdx.x == 0) {
            *p.ticket = 0ull;
            *p.exit_count = 0u;
        }
        __threadfence();
    }
}

}  // namespace bulk
