// uhmv_mrhs.cuh -- multi-RHS uniform-H product on FP64 tensor cores (BASELINE config 5).
//
// W = A X with X (n_in x R), R a multiple of 16 complex right-hand sides.  Same op program,
// fused ticket order and dependency counters as the single-RHS engines, but every segment is a
// small complex GEMM run on DMMA (mma.sync.aligned.m16n8k16.row.col.f64, SASS DMMA) through
// the complex -> real embedding:
//   N segment  out[n][r] += sum_k T[n][k] in[k][r]
//       D (2R' x N) += A' (2R' x 2K) * B' (2K x N):  B' column-major == the stored complex T
//       row-major read as reals (no repacking); A'[2r+d][2k+c] = {ir, -ii; ii, ir}[d][c].
//   H segment  out[j][r] += sum_k conj(T[k][j]) in[k][r]
//       B'[2k+c][j] = (c ? Ti : Tr)[k][j];   A'[2r+d][2k+c] = {ir, ii; ii, -ir}[d][c].
// Each warp owns 16 complex RHS (two 16-row m-tiles) and a block of 16 outputs (two n-tiles);
// T fragments stream from HBM, input fragments come from x / work (L2-resident), a segment
// group (consecutive segments with the same outputs) accumulates in registers and is flushed
// once (fp64 red.add into the zeroed w, or add into work outputs zeroed at op start).
//
// Fragment layouts of m16n8k16 f64 (per lane l, g = l >> 2, t = l & 3):
//   A v=0..7: m = g + 8*(v&1), k = t + 4*(v>>1)      B v=0..3: k = t + 4*v, n = g
//   D v=0..3: m = g + 8*(v>>1), n = 2*t + (v&1)

#pragma once

namespace mrhs {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kRC = 16;  // complex RHS per warp pass (two m-tiles of 16 real rows)

struct Params {
    const double2* arena;
    double2* work;  // work_len x nrhs
    const double2* x;
    double2* w;
    const int32_t* ops;
    const int64_t* runs;
    const int32_t* waits;
    const int32_t* sigs;
    const int32_t* fused_order;
    const int64_t* mr_segs;
    const int32_t* mr_ranges;
    int32_t op_count;
    int32_t nrhs;  // row stride of x / work / w in complex elements (multiple of kRC)
    uint32_t* counters;
    unsigned long long* ticket;
    uint32_t* exit_count;
    int32_t n_counters;
    unsigned long long* prof;  // diagnostics: per-CTA cycle counters (staged engine), or null
    const CUtensorMap* tmaps;  // staged engine: 2 TMA maps per leading dimension (mr_segs bits 16..)
};

__device__ __forceinline__ void dmma(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

struct Seg {
    int64_t m_off, ld;
    int rows, cols, mode, in_buf;
    int64_t in_abs;
    int out_off;
};

__device__ __forceinline__ Seg load_seg(const Params& p, int i) {
    const int64_t* d = p.mr_segs + (int64_t)i * 8;
    Seg s;
    s.m_off = __ldg(d + 0);
    s.ld = __ldg(d + 1);
    s.rows = (int)__ldg(d + 2);
    s.cols = (int)__ldg(d + 3);
    s.mode = (int)__ldg(d + 4) & 0xFF;  // low byte: mode (bit 8: first-writer flag)
    s.in_buf = (int)__ldg(d + 5);
    s.in_abs = __ldg(d + 6);
    s.out_off = (int)__ldg(d + 7);
    return s;
}

// destination of output vector position o of the op (binary search over its out runs)
__device__ __forceinline__ double2* out_ptr(const Params& p, int out_b, int out_e, int o,
                                            bool* atomic) {
    int lo = out_b, hi = out_e;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((int)__ldg(p.runs + (int64_t)mid * kRunFields + 3) <= o) lo = mid;
        else hi = mid;
    }
    const int64_t* rd = p.runs + (int64_t)lo * kRunFields;
    const int buf = (int)__ldg(rd + 0);
    *atomic = buf == kBufW;  // every w run: fp64 adds onto the zeroed W (whatever the single-RHS flags say)
    return (buf == kBufW ? p.w : p.work) + (__ldg(rd + 1) + (o - __ldg(rd + 3))) * (int64_t)p.nrhs;
}

__global__ void __launch_bounds__(kThreads) uhmv_mrhs_kernel(const Params p) {
    __shared__ int s_op;
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int R = p.nrhs;
    for (;;) {
        if (tid == 0) {
            const unsigned long long tk = atomicAdd(p.ticket, 1ull);
            s_op = (tk < (unsigned long long)p.op_count) ? __ldg(p.fused_order + tk) : -1;
        }
        __syncthreads();
        const int op = s_op;
        __syncthreads();
        if (op < 0) break;
        const int32_t* hp = p.ops + (int64_t)op * 16;
        const int out_b = __ldg(hp + 6), out_e = __ldg(hp + 7);
        const int wb = __ldg(hp + 8), we = __ldg(hp + 9);
        for (int i = wb + tid; i < we; i += kThreads) {
            const int c = __ldg(p.waits + 2 * i);
            const uint32_t need = (uint32_t)__ldg(p.waits + 2 * i + 1);
            while (ld_acquire(p.counters + c) < need) __nanosleep(20);
        }
        // zero the op's work outputs (groups add into them); w is zeroed by the launcher
        for (int r = out_b; r < out_e; ++r) {
            const int64_t* rd = p.runs + (int64_t)r * kRunFields;
            if ((int)__ldg(rd + 0) == kBufW) continue;
            double2* dp = p.work + __ldg(rd + 1) * (int64_t)R;
            const int64_t n = (int64_t)__ldg(rd + 2) * R;
            for (int64_t i = tid; i < n; i += kThreads) __stcg(dp + i, make_double2(0.0, 0.0));
        }
        __syncthreads();
        const int sb = __ldg(p.mr_ranges + 3 * op), se = __ldg(p.mr_ranges + 3 * op + 1);
        int s = sb;
        while (s < se) {
            const Seg s0 = load_seg(p, s);
            const int nout = (s0.mode == kModeN) ? s0.rows : s0.cols;
            int e = s + 1;
            while (e < se) {  // group: same outputs
                const Seg sn = load_seg(p, e);
                const int no = (sn.mode == kModeN) ? sn.rows : sn.cols;
                if (sn.mode != s0.mode || sn.out_off != s0.out_off || no != nout) break;
                ++e;
            }
            if (s0.mode == kModeS) {
                // partial-vector reduction: out[j][r] = sum_k W[k][j][r]
                const int64_t tot = (int64_t)nout * R;
                for (int64_t q = tid; q < tot; q += kThreads) {
                    const int j = (int)(q / R), r = (int)(q % R);
                    double2 acc = make_double2(0.0, 0.0);
                    for (int si = s; si < e; ++si) {
                        const Seg sg = load_seg(p, si);
                        for (int k = 0; k < sg.rows; ++k) {
                            const double2 v = __ldcg(p.work + (sg.m_off + k * sg.ld + j) * (int64_t)R + r);
                            acc.x += v.x;
                            acc.y += v.y;
                        }
                    }
                    bool at;
                    double2* dp = out_ptr(p, out_b, out_e, s0.out_off + j, &at) + r;
                    const double2 o = __ldcg(dp);
                    __stcg(dp, make_double2(o.x + acc.x, o.y + acc.y));
                }
                s = e;
                continue;
            }
            const bool hm = (s0.mode == kModeH);
            // warp work items: (RHS chunk, block of 16 outputs)
            const int n_rc = R / kRC;
            const int n_nb = (nout + 15) / 16;
            for (int item = warp; item < n_rc * n_nb; item += kWarps) {
                const int rc = item % n_rc, nb = item / n_rc;
                const int rbase = rc * kRC, nbase = nb * 16;
                double acc[2][2][4];
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 2; ++b)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[a][b][v] = 0.0;
                for (int si = s; si < e; ++si) {
                    const Seg sg = load_seg(p, si);
                    const double* T = reinterpret_cast<const double*>(p.arena + sg.m_off);
                    const double2* IN = (sg.in_buf == kBufX ? p.x : p.work) + sg.in_abs * (int64_t)R + rbase;
                    const int K2 = 2 * (hm ? sg.rows : sg.cols);
                    const int nlim = hm ? sg.cols : sg.rows;
                    for (int kb = 0; kb < K2; kb += 16) {
                        double afr[2][8], bfr[2][4];
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
                            for (int v = 0; v < 8; ++v) {
                                const int r = mt * 8 + (lane >> 3) + 4 * (v & 1);
                                const int d = g & 1;
                                const int kp = kb + t + 4 * (v >> 1);
                                const int c = kp & 1;
                                double val = 0.0;
                                if (kp < K2) {
                                    // N: {ir,-ii; ii,ir}   H: {ir,ii; ii,-ir}.  x is read-only; a
                                    // work row (R >= 16 complex, 256-B aligned) is written once per
                                    // launch before any reader passes its dependency poll, whose
                                    // ld.acquire.gpu invalidates L1
                                    const double2 z = IN[(int64_t)(kp >> 1) * R + r];
                                    val = (d ^ c) ? z.y : z.x;
                                    if (!hm && d == 0 && c == 1) val = -val;
                                    if (hm && d == 1 && c == 1) val = -val;
                                }
                                afr[mt][v] = val;
                            }
                        }
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                const int kp = kb + t + 4 * v;
                                const int n = nbase + nt * 8 + g;
                                double val = 0.0;
                                if (kp < K2 && n < nlim) {
                                    if (!hm)  // T_real[n][kp]
                                        val = __ldg(T + 2 * ((int64_t)n * sg.ld) + kp);
                                    else  // (kp&1 ? Ti : Tr)[kp>>1][n]
                                        val = __ldg(T + 2 * ((int64_t)(kp >> 1) * sg.ld + n) + (kp & 1));
                                }
                                bfr[nt][v] = val;
                            }
                        }
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                            for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt], afr[mt], bfr[nt]);
                    }
                }
                // flush the 16 x 16 complex block
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int r = mt * 8 + (lane >> 3) + 4 * (v >> 1);
                            const int d = g & 1;
                            const int n = nbase + nt * 8 + 2 * t + (v & 1);
                            if (n >= nout) continue;
                            bool at;
                            double* dp = reinterpret_cast<double*>(
                                             out_ptr(p, out_b, out_e, s0.out_off + n, &at) + rbase + r) + d;
                            if (at) {
                                red_add_f64(dp, acc[mt][nt][v]);
                            } else {
                                __stcg(dp, __ldcg(dp) + acc[mt][nt][v]);
                            }
                        }
            }
            s = e;
            __syncthreads();  // the next group may add into the same outputs
        }
        __syncthreads();
        if (tid == 0) {
            const int gb = __ldg(hp + 10), ge = __ldg(hp + 11);
            if (ge > gb) {
                __threadfence();
                for (int i = gb; i < ge; ++i) atomicAdd(p.counters + __ldg(p.sigs + i), 1u);
            }
        }
    }
    if (tid == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(p.exit_count, 1u);
        s_last = (prev == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        for (int i = tid; i < p.n_counters; i += kThreads) p.counters[i] = 0u;
        if (tid == 0) {
            *p.ticket = 0ull;
            *p.exit_count = 0u;
        }
        __threadfence();
    }
}

// FP64 tensor-core peak probe: independent DMMA chains in registers, no memory traffic.
__global__ void __launch_bounds__(128) dmma_peak_kernel(int iters, double* sink) {
    double a[8], b[4], c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0}, c2[4] = {0, 0, 0, 0},
                      c3[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (blockIdx.x + i);
    for (int it = 0; it < iters; ++it) {
        dmma(c0, a, b);
        dmma(c1, a, b);
        dmma(c2, a, b);
        dmma(c3, a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c0[i] + c1[i] + c2[i] + c3[i];
    if (s == 12345.678) *sink = s;
}

}  // namespace mrhs
