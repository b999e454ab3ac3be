// uhmv.cu -- sm_100a kernels + C ABI for the uniform-H matrix-vector product.
//
// One kernel body executes "ops" of a packed program (paper_2405_15573_b200/packer.py):
//   gather input runs -> shared-memory vector xin
//   sum of GEMV segments streamed from HBM (complex128, 16 B per lane per load)
//   scatter the shared-memory output vector (store or add)
// This replaces the dict walk and NumPy GEMVs of matvec_uh
// (/root/reference/pkg/src/uhm_kit/uniform.py:509-556):
//   phase 1 V_t^H x|_t  ........ P1 ops (H segments) + RED ops (S segments)
//   stage_b = s_y^H pre ........ U ops (H segments over the concatenated s_y of a cluster)
//   acc_s = sum s_x stage ...... Z ops (one N segment over the concatenated coupling row X_s)
//   w|_s += U_s acc ............ FAR ops (N segments, owned output rows, no atomics)
//   dense w|_r += D v|_c ....... NEAR ops (N segments; adjoint: H segments)
//
// Thread mapping (128 threads = 4 warps = 16 row-groups of 8 lanes): a row-group streams one
// matrix row at a time, its 8 lanes covering 8 consecutive complex128 (128 B, one L2 line) per
// load, so every warp-wide load instruction moves 4 fully used 128-B lines.
//   N segment: out[r] = sum_j M[r,j] xin[j]  -- row r owned by row-group (out_off+r) % 16,
//              8-lane shuffle reduction, owner writes the shared-memory output: no atomics.
//   H segment: out[j] = sum_r conj(M[r,j]) xin[r] -- lane accumulators per column j = g+8k,
//              reduced over row-groups with shuffles + a fixed-order cross-warp sum
//              (deterministic, bit-reproducible).
//   S segment: out[j] = sum_r M[r,j] (partial-vector reduction, coherent ld.cg loads).
//
// Modes: PHASED = one launch per phase (one CTA per op); FUSED = one persistent launch where
// CTAs claim ops from a ticket counter in a topological order and spin on per-op dependency
// counters (ld.acquire.gpu) -- the nearfield ops fill the dependency bubbles of the farfield
// chain.  Waits only target ops with a smaller ticket, which were claimed by running CTAs, so
// progress does not depend on co-residency.  The last CTA to exit resets all counters, so the
// launch is self-cleaning and CUDA-graph capturable.

#include <cuda.h>  // CUtensorMap (TMA descriptors of the multi-RHS engine)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/uhmv.h"

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kLanesPerRow = 8;
constexpr int kRowGroups = kThreads / kLanesPerRow;  // 16
constexpr int kHAcc = 4;                             // H/S accumulators per lane
constexpr int kHColsMax = kHAcc * kLanesPerRow;      // 32 (= packer.HCOLS_MAX)

constexpr int kModeN = 0, kModeH = 1, kModeS = 2;
constexpr int kModeNW = 3;  // bulk pieces: N rows of a wide-row op, one warp per row (packer.MODE_NW)
constexpr int kBufArena = 0, kBufWork = 1, kBufX = 2, kBufW = 3;
constexpr int kOpFields = 16, kSegFields = 8, kRunFields = 5;

struct ExecParams {
    const double2* arena;
    double2* work;
    const double2* x;
    double2* w;
    const int32_t* ops;
    const int64_t* segs;
    const int64_t* runs;
    const int32_t* waits;
    const int32_t* sigs;
    const int32_t* fused_order;
    int32_t op_begin;
    int32_t op_count;
    uint32_t* counters;
    unsigned long long* ticket;
    uint32_t* exit_count;
    int32_t n_counters;
    int32_t in_max;
    int32_t out_max;
};

__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p));
    return r;
}

// fp64 reduction into global memory without a returned value: one RED.E.ADD.F64 (the generic
// atomicAdd(double*) also emits a shared-memory CAS loop behind an address-space test)
__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "d"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// acc += m * x
__device__ __forceinline__ void cmac(double& ar, double& ai, const double2 m, const double2 x) {
    ar = fma(m.x, x.x, ar);
    ar = fma(-m.y, x.y, ar);
    ai = fma(m.x, x.y, ai);
    ai = fma(m.y, x.x, ai);
}

// acc += conj(m) * x
__device__ __forceinline__ void cmac_conj(double& ar, double& ai, const double2 m, const double2 x) {
    ar = fma(m.x, x.x, ar);
    ar = fma(m.y, x.y, ar);
    ai = fma(m.x, x.y, ai);
    ai = fma(-m.y, x.x, ai);
}

struct SegDesc {
    int64_t m_off;
    int32_t buf, rows, cols, ld, mode, in_off, out_off;
};

__device__ __forceinline__ SegDesc load_seg(const int64_t* segs, int s) {
    const int64_t* d = segs + (int64_t)s * kSegFields;
    SegDesc r;
    r.m_off = __ldg(d + 0);
    r.buf = (int32_t)__ldg(d + 1);
    r.rows = (int32_t)__ldg(d + 2);
    r.cols = (int32_t)__ldg(d + 3);
    r.ld = (int32_t)__ldg(d + 4);
    r.mode = (int32_t)__ldg(d + 5);
    r.in_off = (int32_t)__ldg(d + 6);
    r.out_off = (int32_t)__ldg(d + 7);
    return r;
}

// ---- N group: consecutive N segments sharing (out_off, rows) ------------------------------
__device__ __forceinline__ void run_ngroup(const ExecParams& p, int s_begin, int s_end, int rows,
                                           int out_off, const double2* xin, double2* outv) {
    const int tid = threadIdx.x;
    const int g = tid & (kLanesPerRow - 1);
    const int rg = tid / kLanesPerRow;
    const unsigned gmask = 0xffu << ((tid & 31) & ~(kLanesPerRow - 1));
    int r0 = (rg - (out_off % kRowGroups)) % kRowGroups;
    if (r0 < 0) r0 += kRowGroups;
    for (int r = r0; r < rows; r += kRowGroups) {
        double ar = 0.0, ai = 0.0;
        for (int s = s_begin; s < s_end; ++s) {
            const SegDesc d = load_seg(p.segs, s);
            const double2* M = p.arena + d.m_off + (int64_t)r * d.ld;
            const double2* xv = xin + d.in_off;
            const int cols = d.cols;
            int j = g;
            for (; j + 3 * kLanesPerRow < cols; j += 4 * kLanesPerRow) {
                const double2 m0 = ld_stream(M + j);
                const double2 m1 = ld_stream(M + j + kLanesPerRow);
                const double2 m2 = ld_stream(M + j + 2 * kLanesPerRow);
                const double2 m3 = ld_stream(M + j + 3 * kLanesPerRow);
                cmac(ar, ai, m0, xv[j]);
                cmac(ar, ai, m1, xv[j + kLanesPerRow]);
                cmac(ar, ai, m2, xv[j + 2 * kLanesPerRow]);
                cmac(ar, ai, m3, xv[j + 3 * kLanesPerRow]);
            }
            for (; j < cols; j += kLanesPerRow) cmac(ar, ai, ld_stream(M + j), xv[j]);
        }
#pragma unroll
        for (int o = 1; o < kLanesPerRow; o <<= 1) {
            ar += __shfl_xor_sync(gmask, ar, o);
            ai += __shfl_xor_sync(gmask, ai, o);
        }
        if (g == 0) {
            double2 v = outv[out_off + r];
            v.x += ar;
            v.y += ai;
            outv[out_off + r] = v;
        }
    }
}

// ---- H / S group: consecutive segments sharing (mode, out_off, cols), cols <= kHColsMax ----
template <int MODE>
__device__ __forceinline__ void run_hgroup(const ExecParams& p, int s_begin, int s_end, int cols,
                                           int out_off, const double2* xin, double2* outv,
                                           double2* red) {
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int g = tid & (kLanesPerRow - 1);
    const int rg = tid / kLanesPerRow;
    double ar[kHAcc], ai[kHAcc];
#pragma unroll
    for (int k = 0; k < kHAcc; ++k) ar[k] = ai[k] = 0.0;
    for (int s = s_begin; s < s_end; ++s) {
        const SegDesc d = load_seg(p.segs, s);
        const double2* base = (MODE == kModeS) ? p.work : p.arena;
        for (int r = rg; r < d.rows; r += kRowGroups) {
            const double2* M = base + d.m_off + (int64_t)r * d.ld;
            double2 m[kHAcc];
#pragma unroll
            for (int k = 0; k < kHAcc; ++k) {
                const int j = g + k * kLanesPerRow;
                if (j < cols) {
                    m[k] = (MODE == kModeS) ? __ldcg(M + j) : ld_stream(M + j);
                } else {
                    m[k] = make_double2(0.0, 0.0);
                }
            }
            if (MODE == kModeS) {
#pragma unroll
                for (int k = 0; k < kHAcc; ++k) {
                    ar[k] += m[k].x;
                    ai[k] += m[k].y;
                }
            } else {
                const double2 xv = xin[d.in_off + r];
#pragma unroll
                for (int k = 0; k < kHAcc; ++k) cmac_conj(ar[k], ai[k], m[k], xv);
            }
        }
    }
    // reduce over the 4 row-groups of the warp (lanes g, g+8, g+16, g+24)
#pragma unroll
    for (int k = 0; k < kHAcc; ++k) {
        ar[k] += __shfl_xor_sync(0xffffffffu, ar[k], 8);
        ai[k] += __shfl_xor_sync(0xffffffffu, ai[k], 8);
        ar[k] += __shfl_xor_sync(0xffffffffu, ar[k], 16);
        ai[k] += __shfl_xor_sync(0xffffffffu, ai[k], 16);
    }
    if (lane < kLanesPerRow) {
#pragma unroll
        for (int k = 0; k < kHAcc; ++k) {
            const int j = g + k * kLanesPerRow;
            if (j < cols) red[warp * kHColsMax + j] = make_double2(ar[k], ai[k]);
        }
    }
    __syncthreads();
    for (int j = tid; j < cols; j += kThreads) {
        double2 acc = outv[out_off + j];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const double2 v = red[w * kHColsMax + j];
            acc.x += v.x;
            acc.y += v.y;
        }
        outv[out_off + j] = acc;
    }
    __syncthreads();
}

template <bool FUSED>
__device__ void run_op(const ExecParams& p, int op, double2* xin, double2* outv, double2* red,
                       int* hdr) {
    const int tid = threadIdx.x;
    if (tid < kOpFields) hdr[tid] = __ldg(p.ops + (int64_t)op * kOpFields + tid);
    __syncthreads();
    const int n_out = hdr[1];
    const int in_b = hdr[2], in_e = hdr[3];
    const int seg_b = hdr[4], seg_e = hdr[5];
    const int out_b = hdr[6], out_e = hdr[7];
    if (FUSED) {
        if (tid == 0) {
            const int wb = hdr[8], we = hdr[9];
            for (int i = wb; i < we; ++i) {
                const int c = __ldg(p.waits + 2 * i);
                const uint32_t need = (uint32_t)__ldg(p.waits + 2 * i + 1);
                while (ld_acquire(p.counters + c) < need) __nanosleep(32);
            }
        }
        __syncthreads();
    }
    // gather the op's input vector into shared memory
    for (int r = in_b; r < in_e; ++r) {
        const int64_t* rd = p.runs + (int64_t)r * kRunFields;
        const int buf = (int)__ldg(rd + 0);
        const int64_t off = __ldg(rd + 1);
        const int len = (int)__ldg(rd + 2);
        const int dst = (int)__ldg(rd + 3);
        if (buf == kBufX) {
            for (int i = tid; i < len; i += kThreads) xin[dst + i] = __ldg(p.x + off + i);
        } else {
            for (int i = tid; i < len; i += kThreads) xin[dst + i] = __ldcg(p.work + off + i);
        }
    }
    for (int i = tid; i < n_out; i += kThreads) outv[i] = make_double2(0.0, 0.0);
    __syncthreads();

    int s = seg_b;
    while (s < seg_e) {
        const SegDesc d = load_seg(p.segs, s);
        int e = s + 1;
        if (d.mode == kModeN) {
            while (e < seg_e) {
                const SegDesc n = load_seg(p.segs, e);
                if (n.mode != kModeN || n.out_off != d.out_off || n.rows != d.rows) break;
                ++e;
            }
            run_ngroup(p, s, e, d.rows, d.out_off, xin, outv);
        } else {
            while (e < seg_e) {
                const SegDesc n = load_seg(p.segs, e);
                if (n.mode != d.mode || n.out_off != d.out_off || n.cols != d.cols) break;
                ++e;
            }
            // N groups precede H/S groups (packer order); the barrier inside run_hgroup orders
            // the owner-written N rows before the cross-warp sums touch the output.
            if (d.mode == kModeH)
                run_hgroup<kModeH>(p, s, e, d.cols, d.out_off, xin, outv, red);
            else
                run_hgroup<kModeS>(p, s, e, d.cols, d.out_off, xin, outv, red);
        }
        s = e;
    }
    __syncthreads();
    // scatter the output vector
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
            for (int i = tid; i < len; i += kThreads) {
                const double2 v = outv[dst + i];
                red_add_f64(&dp[i].x, v.x);
                red_add_f64(&dp[i].y, v.y);
            }
            continue;
        }
        for (int i = tid; i < len; i += kThreads) {
            double2 v = outv[dst + i];
            if (add) {
                const double2 o = __ldcg(dp + i);
                v.x += o.x;
                v.y += o.y;
            }
            __stcg(dp + i, v);
        }
    }
    if (FUSED) {
        __syncthreads();
        if (tid == 0) {
            const int sb = hdr[10], se = hdr[11];
            if (se > sb) {
                __threadfence();
                for (int i = sb; i < se; ++i) atomicAdd(p.counters + __ldg(p.sigs + i), 1u);
            }
        }
    }
    __syncthreads();
}

}  // namespace

#include "uhmv_bulk.cuh"
#include "uhmv_mrhs.cuh"
#include "uhmv_mrtc.cuh"

namespace {

struct SmemLayout {
    int xin_off, out_off, red_off, hdr_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(int in_max, int out_max) {
    SmemLayout L;
    L.xin_off = 0;
    L.out_off = L.xin_off + in_max * 16;
    L.red_off = L.out_off + out_max * 16;
    L.hdr_off = L.red_off + kWarps * kHColsMax * 16;
    L.total = L.hdr_off + (kOpFields + 4) * 4;
    return L;
}

__global__ void __launch_bounds__(kThreads) uhmv_phase_kernel(const ExecParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLayout L = smem_layout(p.in_max, p.out_max);
    double2* xin = reinterpret_cast<double2*>(smem + L.xin_off);
    double2* outv = reinterpret_cast<double2*>(smem + L.out_off);
    double2* red = reinterpret_cast<double2*>(smem + L.red_off);
    int* hdr = reinterpret_cast<int*>(smem + L.hdr_off);
    run_op<false>(p, p.op_begin + (int)blockIdx.x, xin, outv, red, hdr);
}

__global__ void __launch_bounds__(kThreads) uhmv_fused_kernel(const ExecParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLayout L = smem_layout(p.in_max, p.out_max);
    double2* xin = reinterpret_cast<double2*>(smem + L.xin_off);
    double2* outv = reinterpret_cast<double2*>(smem + L.out_off);
    double2* red = reinterpret_cast<double2*>(smem + L.red_off);
    int* hdr = reinterpret_cast<int*>(smem + L.hdr_off);
    int* slot = hdr + kOpFields;
    for (;;) {
        if (threadIdx.x == 0) {
            const unsigned long long t = atomicAdd(p.ticket, 1ull);
            slot[0] = (t < (unsigned long long)p.op_count) ? __ldg(p.fused_order + t) : -1;
        }
        __syncthreads();
        const int op = slot[0];
        __syncthreads();
        if (op < 0) break;
        run_op<true>(p, op, xin, outv, red, hdr);
    }
    // self-reset: the last CTA out zeroes the counters for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(p.exit_count, 1u);
        slot[1] = (prev == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (slot[1]) {
        __threadfence();
        for (int i = threadIdx.x; i < p.n_counters; i += kThreads) p.counters[i] = 0u;
        if (threadIdx.x == 0) {
            *p.ticket = 0ull;
            *p.exit_count = 0u;
        }
        __threadfence();
    }
}

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(UHMV_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

// Launch serialisation of plans that share device state.  One launch of a plan's programs
// owns the ticket / counters / exit count / work buffer (and uhmv_matvec_host the scratch
// vectors) until it exits, so two launches of the same state must never overlap -- e.g. two
// streams, or two host threads, calling uhmv_execute on one plan.  Plans are grouped by their
// ticket pointer (the multi-RHS plan shares its parent's, device.py share_with): a group has
// one host mutex held while a call enqueues, and one event recorded after each launch that a
// launch on a DIFFERENT stream waits for.  Same-stream calls cost one cudaEventRecord.  While
// the stream is being captured into a graph the event ordering is skipped (the captured graph
// must then be replayed on one stream at a time).
struct SyncState {
    std::mutex mu;
    cudaEvent_t ev = nullptr;
    cudaStream_t last = nullptr;
    bool recorded = false;
    int refs = 0;
};
static std::mutex g_sync_mu;
static std::map<const void*, SyncState*> g_sync;

static SyncState* sync_acquire(const void* key) {
    std::lock_guard<std::mutex> g(g_sync_mu);
    SyncState*& s = g_sync[key];
    if (!s) s = new SyncState();
    ++s->refs;
    return s;
}
static void sync_release(const void* key, SyncState* s) {
    if (!s) return;
    std::lock_guard<std::mutex> g(g_sync_mu);
    if (--s->refs == 0) {
        if (s->ev) cudaEventDestroy(s->ev);
        g_sync.erase(key);
        delete s;
    }
}

struct uhmv_plan {
    uhmv_desc d;
    SyncState* sync;  // shared by every plan on the same ticket (see SyncState)
    int fused_grid[2];
    int smem[2];
    int bulk_grid[2];
    int bulk_full_grid[2];  // resident CTAs per SM x SMs (the peer launch splits it over ranks)
    // host-I/O programs (uhmv_plan_set_io): x read from / w drained to pinned host buffers
    bool has_io;
    uhmv_program io[2];
    uint32_t* io_counters;
    int io_grid[2], io_smem[2], io_nstage[2];
    const void* io_x_host;  // last mapped pointers (cudaPointerGetAttributes is ~1 us a call)
    void* io_x_dev;
    const void* io_w_host;
    void* io_w_dev;
    // CUDA graphs of the whole host call (copies / memset / kernel) per direction, for pinned
    // buffers: one graph launch replaces four API calls (UHMV_HOST_GRAPH=0 disables)
    cudaGraphExec_t hg_exec[2];
    const void* hg_x[2];
    void* hg_w[2];
    int hg_mode[2];
    int hg_io[2];
    cudaGraphExec_t hg_alt[2];  // the graph of the other host path (io vs copy), kept for replay
    const void* ha_x[2];
    void* ha_w[2];
    int ha_mode[2];
    int ha_io[2];
    int host_path[2];       // pinned host calls: 1 host-I/O launch (when attached), 0 copy path
    int last_host_path[2];  // path the last uhmv_matvec_host took: 1 io, 0 copy, -1 pageable
    cudaEvent_t mm_start;   // uhmv_matmat_host: orders its streams after the caller's
    cudaStream_t cap_stream;  // capture stream (the caller's may be the legacy default stream)
    // pipelined host-buffer multi-RHS (uhmv_matmat_host): copy-in / compute / copy-out streams
    cudaStream_t mm_stream[3];
    cudaEvent_t mm_ev[3][2];
    int no_graphs;
    int bulk_smem[2];
    int bulk_nstage[2];
    int sm_count;
    int debug_skip_waits;  // diagnostics only (UHMV_DEBUG_SKIP_WAITS): results are wrong
    unsigned long long* prof;  // diagnostics only (uhmv_plan_set_profile)
    unsigned long long* trace;  // diagnostics only (uhmv_plan_set_trace)
    int debug_flags;           // diagnostics only (UHMV_DEBUG_FLAGS): results are wrong
    int mrhs_grid;
    int mrtc_grid;
    int mrhs_engine;  // 0: staged tensor-core engine (mrtc), 1: register engine (UHMV_MRHS_ENGINE=simple)
};

extern "C" {

int uhmv_abi_version(void) { return UHMV_ABI_VERSION; }

const char* uhmv_last_error(void) { return g_last_error.c_str(); }

static int check_program(const uhmv_program& pr, const char* name) {
    if (pr.n_ops < 0 || pr.n_phases < 0 || pr.n_phases > UHMV_MAX_PHASES)
        return fail(UHMV_EINVAL, std::string(name) + ": bad op/phase count");
    if (pr.n_ops > 0 && (!pr.ops || !pr.segs || !pr.runs || !pr.fused_order))
        return fail(UHMV_EINVAL, std::string(name) + ": null table pointer");
    if (pr.in_max < 0 || pr.out_max < 0 || pr.n_counters < 0)
        return fail(UHMV_EINVAL, std::string(name) + ": negative size");
    for (int i = 0; i < pr.n_phases; ++i)
        if (pr.phase_lo[i] < 0 || pr.phase_hi[i] < pr.phase_lo[i] || pr.phase_hi[i] > pr.n_ops)
            return fail(UHMV_EINVAL, std::string(name) + ": bad phase bounds");
    return UHMV_OK;
}

// TMA tensor maps over the arena for the staged multi-RHS engine: for every leading dimension
// L the arena is viewed as a 2-D tensor of ceil(arena_len / L) rows x 2L doubles (row stride
// 16 L bytes), so a segment at element offset m_off starts at (row, col) = divmod(m_off, L)
// whatever its alignment.  Box 0 (N segments): 16 rows x 16 complex; box 1 (H segments):
// 16 rows x 80 complex.  Columns past 2L are zero-filled by the TMA unit.
static int encode_tmaps(const uhmv_desc* d, const uhmv_program& pr, const char* name) {
    if (pr.n_tmaps <= 0) return UHMV_OK;
    if (!pr.tmap_lds || !pr.tmaps) return fail(UHMV_EINVAL, std::string(name) + ": null tensor-map buffers");
    if (reinterpret_cast<uintptr_t>(pr.tmaps) % 64 || reinterpret_cast<uintptr_t>(d->arena) % 16)
        return fail(UHMV_EINVAL, std::string(name) + ": misaligned tensor-map buffer or arena");
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return fail(UHMV_ECUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    std::vector<CUtensorMap> maps(2 * (size_t)pr.n_tmaps);
    for (int i = 0; i < pr.n_tmaps; ++i) {
        const int64_t L = pr.tmap_lds[i];
        if (L <= 0 || L > (1 << 24)) return fail(UHMV_EINVAL, std::string(name) + ": bad leading dimension");
        const cuuint64_t rows = (cuuint64_t)((d->arena_len + L - 1) / L);
        const cuuint64_t gdim[2] = {(cuuint64_t)(2 * L), rows > 0 ? rows : 1};
        const cuuint64_t gstride[1] = {(cuuint64_t)(16 * L)};
        const cuuint32_t estride[2] = {1, 1};
        for (int b = 0; b < 2; ++b) {
            const cuuint32_t box[2] = {b == 0 ? 2u * mrtc::kKC : 2u * mrtc::kNP, (cuuint32_t)mrtc::kKC};
            CUresult r = encode(&maps[2 * i + b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(d->arena),
                                gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                return fail(UHMV_ECUDA, std::string(name) + ": cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        }
    }
    cudaError_t e = cudaMemcpy(pr.tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(tensor maps)");
    return UHMV_OK;
}

// Shared-memory stages, dynamic shared memory and persistent grid of the bulk engine for one
// program (as many stages as fit with the requested CTAs per SM).
static int size_bulk(int device, int sm_count, const uhmv_program* pr, int* nstage, int* smem, int* grid,
                     int* full_grid) {
    int smem_sm = 0, smem_optin = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    int want_ctas = 3;
    if (const char* ev = getenv("UHMV_BULK_CTAS")) want_ctas = atoi(ev) > 0 ? atoi(ev) : 3;
    int want_stages = 0;
    if (const char* ev = getenv("UHMV_NSTAGE")) want_stages = atoi(ev);
    int budget = smem_sm / want_ctas - 1024;
    if (budget > smem_optin) budget = smem_optin;
    const int sbytes = (pr->stage_elems > 0 ? pr->stage_elems : 1408) * 16;
    const int fixed = bulk::layout(0, sbytes, pr->xin_max, pr->out_max).total;
    int ns = (budget - fixed) / sbytes;
    if (want_stages > 0) ns = want_stages;
    if (ns > 12) ns = 12;
    if (ns < 2) ns = 2;
    *nstage = ns;
    *smem = bulk::layout(ns, sbytes, pr->xin_max, pr->out_max).total;
    if (*smem > smem_optin) return fail(UHMV_EINVAL, "bulk engine shared memory exceeds the opt-in limit");
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bulk::uhmv_bulk_kernel<false>,
                                                                  bulk::kThreads, *smem);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy(bulk)");
    if (per_sm < 1) per_sm = 1;
    *full_grid = per_sm * sm_count;
    *grid = *full_grid;
    if (*grid > pr->n_ops) *grid = pr->n_ops > 0 ? pr->n_ops : 1;
    return UHMV_OK;
}

int uhmv_plan_create(const uhmv_desc* desc, uhmv_plan** out) {
    if (!desc || !out) return fail(UHMV_EINVAL, "uhmv_plan_create: null argument");
    *out = nullptr;
    if (desc->abi_version != UHMV_ABI_VERSION)
        return fail(UHMV_EINVAL, "uhmv_plan_create: ABI version mismatch");
    if (desc->n_rows < 0 || desc->n_cols < 0) return fail(UHMV_EINVAL, "negative shape");
    if (!desc->counters || !desc->ticket || !desc->exit_count || !desc->arena || !desc->work)
        return fail(UHMV_EINVAL, "uhmv_plan_create: null device buffer");
    int rc = check_program(desc->fwd, "fwd");
    if (rc) return rc;
    rc = check_program(desc->adj, "adj");
    if (rc) return rc;
    cudaError_t e = cudaSetDevice(desc->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    uhmv_plan* p = new (std::nothrow) uhmv_plan;
    if (!p) return fail(UHMV_ENOMEM, "uhmv_plan_create: out of host memory");
    std::memset(p, 0, sizeof(*p));
    p->d = *desc;
    if ((rc = encode_tmaps(desc, desc->fwd, "fwd")) || (rc = encode_tmaps(desc, desc->adj, "adj"))) {
        delete p;
        return rc;
    }
    e = cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, desc->device);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "cudaDeviceGetAttribute");
    }
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, desc->device);
    const uhmv_program* progs[2] = {&desc->fwd, &desc->adj};
    int need = 0;
    for (int k = 0; k < 2; ++k) {
        p->smem[k] = smem_layout(progs[k]->in_max, progs[k]->out_max).total;
        if (p->smem[k] > need) need = p->smem[k];
    }
    if (need > smem_optin) {
        delete p;
        return fail(UHMV_EINVAL, "op vectors exceed shared memory (" + std::to_string(need) +
                                     " > " + std::to_string(smem_optin) + " bytes)");
    }
    // the attribute is per function, shared by every plan: always allow the opt-in maximum
    e = cudaFuncSetAttribute(uhmv_phase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem_optin);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(uhmv_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_optin);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "cudaFuncSetAttribute");
    }
    for (int k = 0; k < 2; ++k) {
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, uhmv_fused_kernel, kThreads,
                                                          p->smem[k]);
        if (e != cudaSuccess) {
            delete p;
            return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
        }
        if (per_sm < 1) per_sm = 1;
        int grid = per_sm * p->sm_count;
        if (grid > progs[k]->n_ops) grid = progs[k]->n_ops > 0 ? progs[k]->n_ops : 1;
        p->fused_grid[k] = grid;
    }
    // bulk engine: as many 16-KiB stages as fit with the requested CTAs per SM
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, desc->device);
    int want_ctas = 3;
    if (const char* ev = getenv("UHMV_BULK_CTAS")) want_ctas = atoi(ev) > 0 ? atoi(ev) : 3;
    int want_stages = 0;
    if (const char* ev = getenv("UHMV_NSTAGE")) want_stages = atoi(ev);
    int bulk_need = 0;
    for (int k = 0; k < 2; ++k) {
        const uhmv_program* pr = progs[k];
        int budget = smem_sm / want_ctas - 1024;
        if (budget > smem_optin) budget = smem_optin;
        const int sbytes = (pr->stage_elems > 0 ? pr->stage_elems : 1408) * 16;
        const int fixed = bulk::layout(0, sbytes, pr->xin_max, pr->out_max).total;
        int ns = (budget - fixed) / sbytes;
        if (want_stages > 0) ns = want_stages;
        if (ns > 12) ns = 12;
        if (ns < 2) ns = 2;
        p->bulk_nstage[k] = ns;
        p->bulk_smem[k] = bulk::layout(ns, sbytes, pr->xin_max, pr->out_max).total;
        if (p->bulk_smem[k] > bulk_need) bulk_need = p->bulk_smem[k];
    }
    if (bulk_need > smem_optin) {
        delete p;
        return fail(UHMV_EINVAL, "bulk engine shared memory exceeds the opt-in limit");
    }
    e = cudaFuncSetAttribute(bulk::uhmv_bulk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem_optin);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(bulk::uhmv_bulk_sym_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_optin);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(bulk::uhmv_bulk_sym_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_optin);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(bulk::uhmv_bulk_peer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_optin);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(bulk::uhmv_bulk_io_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_optin);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(bulk::uhmv_bulk_kernel<true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
    // the whole shared-memory carveout: several CTAs per SM need it (the driver's default
    // choice can leave room for one CTA of ~110 KB only)
    for (const void* fn : {(const void*)bulk::uhmv_bulk_xwin_kernel<false>, (const void*)bulk::uhmv_bulk_xwin_kernel<true>})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
    for (const void* fn : {(const void*)bulk::uhmv_bulk_kernel<false>, (const void*)bulk::uhmv_bulk_kernel<true>,
                           (const void*)bulk::uhmv_bulk_xwin_kernel<false>, (const void*)bulk::uhmv_bulk_xwin_kernel<true>,
                           (const void*)bulk::uhmv_bulk_sym_kernel<false>, (const void*)bulk::uhmv_bulk_sym_kernel<true>,
                           (const void*)bulk::uhmv_bulk_io_kernel, (const void*)bulk::uhmv_bulk_peer_kernel})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "cudaFuncSetAttribute(bulk)");
    }
    for (int k = 0; k < 2; ++k) {
        int per_sm = 0;
        const bool sym = (progs[k]->flags & UHMV_PROG_SYM) != 0;
        const bool xw = (progs[k]->flags & UHMV_PROG_XWIN) != 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, sym ? (const void*)bulk::uhmv_bulk_sym_kernel<false>
                         : xw ? (const void*)bulk::uhmv_bulk_xwin_kernel<false> : (const void*)bulk::uhmv_bulk_kernel<false>,
            bulk::kThreads, p->bulk_smem[k]);
        if (e != cudaSuccess) {
            delete p;
            return cuda_fail(e, "occupancy(bulk)");
        }
        if (per_sm < 1) per_sm = 1;
        int grid = per_sm * p->sm_count;
        p->bulk_full_grid[k] = grid;
        if (grid > progs[k]->n_ops) grid = progs[k]->n_ops > 0 ? progs[k]->n_ops : 1;
        p->bulk_grid[k] = grid;
    }
    {
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mrhs::uhmv_mrhs_kernel,
                                                          mrhs::kThreads, 0);
        if (e != cudaSuccess) {
            delete p;
            return cuda_fail(e, "occupancy(mrhs)");
        }
        p->mrhs_grid = (per_sm < 1 ? 1 : per_sm) * p->sm_count;
        e = cudaFuncSetAttribute(mrtc::uhmv_mrtc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 mrtc::kSmemBytes);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(mrtc::uhmv_mrtc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     mrtc::kSmemBytes);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mrtc::uhmv_mrtc_kernel<false>,
                                                              mrtc::kThreads, mrtc::kSmemBytes);
        if (e != cudaSuccess) {
            delete p;
            return cuda_fail(e, "occupancy(mrtc)");
        }
        p->mrtc_grid = (per_sm < 1 ? 1 : per_sm) * p->sm_count;
        const char* ev = getenv("UHMV_MRHS_ENGINE");
        p->mrhs_engine = (ev && strcmp(ev, "simple") == 0) ? 1 : 0;
    }
#ifdef UHMV_DIAGNOSTICS  // diagnostics builds only (UHMV_NVCC_EXTRA=-DUHMV_DIAGNOSTICS): wrong results
    if (const char* ev = getenv("UHMV_DEBUG_SKIP_WAITS")) p->debug_skip_waits = atoi(ev);
    if (const char* ev = getenv("UHMV_DEBUG_FLAGS")) p->debug_flags = atoi(ev);
#endif
    p->host_path[0] = p->host_path[1] = 1;
    p->sync = sync_acquire(desc->ticket);
    if (const char* ev = getenv("UHMV_HOST_GRAPH")) p->no_graphs = (atoi(ev) == 0);
    *out = p;
    return UHMV_OK;
}

static bulk::Params make_bulk_params(const uhmv_plan* plan, const uhmv_program& pr, int k,
                                     const void* x, void* w) {
    bulk::Params bp;
    bp.arena = static_cast<const double2*>(plan->d.arena);
    bp.work = static_cast<double2*>(plan->d.work);
    bp.x = static_cast<const double2*>(x);
    bp.w = static_cast<double2*>(w);
    bp.ops = pr.ops;
    bp.pieces = pr.pieces;
    bp.runs = pr.runs;
    bp.waits = pr.waits;
    bp.sigs = pr.sigs;
    bp.fused_order = pr.fused_order;
    bp.op_count = pr.n_ops;
    bp.nstage = plan->bulk_nstage[k];
    bp.stage_bytes = (pr.stage_elems > 0 ? pr.stage_elems : 1408) * 16;
    bp.counters = plan->d.counters;
    bp.ticket = plan->d.ticket;
    bp.exit_count = plan->d.exit_count;
    bp.n_counters = pr.n_counters;
    bp.xin_max = pr.xin_max;
    bp.out_max = pr.out_max;
    bp.skip_waits = plan->debug_skip_waits;
    bp.prof = plan->prof;
    bp.trace = plan->prof ? plan->trace : nullptr;
    bp.dbg = plan->debug_flags;
    bp.x_host = nullptr;
    bp.w_host = nullptr;
    bp.diag = nullptr;
    return bp;
}

static ExecParams make_params(const uhmv_plan* plan, const uhmv_program& pr, const void* x,
                              void* w) {
    ExecParams ep;
    ep.arena = static_cast<const double2*>(plan->d.arena);
    ep.work = static_cast<double2*>(plan->d.work);
    ep.x = static_cast<const double2*>(x);
    ep.w = static_cast<double2*>(w);
    ep.ops = pr.ops;
    ep.segs = pr.segs;
    ep.runs = pr.runs;
    ep.waits = pr.waits;
    ep.sigs = pr.sigs;
    ep.fused_order = pr.fused_order;
    ep.op_begin = 0;
    ep.op_count = pr.n_ops;
    ep.counters = plan->d.counters;
    ep.ticket = plan->d.ticket;
    ep.exit_count = plan->d.exit_count;
    ep.n_counters = pr.n_counters;
    ep.in_max = pr.in_max;
    ep.out_max = pr.out_max;
    return ep;
}

// Serialises one enqueue of a plan group (see SyncState): holds the group's mutex, orders the
// launch after the group's previous launch when that ran on another stream, and records the
// group's event after it.
class Serial {
  public:
    Serial(uhmv_plan* p, cudaStream_t st) : s_(p->sync), st_(st), lk_(p->sync->mu) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
            cudaGetLastError();
            cs = cudaStreamCaptureStatusNone;
        }
        cap_ = cs != cudaStreamCaptureStatusNone;
    }
    int begin() {
        if (cap_ || !s_->recorded || s_->last == st_) return UHMV_OK;
        cudaError_t e = cudaStreamWaitEvent(st_, s_->ev, 0);
        return e == cudaSuccess ? UHMV_OK : cuda_fail(e, "cudaStreamWaitEvent (plan serialisation)");
    }
    int end() {
        if (cap_) return UHMV_OK;
        cudaError_t e = cudaSuccess;
        if (!s_->ev) e = cudaEventCreateWithFlags(&s_->ev, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(s_->ev, st_);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord (plan serialisation)");
        s_->recorded = true;
        s_->last = st_;
        return UHMV_OK;
    }

  private:
    SyncState* s_;
    cudaStream_t st_;
    std::unique_lock<std::mutex> lk_;
    bool cap_ = false;
};

static int execute_phases_impl(uhmv_plan* plan, const void* x, void* w, int adjoint, int phase_lo, int phase_hi,
                               void* stream);
static int execute_impl(uhmv_plan* plan, const void* x, void* w, int adjoint, int mode, void* stream);
static int execute_mrhs_impl(uhmv_plan* plan, const void* x, void* w, void* work_mr, int nrhs, int adjoint,
                             void* stream);

// Public enqueue entry points: argument check, then the guarded implementation.
extern "C++" {
template <class F>
static int serialised(uhmv_plan* plan, void* stream, F&& body) {
    Serial g(plan, static_cast<cudaStream_t>(stream));
    int rc = g.begin();
    if (rc) return rc;
    rc = body();
    const int rc2 = g.end();
    return rc ? rc : rc2;
}
}  // extern "C++"

int uhmv_execute_phases(uhmv_plan* plan, const void* x, void* w, int adjoint, int phase_lo, int phase_hi,
                        void* stream) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_execute_phases: null plan");
    return serialised(plan, stream, [&] { return execute_phases_impl(plan, x, w, adjoint, phase_lo, phase_hi, stream); });
}

int uhmv_execute(uhmv_plan* plan, const void* x, void* w, int adjoint, int mode, void* stream) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_execute: null plan");
    return serialised(plan, stream, [&] { return execute_impl(plan, x, w, adjoint, mode, stream); });
}

int uhmv_execute_mrhs(uhmv_plan* plan, const void* x, void* w, void* work_mr, int nrhs, int adjoint, void* stream) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_execute_mrhs: null plan");
    return serialised(plan, stream, [&] { return execute_mrhs_impl(plan, x, w, work_mr, nrhs, adjoint, stream); });
}

static int execute_phases_impl(uhmv_plan* plan, const void* x, void* w, int adjoint, int phase_lo, int phase_hi,
                               void* stream) {
    const uhmv_program& pr = adjoint ? plan->d.adj : plan->d.fwd;
    const int k = adjoint ? 1 : 0;
    if (pr.flags & UHMV_PROG_SYM)
        return fail(UHMV_EINVAL, "uhmv_execute_phases: symmetric single-triangle programs run on the bulk engine only");
    if (phase_lo < 0 || phase_hi > pr.n_phases || phase_lo > phase_hi)
        return fail(UHMV_EINVAL, "uhmv_execute_phases: bad phase range");
    if (pr.n_ops > 0 && (!x || !w)) return fail(UHMV_EINVAL, "null vector pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n_out = adjoint ? plan->d.n_cols : plan->d.n_rows;
    if (phase_lo == 0 && n_out > 0 && pr.zero_output) {  // NEAR/FAR add into a zeroed output
        cudaError_t e0 = cudaMemsetAsync(w, 0, (size_t)n_out * 16, st);
        if (e0 != cudaSuccess) return cuda_fail(e0, "cudaMemsetAsync(w)");
    }
    ExecParams ep = make_params(plan, pr, x, w);
    for (int ph = phase_lo; ph < phase_hi; ++ph) {
        const int n = pr.phase_hi[ph] - pr.phase_lo[ph];
        if (n <= 0) continue;
        ep.op_begin = pr.phase_lo[ph];
        uhmv_phase_kernel<<<n, kThreads, plan->smem[k], st>>>(ep);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "uhmv_phase_kernel launch");
    return UHMV_OK;
}

static int execute_impl(uhmv_plan* plan, const void* x, void* w, int adjoint, int mode, void* stream) {
    const uhmv_program& pr = adjoint ? plan->d.adj : plan->d.fwd;
    if (mode == UHMV_MODE_PHASED)
        return execute_phases_impl(plan, x, w, adjoint, 0, pr.n_phases, stream);
    if (mode != UHMV_MODE_FUSED && mode != UHMV_MODE_BULK)
        return fail(UHMV_EINVAL, "uhmv_execute: unknown mode");
    if ((pr.flags & UHMV_PROG_SYM) && mode != UHMV_MODE_BULK)
        return fail(UHMV_EINVAL, "uhmv_execute: symmetric single-triangle programs run on the bulk engine only");
    const int64_t n_out = adjoint ? plan->d.n_cols : plan->d.n_rows;
    if (n_out > 0 && pr.zero_output && !(plan->debug_flags & 4)) {  // NEAR/FAR add into a zeroed output
        if (!w) return fail(UHMV_EINVAL, "null output pointer");
        cudaError_t e0 = cudaMemsetAsync(w, 0, (size_t)n_out * 16, static_cast<cudaStream_t>(stream));
        if (e0 != cudaSuccess) return cuda_fail(e0, "cudaMemsetAsync(w)");
    }
    if (pr.n_ops == 0) return UHMV_OK;
    if (!x || !w) return fail(UHMV_EINVAL, "null vector pointer");
    const int k = adjoint ? 1 : 0;
    if (mode == UHMV_MODE_BULK) {
        if (!pr.pieces) return fail(UHMV_EINVAL, "bulk mode needs the piece table");
        bulk::Params bp = make_bulk_params(plan, pr, k, x, w);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const bool sym = (pr.flags & UHMV_PROG_SYM) != 0;
        if (pr.flags & UHMV_PROG_XWIN) {
            if (bp.prof)
                bulk::uhmv_bulk_xwin_kernel<true><<<plan->bulk_grid[k], bulk::kThreads, plan->bulk_smem[k], st>>>(bp);
            else
                bulk::uhmv_bulk_xwin_kernel<false><<<plan->bulk_grid[k], bulk::kThreads, plan->bulk_smem[k], st>>>(bp);
        } else if (bp.prof && sym)
            bulk::uhmv_bulk_sym_kernel<true><<<plan->bulk_grid[k], bulk::kThreads, plan->bulk_smem[k], st>>>(bp);
        else if (sym)
            bulk::uhmv_bulk_sym_kernel<false><<<plan->bulk_grid[k], bulk::kThreads, plan->bulk_smem[k], st>>>(bp);
        else if (bp.prof)
            bulk::uhmv_bulk_kernel<true><<<plan->bulk_grid[k], bulk::kThreads, plan->bulk_smem[k], st>>>(bp);
        else
            bulk::uhmv_bulk_kernel<false><<<plan->bulk_grid[k], bulk::kThreads, plan->bulk_smem[k], st>>>(bp);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "uhmv_bulk_kernel launch");
        return UHMV_OK;
    }
    ExecParams ep = make_params(plan, pr, x, w);
    uhmv_fused_kernel<<<plan->fused_grid[k], kThreads, plan->smem[k],
                        static_cast<cudaStream_t>(stream)>>>(ep);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "uhmv_fused_kernel launch");
    return UHMV_OK;
}

static uint32_t* g_peer_diag = nullptr;
static int g_peer_spin_log2 = 28;

int uhmv_peer_set_diag(void* host_mapped, int spin_log2) {
    g_peer_diag = static_cast<uint32_t*>(host_mapped);
    g_peer_spin_log2 = (spin_log2 >= 10 && spin_log2 <= 40) ? spin_log2 : 28;
    return UHMV_OK;
}

static void drop_host_graphs(uhmv_plan* plan);

int uhmv_plan_set_io(uhmv_plan* plan, const uhmv_program* fwd, const uhmv_program* adj, uint32_t* counters) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_plan_set_io: null plan");
    std::lock_guard<std::mutex> guard(plan->sync->mu);
    if (!fwd && !adj) {  // detach
        plan->has_io = false;
        drop_host_graphs(plan);
        return UHMV_OK;
    }
    if (!fwd || !adj || !counters) return fail(UHMV_EINVAL, "uhmv_plan_set_io: null argument");
    int rc = check_program(*fwd, "io fwd");
    if (rc || (rc = check_program(*adj, "io adj"))) return rc;
    if ((fwd->flags | adj->flags) & (UHMV_PROG_SYM | UHMV_PROG_XWIN))
        return fail(UHMV_EINVAL, "uhmv_plan_set_io: symmetric / windowed programs have no host-I/O engine");
    cudaError_t e = cudaSetDevice(plan->d.device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    const uhmv_program* progs[2] = {fwd, adj};
    for (int k = 0; k < 2; ++k) {
        if (progs[k]->n_ops > 0 && !progs[k]->pieces) return fail(UHMV_EINVAL, "io program without pieces");
        int full = 0;
        if ((rc = size_bulk(plan->d.device, plan->sm_count, progs[k], &plan->io_nstage[k], &plan->io_smem[k],
                            &plan->io_grid[k], &full)))
            return rc;
        plan->io[k] = *progs[k];
    }
    plan->io_counters = counters;
    plan->has_io = true;
    drop_host_graphs(plan);  // captured graphs hold the previous programs
    return UHMV_OK;
}

// Device pointer of a pinned (page-locked) host buffer, or null for pageable memory.
static void* mapped_ptr(const void* host) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
        cudaGetLastError();  // clear the sticky-free error of an unregistered pointer
        return nullptr;
    }
    return (a.type == cudaMemoryTypeHost && a.devicePointer) ? a.devicePointer : nullptr;
}

int uhmv_execute_peer(uhmv_plan* const* plans, int nplans, int rank0, int world,
                      const uhmv_peer_rank* ranks, const void* x, void* const* w, int adjoint,
                      uint32_t epoch, void* stream) {
    if (!plans || !ranks || !w || !x) return fail(UHMV_EINVAL, "uhmv_execute_peer: null argument");
    if (world < 1 || world > bulk::kMaxRanks || nplans < 1 || rank0 < 0 || rank0 + nplans > world)
        return fail(UHMV_EINVAL, "uhmv_execute_peer: bad rank range");
    if (epoch == 0) return fail(UHMV_EINVAL, "uhmv_execute_peer: epochs start at 1");
    for (int q = 0; q < world; ++q)
        if (!ranks[q].work || !ranks[q].counters || !ranks[q].done || ranks[q].work_len < 0)
            return fail(UHMV_EINVAL, "uhmv_execute_peer: null peer buffer");
    const int k = adjoint ? 1 : 0;
    for (int i = 0; i < nplans; ++i)
        if ((adjoint ? plans[i]->d.adj : plans[i]->d.fwd).flags & (UHMV_PROG_SYM | UHMV_PROG_XWIN))
            return fail(UHMV_EINVAL, "uhmv_execute_peer: symmetric / windowed programs have no peer engine");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int grid = 0, smem = 0;
    for (int i = 0; i < nplans; ++i) {
        if (!plans[i]) return fail(UHMV_EINVAL, "uhmv_execute_peer: null plan");
        const uhmv_program& pr = adjoint ? plans[i]->d.adj : plans[i]->d.fwd;
        if (pr.n_ops > 0 && !pr.pieces) return fail(UHMV_EINVAL, "peer execution needs the piece table");
        if (plans[i]->bulk_smem[k] > smem) smem = plans[i]->bulk_smem[k];
        // every CTA must be resident (ranks wait on one another inside the launch): the
        // smallest full grid, i.e. the one of the largest shared-memory footprint
        if (i == 0 || plans[i]->bulk_full_grid[k] < grid) grid = plans[i]->bulk_full_grid[k];
        if (!w[i]) return fail(UHMV_EINVAL, "uhmv_execute_peer: null output");
        bool seen = false;  // zero every distinct output once (NEAR/FAR add into it)
        for (int j = 0; j < i; ++j) seen = seen || (w[j] == w[i]);
        const int64_t n_out = adjoint ? plans[i]->d.n_cols : plans[i]->d.n_rows;
        if (!seen && n_out > 0) {
            cudaError_t e0 = cudaMemsetAsync(w[i], 0, (size_t)n_out * 16, st);
            if (e0 != cudaSuccess) return cuda_fail(e0, "cudaMemsetAsync(w)");
        }
    }
    {
        // every CTA of the launch must be co-resident: the grid comes from the occupancy of the
        // peer kernel itself at the launch's shared memory (it can differ from the bulk kernel's)
        int per_sm = 0;
        cudaError_t eo = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bulk::uhmv_bulk_peer_kernel,
                                                                       bulk::kThreads, smem);
        if (eo != cudaSuccess) return cuda_fail(eo, "occupancy(bulk_peer)");
        if (per_sm * plans[0]->sm_count < grid) grid = per_sm * plans[0]->sm_count;
    }
    if (grid < nplans) return fail(UHMV_EINVAL, "uhmv_execute_peer: fewer co-resident CTAs than ranks");
    bulk::PeerLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.nranks = nplans;
    for (int i = 0; i < nplans; ++i) {
        const int r = rank0 + i;
        const uhmv_program& pr = adjoint ? plans[i]->d.adj : plans[i]->d.fwd;
        bulk::Params bp = make_bulk_params(plans[i], pr, k, x, w[i]);
        bp.prof = nullptr;
        bp.rank = r;
        bp.world = world;
        bp.epoch = epoch;
        const long long lo = ((long long)i * grid + nplans - 1) / nplans;
        const long long hi = ((long long)(i + 1) * grid + nplans - 1) / nplans;
        bp.n_ctas = (int32_t)(hi - lo);
        for (int q = 0; q < world; ++q) {
            bp.peer_work[q] = static_cast<double2*>(ranks[q].work) + (epoch & 1u) * ranks[q].work_len;
            bp.peer_counters[q] = ranks[q].counters;
            bp.peer_done[q] = ranks[q].done;
        }
        bp.diag = g_peer_diag;
        bp.spin_log2 = g_peer_spin_log2;
        bp.work = bp.peer_work[r];
        bp.counters = ranks[r].counters;
        bp.done = ranks[r].done;
        L.r[i] = bp;
    }
    // serialise against other launches of each involved plan group (locked in address order)
    std::vector<uhmv_plan*> grp;
    for (int i = 0; i < nplans; ++i) {
        bool dup = false;
        for (uhmv_plan* q : grp) dup = dup || (q->sync == plans[i]->sync);
        if (!dup) grp.push_back(plans[i]);
    }
    std::sort(grp.begin(), grp.end(), [](const uhmv_plan* a, const uhmv_plan* b) { return a->sync < b->sync; });
    std::vector<std::unique_ptr<Serial>> guards;
    for (uhmv_plan* q : grp) {
        guards.emplace_back(new Serial(q, st));
        const int r = guards.back()->begin();
        if (r) return r;
    }
    bulk::uhmv_bulk_peer_kernel<<<grid, bulk::kThreads, smem, st>>>(L);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "uhmv_bulk_peer_kernel launch");
    for (auto& g : guards) {
        const int r = g->end();
        if (r) return r;
    }
    return UHMV_OK;
}

static int execute_mrhs_impl(uhmv_plan* plan, const void* x, void* w, void* work_mr, int nrhs, int adjoint,
                             void* stream) {
    if (((adjoint ? plan->d.adj : plan->d.fwd).flags & UHMV_PROG_SYM))
        return fail(UHMV_EINVAL, "uhmv_execute_mrhs: no multi-RHS engine for symmetric single-triangle programs");
    if (nrhs <= 0 || nrhs % mrhs::kRC) return fail(UHMV_EINVAL, "nrhs must be a multiple of 16");
    const uhmv_program& pr = adjoint ? plan->d.adj : plan->d.fwd;
    if (!pr.mr_segs || !pr.mr_ranges) return fail(UHMV_EINVAL, "program has no multi-RHS tables");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n_out = adjoint ? plan->d.n_cols : plan->d.n_rows;
    if (n_out > 0 && (pr.zero_output || (pr.flags & UHMV_PROG_WORDER))) {  // the engines add into W
        cudaError_t e0 = cudaMemsetAsync(w, 0, (size_t)n_out * nrhs * 16, st);
        if (e0 != cudaSuccess) return cuda_fail(e0, "cudaMemsetAsync(W)");
    }
    if (pr.n_ops == 0) return UHMV_OK;
    if (!x || !w || !work_mr) return fail(UHMV_EINVAL, "null matrix pointer");
    mrhs::Params mp;
    mp.arena = static_cast<const double2*>(plan->d.arena);
    mp.work = static_cast<double2*>(work_mr);
    mp.x = static_cast<const double2*>(x);
    mp.w = static_cast<double2*>(w);
    mp.ops = pr.ops;
    mp.runs = pr.runs;
    mp.waits = pr.waits;
    mp.sigs = pr.sigs;
    mp.fused_order = pr.fused_order;
    mp.mr_segs = pr.mr_segs;
    mp.mr_ranges = pr.mr_ranges;
    mp.op_count = pr.n_ops;
    mp.nrhs = nrhs;
    mp.counters = plan->d.counters;
    mp.ticket = plan->d.ticket;
    mp.exit_count = plan->d.exit_count;
    mp.n_counters = pr.n_counters;
    mp.prof = nullptr;
    mp.tmaps = static_cast<const CUtensorMap*>(pr.tmaps);
    if (plan->mrhs_engine == 1) {
        int grid = plan->mrhs_grid < pr.n_ops ? plan->mrhs_grid : pr.n_ops;
        mrhs::uhmv_mrhs_kernel<<<grid, mrhs::kThreads, 0, st>>>(mp);
    } else {
        if (pr.n_tmaps <= 0 && pr.n_ops > 0) return fail(UHMV_EINVAL, "multi-RHS program without tensor maps");
        int grid = plan->mrtc_grid < pr.n_ops ? plan->mrtc_grid : pr.n_ops;
        mp.prof = plan->prof;
        if (mp.prof)
            mrtc::uhmv_mrtc_kernel<true><<<grid, mrtc::kThreads, mrtc::kSmemBytes, st>>>(mp);
        else
            mrtc::uhmv_mrtc_kernel<false><<<grid, mrtc::kThreads, mrtc::kSmemBytes, st>>>(mp);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "multi-RHS kernel launch");
    return UHMV_OK;
}

// Enqueue one host-buffer matvec on st (no synchronize): the host-I/O launch (io = true;
// x_dev / w_dev are the device-visible pointers of the pinned buffers) or H2D copy + execute
// + D2H copy.
static int enqueue_host(uhmv_plan* plan, const void* x_host, void* w_host, int adjoint, int mode, cudaStream_t st,
                        bool io, const void* x_dev, void* w_dev) {
    const int64_t n_in = adjoint ? plan->d.n_rows : plan->d.n_cols;
    const int64_t n_out = adjoint ? plan->d.n_cols : plan->d.n_rows;
    const int k = adjoint ? 1 : 0;
    if (io) {
        // ONE launch reads x over PCIe (P1 ops) and drains finished output leaves to w_host
        // as they complete -- no separate H2D / D2H copies
        cudaError_t e0 = cudaMemsetAsync(plan->d.w_scratch, 0, (size_t)n_out * 16, st);
        if (e0 != cudaSuccess) return cuda_fail(e0, "cudaMemsetAsync(w)");
        const uhmv_program& pr = plan->io[k];
        bulk::Params bp = make_bulk_params(plan, pr, k, plan->d.x_scratch, plan->d.w_scratch);
        bp.nstage = plan->io_nstage[k];
        bp.counters = plan->io_counters;
        bp.prof = nullptr;
        bp.trace = nullptr;
        bp.x_host = static_cast<const double2*>(x_dev);
        bp.w_host = static_cast<double2*>(w_dev);
        bulk::uhmv_bulk_io_kernel<<<plan->io_grid[k], bulk::kThreads, plan->io_smem[k], st>>>(bp);
        e0 = cudaGetLastError();
        if (e0 != cudaSuccess) return cuda_fail(e0, "uhmv_bulk_kernel (host I/O) launch");
        return UHMV_OK;
    }
    cudaError_t e = cudaMemcpyAsync(plan->d.x_scratch, x_host, (size_t)n_in * 16, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy of x");
    int rc = execute_impl(plan, plan->d.x_scratch, plan->d.w_scratch, adjoint, mode, st);
    if (rc) return rc;
    e = cudaMemcpyAsync(w_host, plan->d.w_scratch, (size_t)n_out * 16, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy of w");
    return UHMV_OK;
}

static void drop_host_graphs(uhmv_plan* plan) {
    for (int k = 0; k < 2; ++k) {
        if (plan->hg_exec[k]) cudaGraphExecDestroy(plan->hg_exec[k]);
        if (plan->hg_alt[k]) cudaGraphExecDestroy(plan->hg_alt[k]);
        plan->hg_exec[k] = nullptr;
        plan->hg_alt[k] = nullptr;
    }
}

int uhmv_host_pinned(const void* host) { return (host && mapped_ptr(host) != nullptr) ? 1 : 0; }

int uhmv_plan_set_host_path(uhmv_plan* plan, int adjoint, int path) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_plan_set_host_path: null plan");
    if (path != 0 && path != 1) return fail(UHMV_EINVAL, "uhmv_plan_set_host_path: path must be 0 or 1");
    std::lock_guard<std::mutex> g(plan->sync->mu);
    plan->host_path[adjoint ? 1 : 0] = path;  // the cached graphs of both paths stay valid
    return UHMV_OK;
}

// The captured graph of a pinned host call: the current one per direction, plus the last graph of
// the other path (so alternating paths, e.g. while choosing between them, replays instead of
// recapturing).
static int host_graph(uhmv_plan* plan, int k, const void* x_host, void* w_host, int mode, bool io,
                      cudaGraphExec_t* out) {
    auto same = [&](const void* gx, void* gw, int gm, int gio) {
        return gx == x_host && gw == w_host && gm == mode && gio == (int)io;
    };
    if (plan->hg_exec[k] && same(plan->hg_x[k], plan->hg_w[k], plan->hg_mode[k], plan->hg_io[k])) {
        *out = plan->hg_exec[k];
        return UHMV_OK;
    }
    if (plan->hg_alt[k] && same(plan->ha_x[k], plan->ha_w[k], plan->ha_mode[k], plan->ha_io[k])) {
        std::swap(plan->hg_exec[k], plan->hg_alt[k]);
        std::swap(plan->hg_x[k], plan->ha_x[k]);
        std::swap(plan->hg_w[k], plan->ha_w[k]);
        std::swap(plan->hg_mode[k], plan->ha_mode[k]);
        std::swap(plan->hg_io[k], plan->ha_io[k]);
        *out = plan->hg_exec[k];
        return UHMV_OK;
    }
    cudaError_t e;
    if (!plan->cap_stream) {
        e = cudaStreamCreateWithFlags(&plan->cap_stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate (graph capture)");
    }
    e = cudaStreamBeginCapture(plan->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamBeginCapture");
    const int rc = enqueue_host(plan, x_host, w_host, k, mode, plan->cap_stream, io, plan->io_x_dev, plan->io_w_dev);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(plan->cap_stream, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    // the current graph becomes the alternate one (the previous alternate is dropped)
    if (plan->hg_alt[k]) cudaGraphExecDestroy(plan->hg_alt[k]);
    plan->hg_alt[k] = plan->hg_exec[k];
    plan->ha_x[k] = plan->hg_x[k];
    plan->ha_w[k] = plan->hg_w[k];
    plan->ha_mode[k] = plan->hg_mode[k];
    plan->ha_io[k] = plan->hg_io[k];
    plan->hg_exec[k] = ex;
    plan->hg_x[k] = x_host;
    plan->hg_w[k] = w_host;
    plan->hg_mode[k] = mode;
    plan->hg_io[k] = (int)io;
    *out = ex;
    return UHMV_OK;
}

int uhmv_matvec_host(uhmv_plan* plan, const void* x_host, void* w_host, int adjoint, int mode,
                     void* stream) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_matvec_host: null plan");
    if (!plan->d.x_scratch || !plan->d.w_scratch)
        return fail(UHMV_EINVAL, "uhmv_matvec_host: plan has no scratch vectors");
    if (!x_host || !w_host) return fail(UHMV_EINVAL, "uhmv_matvec_host: null host pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int k = adjoint ? 1 : 0;
    const int rc = serialised(plan, stream, [&]() -> int {
        // device-visible pointers of pinned buffers (or null), queried every call (~1 us): a
        // cached answer could outlive the allocation it described
        plan->io_x_dev = mapped_ptr(x_host);
        plan->io_x_host = x_host;
        plan->io_w_dev = mapped_ptr(w_host);
        plan->io_w_host = w_host;
        const bool pinned = plan->io_x_dev && plan->io_w_dev;
        const bool io = pinned && plan->has_io && plan->host_path[k] == 1 && mode == UHMV_MODE_BULK &&
                        plan->io[k].n_ops > 0;
        plan->last_host_path[k] = !pinned ? -1 : (io ? 1 : 0);
        if (pinned && !plan->no_graphs && !plan->prof) {
            cudaGraphExec_t ex = nullptr;
            const int r = host_graph(plan, k, x_host, w_host, mode, io, &ex);
            if (r) return r;
            cudaError_t e = cudaGraphLaunch(ex, st);
            return e == cudaSuccess ? UHMV_OK : cuda_fail(e, "cudaGraphLaunch");
        }
        return enqueue_host(plan, x_host, w_host, adjoint, mode, st, io, plan->io_x_dev, plan->io_w_dev);
    });
    // the caller's buffers may still be read / written by copies already enqueued: always drain
    cudaError_t e = cudaStreamSynchronize(st);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "uhmv_matvec_host synchronize");
    return UHMV_OK;
}

int uhmv_plan_last_host_path(const uhmv_plan* plan, int adjoint) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_plan_last_host_path: null plan");
    return plan->last_host_path[adjoint ? 1 : 0];
}

int uhmv_matmat_host(uhmv_plan* plan, const void* X_host, void* W_host, int nrhs, void* X_dev, void* W_dev,
                     void* work_mr, int chunk, int adjoint, void* stream) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_matmat_host: null plan");
    if (!X_host || !W_host || !X_dev || !W_dev || !work_mr) return fail(UHMV_EINVAL, "uhmv_matmat_host: null buffer");
    if (chunk <= 0 || chunk % 16 || nrhs <= 0 || nrhs % chunk)
        return fail(UHMV_EINVAL, "uhmv_matmat_host: chunk must be a multiple of 16 dividing nrhs");
    const int64_t n_in = adjoint ? plan->d.n_rows : plan->d.n_cols;
    const int64_t n_out = adjoint ? plan->d.n_cols : plan->d.n_rows;
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    Serial guard(plan, caller);
    int rc = guard.begin();
    if (rc) return rc;
    cudaError_t e;
    for (int i = 0; i < 3; ++i) {
        if (!plan->mm_stream[i]) {
            e = cudaStreamCreateWithFlags(&plan->mm_stream[i], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate (matmat_host)");
            for (int b = 0; b < 2; ++b) {
                e = cudaEventCreateWithFlags(&plan->mm_ev[i][b], cudaEventDisableTiming);
                if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate (matmat_host)");
            }
        }
    }
    if (!plan->mm_start) {
        e = cudaEventCreateWithFlags(&plan->mm_start, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate (matmat_host)");
    }
    cudaStream_t s_in = plan->mm_stream[0], s_cmp = plan->mm_stream[1], s_out = plan->mm_stream[2];
    // every enqueue below is checked; after the first failure nothing more is enqueued, and the
    // three streams are drained before returning (copies may still read X_host / write W_host)
    auto ck = [&](cudaError_t err, const char* what) {
        if (err != cudaSuccess && rc == UHMV_OK) rc = cuda_fail(err, what);
        return rc == UHMV_OK;
    };
    // order after the caller's prior work on its stream (and the plan group's previous launch)
    if (ck(cudaEventRecord(plan->mm_start, caller), "cudaEventRecord") &&
        ck(cudaStreamWaitEvent(s_in, plan->mm_start, 0), "cudaStreamWaitEvent"))
        ck(cudaStreamWaitEvent(s_cmp, plan->mm_start, 0), "cudaStreamWaitEvent");
    const int nchunk = nrhs / chunk;
    const size_t xc = (size_t)n_in * chunk * 16, wc = (size_t)n_out * chunk * 16;
    for (int c = 0; c < nchunk && rc == UHMV_OK; ++c) {
        const int b = c & 1;
        char* xd = static_cast<char*>(X_dev) + b * xc;
        char* wd = static_cast<char*>(W_dev) + b * wc;
        // chunk c-2 must be done reading xd before its H2D overwrite
        if (c >= 2 && !ck(cudaStreamWaitEvent(s_in, plan->mm_ev[1][b], 0), "cudaStreamWaitEvent")) break;
        // H2D of the chunk's columns: rows of chunk * 16 B out of rows of nrhs * 16 B
        if (!ck(cudaMemcpy2DAsync(xd, (size_t)chunk * 16, static_cast<const char*>(X_host) + (size_t)c * chunk * 16,
                                  (size_t)nrhs * 16, (size_t)chunk * 16, (size_t)n_in, cudaMemcpyHostToDevice, s_in),
                "H2D copy of X") ||
            !ck(cudaEventRecord(plan->mm_ev[0][b], s_in), "cudaEventRecord") ||
            !ck(cudaStreamWaitEvent(s_cmp, plan->mm_ev[0][b], 0), "cudaStreamWaitEvent"))
            break;
        // chunk c-2's W must be copied out before wd is rewritten
        if (c >= 2 && !ck(cudaStreamWaitEvent(s_cmp, plan->mm_ev[2][b], 0), "cudaStreamWaitEvent")) break;
        const int r = execute_mrhs_impl(plan, xd, wd, work_mr, chunk, adjoint, s_cmp);
        if (r) {
            rc = r;
            break;
        }
        if (!ck(cudaEventRecord(plan->mm_ev[1][b], s_cmp), "cudaEventRecord") ||
            !ck(cudaStreamWaitEvent(s_out, plan->mm_ev[1][b], 0), "cudaStreamWaitEvent") ||
            !ck(cudaMemcpy2DAsync(static_cast<char*>(W_host) + (size_t)c * chunk * 16, (size_t)nrhs * 16, wd,
                                  (size_t)chunk * 16, (size_t)chunk * 16, (size_t)n_out, cudaMemcpyDeviceToHost, s_out),
                "D2H copy of W") ||
            !ck(cudaEventRecord(plan->mm_ev[2][b], s_out), "cudaEventRecord"))
            break;
    }
    // drain all three streams whatever happened
    const cudaError_t e1 = cudaStreamSynchronize(s_in);
    const cudaError_t e2 = cudaStreamSynchronize(s_cmp);
    const cudaError_t e3 = cudaStreamSynchronize(s_out);
    if (rc) return rc;
    if (!ck(e1, "uhmv_matmat_host synchronize") || !ck(e2, "uhmv_matmat_host synchronize") ||
        !ck(e3, "uhmv_matmat_host synchronize"))
        return rc;
    return guard.end();
}

int uhmv_plan_info(const uhmv_plan* plan, int adjoint, int mode, int* grid, int* smem_bytes,
                   int* threads_per_cta, int* stages) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_plan_info: null plan");
    const int k = adjoint ? 1 : 0;
    const bool b = (mode == UHMV_MODE_BULK);
    if (grid) *grid = b ? plan->bulk_grid[k] : plan->fused_grid[k];
    if (smem_bytes) *smem_bytes = b ? plan->bulk_smem[k] : plan->smem[k];
    if (threads_per_cta) *threads_per_cta = b ? bulk::kThreads : kThreads;
    if (stages) *stages = b ? plan->bulk_nstage[k] : 0;
    return UHMV_OK;
}

int uhmv_plan_set_trace(uhmv_plan* plan, void* trace) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_plan_set_trace: null plan");
    plan->trace = static_cast<unsigned long long*>(trace);
    return UHMV_OK;
}

int uhmv_plan_set_profile(uhmv_plan* plan, void* counters) {
    if (!plan) return fail(UHMV_EINVAL, "uhmv_plan_set_profile: null plan");
    plan->prof = static_cast<unsigned long long*>(counters);
    return UHMV_OK;
}

int uhmv_dmma_peak(int device, double* tflops) {
    if (!tflops) return fail(UHMV_EINVAL, "uhmv_dmma_peak: null output");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* sink = nullptr;
    e = cudaMalloc(&sink, sizeof(double));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    const int grid = sms * 8, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    mrhs::dmma_peak_kernel<<<grid, 128>>>(64, sink);  // warm-up
    cudaEventRecord(a);
    mrhs::dmma_peak_kernel<<<grid, 128>>>(iters, sink);
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return cuda_fail(e, "dmma_peak_kernel");
    // 4 MMAs per iteration per warp, m16n8k16 = 16*8*16 multiply-adds = 4096 flops
    const double flops = 4096.0 * 4.0 * iters * (grid * 4.0);
    *tflops = flops / (ms * 1e-3) / 1e12;
    return UHMV_OK;
}

int uhmv_plan_destroy(uhmv_plan* plan) {
    if (plan) {
        {  // wait for the plan group's last launch (its buffers may be freed after this)
            std::lock_guard<std::mutex> g(plan->sync->mu);
            if (plan->sync->recorded) cudaEventSynchronize(plan->sync->ev);
        }
        sync_release(plan->d.ticket, plan->sync);
        drop_host_graphs(plan);
        if (plan->mm_start) cudaEventDestroy(plan->mm_start);
        if (plan->cap_stream) cudaStreamDestroy(plan->cap_stream);
        for (int i = 0; i < 3; ++i) {
            if (!plan->mm_stream[i]) continue;
            for (int b = 0; b < 2; ++b) cudaEventDestroy(plan->mm_ev[i][b]);
            cudaStreamDestroy(plan->mm_stream[i]);
        }
    }
    delete plan;
    return UHMV_OK;
}

}  // extern "C"
