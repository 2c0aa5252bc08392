// tc_wgrad.cu — tcgen05 (sm_100a) BF16 backward-weight for dilation 8.
//
//   dW[k][c][s] = sum_n sum_q X[n][c][q + 8s] * dY[n][k][q]
//
// Implicit GEMM with K = q (16 columns per MMA), M = 128 rows = T taps x CP channels
// (CP = C rounded up to a power of two >= 8, T = 128/CP), N = KP filters (K rounded up to 16):
//   A[(t,c)][kk] = X[c][q + 8(s0 + t)]     B[k][kk] = dY[k][q]     D[(t,c)][k] += A.B^T
// The X window sits in shared memory in a "q-chunk major" layout,
//   byte(c, q) = (q/8)*CP*16 + c*16 + (q%8)*2,
// produced directly by a 4-D TMA box (8 columns x CP channels x chunks). In that layout one tap
// (8 columns) is exactly CP*16 bytes = CP/8 core-matrix row groups, so the T tap-shifted copies
// of the window that form A's rows are just consecutive row groups at a uniform 128 B stride:
// no copies are made, and a different tap group is only a different start address. dY arrives
// as a 128B-swizzled K-major TMA box. Each CTA accumulates G tap groups (G*KP TMEM columns)
// over a contiguous range of (item, 16-column step) work; partials of the CTAs sharing a tap
// range are summed in a fixed order by a second kernel (deterministic; the reference sums
// per-item partials in ascending order, proj/src/conv.cpp:308-314).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace c1d {
namespace {

using namespace sm100;

constexpr int kThreads = 256;
constexpr int kMaxStages = 4;
constexpr uint32_t kTmemCols = 512;
constexpr int kLoaderThreads = 128;  // v3: warps 2, 3, 6, 7 stream X into the ring
constexpr int kW2MaxStages = 6;
constexpr int kW2MaxGrid = 1024;  // CTAs of one launch (the reduce keeps their segment counts in shared memory)
constexpr int kW2Ks = 8;  // v3: K-steps (16 columns) per pipeline stage (the default cap)
constexpr uint32_t kW2SmemBudget = 222 * 1024;  // v3 ring + stages (227 KB max per CTA, minus static + alignment)
// v3 warps: 0 dY TMA, 1 MMA issue, 2/3/6/7 X loaders, 4/5/10/11 accumulator drains (TMEM lane
// quarters 0-3), 8/9 idle
constexpr int kW2Threads = 384;
// Accumulation segments: the tensor core's FP32 accumulation into one TMEM accumulator loses
// ~1.1e-9 (norm-relative) per accumulated product with a consistent sign, so a CTA's chain over its
// whole (item, K-step) split (config 3: ~3.2k K-steps = 52k products per dW entry) drifts to ~6e-5.
// The MMA chain restarts every `seg` K-steps per accumulator copy (the first segment of a CTA is
// shortened by a CTA-dependent amount so the CTAs' drains do not all land at once). The drain
// warps copy each finished segment out of TMEM into its own slot (plain coalesced stores) and
// hand TMEM back to the MMA warp; the reduce sums the (CTA, segment) slots in a fixed order.
// Measured alternatives: red.add into one partial ran at the L2 atomic-unit rate (~48 us per
// drain at config 3); adding each slot into an L2-resident running partial between drains needs
// ~6 TB/s of extra L2 traffic at seg = 256 and stalled the MMAs behind it.
// 256 K-steps = 4096 products per chain: ~4e-6 at config 3 (vs ~6e-5 unsegmented).
constexpr int kW2SegChain = 256;
__device__ __forceinline__ int64_t w2_seg_len(int64_t seg, int nseg_done, int cta, int ks) {
    if (nseg_done > 0) return seg;
    const int64_t first = seg * (8 + (cta & 7)) / 16;  // 1/2 .. 15/16 of a segment
    return ((first + ks - 1) / ks) * ks;
}

struct WPlan {
    int cp, t, kp;
    int ks;             // MMA K-steps (16 columns each) per pipeline stage (multiple of 4)
    int stage_q;        // columns per stage = 16 * ks
    int groups_total;   // ceil(S / T)
    int roles;          // CTA roles (tap-group ranges)
    int gmax;           // groups per role (max)
    int splits;         // CTAs per role
    int x_chunks;       // q-chunks (8 columns) per X stage window
    uint32_t x_bytes, y_bytes, stage_bytes;
    int stages;
    size_t smem_bytes;
};

__host__ __device__ inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

bool make_wplan(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, WPlan* out) {
    if (d != 8 || q % 8 != 0 || q < 8) return false;
    if (c > 128 || k > 256) return false;
    if (n * c >= (int64_t{1} << 31) || n * k >= (int64_t{1} << 31)) return false;
    WPlan p{};
    p.cp = 8;
    while (p.cp < c) p.cp *= 2;
    p.t = 128 / p.cp;
    p.kp = static_cast<int>(ceil_div(k, 16) * 16);
    p.groups_total = static_cast<int>(ceil_div(s, p.t));
    const int gcap = static_cast<int>(kTmemCols) / p.kp;
    if (gcap < 1) return false;
    p.roles = static_cast<int>(ceil_div(p.groups_total, gcap));
    p.gmax = static_cast<int>(ceil_div(p.groups_total, p.roles));
    p.splits = std::max(1, num_sms() / p.roles);
    // X window per stage: stage_q new columns + the tap span of one role's groups + K overrun.
    // Bigger stages amortise the tap-span overlap that every stage re-fetches.
    bool ok = false;
    for (int ks = 16; ks >= 4; ks -= 4) {
        p.ks = ks;
        p.stage_q = 16 * ks;
        p.x_chunks = p.stage_q / 8 + p.gmax * p.t + 1;
        if (p.x_chunks > 256) continue;
        p.x_bytes = static_cast<uint32_t>(p.x_chunks * p.cp * 16);
        p.y_bytes = static_cast<uint32_t>(p.kp * p.stage_q * 2);
        const uint32_t xb = (p.x_bytes + 1023) & ~1023u;
        p.stage_bytes = xb + p.y_bytes;
        p.stages = static_cast<int>(std::min<uint32_t>(kMaxStages, (200 * 1024) / p.stage_bytes));
        if (p.stages < 2) continue;
        ok = true;
        break;
    }
    if (!ok) return false;
    const uint32_t xb = (p.x_bytes + 1023) & ~1023u;
    p.x_bytes = xb;
    p.smem_bytes = static_cast<size_t>(p.stages) * p.stage_bytes + 1024;
    *out = p;
    return true;
}

struct WParams {
    int64_t n_items, c, k, s, q, w_in;
    int64_t steps_per_item, total_steps;  // 16-column K-steps
    WPlan pl;
    float* part;  // [role-split][k][c][s]  (only this role's taps are written)
    unsigned long long* prof;  // optional per-CTA cycle counters (C1D_PROFILE=1)
};

__global__ void __launch_bounds__(kThreads, 1)
    tc_wgrad_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                    const WParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
    __shared__ uint64_t acc_done;
    __shared__ uint32_t tmem_base_s;

    const WPlan& pl = p.pl;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int role = blockIdx.x / pl.splits;
    const int split = blockIdx.x % pl.splits;
    const int g_begin = role * pl.gmax;
    const int g_count = static_cast<int>(imin(pl.gmax, pl.groups_total - g_begin));
    const int tap0 = g_begin * pl.t;  // first tap of this role
    // this CTA's K-steps: [kb, ke) of the flattened (item, step) space
    const int64_t kb = p.total_steps * split / pl.splits;
    const int64_t ke = p.total_steps * (split + 1) / pl.splits;
    const int64_t n_stages_total = [&] {
        // stages never straddle items: count per item segment
        int64_t cnt = 0, cur = kb;
        while (cur < ke) {
            const int64_t item_end = (cur / p.steps_per_item + 1) * p.steps_per_item;
            const int64_t seg_end = imin(ke, item_end);
            cnt += ceil_div(seg_end - cur, pl.ks);
            cur = seg_end;
        }
        return cnt;
    }();

    if (threadIdx.x == 0) {
        for (int s = 0; s < pl.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&acc_done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<kTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;

    if (warp == 0) {
        if (lane == 0 && g_count > 0) {
            prefetch_tmap(&xmap);
            prefetch_tmap(&ymap);
            long long t_wait = 0;
            const long long t_begin = clock64();
            int stage = 0;
            uint32_t phase = 0;
            int64_t cur = kb;
            while (cur < ke) {
                const int64_t item = cur / p.steps_per_item;
                const int64_t item_end = (item + 1) * p.steps_per_item;
                const int64_t seg_end = imin(ke, item_end);
                for (int64_t st = cur; st < seg_end; st += pl.ks) {
                    const int64_t q0 = (st - item * p.steps_per_item) * 16;  // first column of the stage
                    const long long tw = clock64();
                    mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    t_wait += clock64() - tw;
                    const uint32_t fb = smem_u32(&full[stage]);
                    mbar_arrive_expect_tx(fb, static_cast<uint32_t>(pl.x_chunks * pl.cp * 16) + pl.y_bytes);
                    uint8_t* sbase = smem + static_cast<size_t>(stage) * pl.stage_bytes;
                    // X window: q-chunks starting at (q0/8 + tap0), box (8, CP, x_chunks, 1)
                    asm volatile(
                        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                        "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(sbase)),
                        "l"(&xmap), "r"(0), "r"(0), "r"(static_cast<int32_t>(q0 / 8 + tap0)),
                        "r"(static_cast<int32_t>(item)), "r"(fb)
                        : "memory");
                    // dY boxes (64 columns, KP filters, 1 item), 128B swizzle, one per 4 K-steps
                    for (int b = 0; b < pl.ks / 4; ++b)
                        tma_load_3d(smem_u32(sbase + pl.x_bytes + static_cast<uint32_t>(b * pl.kp * 128)), &ymap,
                                    static_cast<int32_t>(q0 + 64 * b), 0, static_cast<int32_t>(item), fb);
                    if (++stage == pl.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                cur = seg_end;
            }
            if (p.prof) {
                p.prof[blockIdx.x * 8 + 0] = t_wait;
                p.prof[blockIdx.x * 8 + 1] = clock64() - t_begin;
            }
        }
    } else if (warp == 1) {
        if (g_count > 0) {
            const uint32_t idesc = make_idesc(128, static_cast<uint32_t>(pl.kp), kFmtBF16, 0, 0);
            long long t_full = 0;
            const long long t_begin = clock64();
            int stage = 0;
            uint32_t phase = 0;
            bool first = true;
            int64_t cur = kb;
            while (cur < ke) {
                const int64_t item = cur / p.steps_per_item;
                const int64_t item_end = (item + 1) * p.steps_per_item;
                const int64_t seg_end = imin(ke, item_end);
                for (int64_t st = cur; st < seg_end; st += pl.ks) {
                    const int nks = static_cast<int>(imin(pl.ks, seg_end - st));
                    const long long tf = clock64();
                    mbar_wait(smem_u32(&full[stage]), phase);
                    t_full += clock64() - tf;
                    tc_fence_after();
                    uint8_t* sbase = smem + static_cast<size_t>(stage) * pl.stage_bytes;
                    const uint64_t a0 = make_smem_desc(smem_u32(sbase), static_cast<uint32_t>(pl.cp * 16), 128,
                                                       kLayoutNone);
                    const uint64_t b0 = make_smem_desc(smem_u32(sbase + pl.x_bytes), 16, 1024, kLayoutSw128);
                    for (int ks = 0; ks < nks; ++ks) {
                        const uint64_t bdesc =
                            desc_advance(b0, static_cast<uint32_t>((ks / 4) * pl.kp * 128 + (ks % 4) * 32));
                        for (int g = 0; g < g_count; ++g) {
                            // group g starts g*T taps later = g*T q-chunks; K-step ks = 2 chunks
                            const uint64_t adesc =
                                desc_advance(a0, static_cast<uint32_t>((g * pl.t + 2 * ks) * pl.cp * 16));
                            if (elect_one())
                                mma_bf16_ss(tmem + static_cast<uint32_t>(g * pl.kp), adesc, bdesc, idesc,
                                            first ? 0u : 1u);
                            __syncwarp();
                        }
                        first = false;
                    }
                    if (elect_one()) mma_commit(smem_u32(&empty[stage]));
                    __syncwarp();
                    if (++stage == pl.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                cur = seg_end;
            }
            if (elect_one()) mma_commit(smem_u32(&acc_done));
            __syncwarp();
            if (p.prof && lane == 0) {
                p.prof[blockIdx.x * 8 + 2] = t_full;
                p.prof[blockIdx.x * 8 + 4] = clock64() - t_begin;
            }
        }
    } else if (warp >= 4) {
        // epilogue: D rows (t, c) x columns (g, k) -> partial[role-split][k][tap][c] (channel-fastest:
        // coalesced stores)
        if (g_count > 0) {
            const int quarter = warp - 4;
            const int row = quarter * 32 + lane;
            const int t = row / pl.cp, c = row % pl.cp;
            const bool have = n_stages_total > 0;
            if (have) {
                mbar_wait_sleep(smem_u32(&acc_done), 0, 1000);
                tc_fence_after();
            }
            float* dst = p.part + static_cast<int64_t>(blockIdx.x) * p.k * p.c * p.s;
            for (int g = 0; g < g_count; ++g) {
                const int64_t tap = tap0 + static_cast<int64_t>(g) * pl.t + t;
                for (int kb2 = 0; kb2 < pl.kp; kb2 += 16) {
                    uint32_t v[16];
                    if (have) {
                        tmem_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                                      static_cast<uint32_t>(g * pl.kp + kb2), v);
                        tmem_ld_wait();
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = 0;
                    }
                    if (c < p.c && tap < p.s) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int64_t kk = kb2 + j;
                            if (kk < p.k) dst[(kk * p.s + tap) * p.c + c] = __uint_as_float(v[j]);
                        }
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<kTmemCols>(tmem);
}

// dw[k][c][s] = sum over the splits of the role owning tap s, in ascending split order; e walks the
// partials' (k, tap, channel) order (coalesced reads).
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, float* __restrict__ dw, int64_t K, int64_t C,
                                    int64_t S, int t, int gmax, int splits) {
    const int64_t count = K * C * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e % C, s = (e / C) % S, k = e / (C * S);
        const int role = static_cast<int>(s / (static_cast<int64_t>(gmax) * t));
        const float* src = part + static_cast<int64_t>(role) * splits * count + e;
        float v = 0.0f;
        for (int sp = 0; sp < splits; ++sp) v += src[static_cast<int64_t>(sp) * count];
        dw[(k * C + c) * S + s] = v;
    }
}

// ============================================================================ v3
// Backward-weight with the tensor core's B operand reused by consecutive MMAs:
//   M = 128 rows = T taps x CP channels (CP = C rounded up to a power of two >= 16, T = 128/CP):
//        A[(t, c)][kk] = X[c][q + 8*(s0 + t)]         q-chunk-major X window (see v1)
//   N = P x KPw rows (KPw = K rounded up to a power of two >= 16, P <= 256/KPw copies):
//        B[(p', k)][kk] = dY[k][q - Bq*(P-1-p')]      copy p' shifted by Bq = 8*T columns
//   D[(t,c)][(p',k)] = sum_q' X[c][q' + 8*(s0 + t + T*(P-1-p'))] dY[k][q']  -> T*P taps per MMA.
// The P copies of dY are P consecutive Bq-column TMA boxes (K-major, 2*Bq-byte swizzle, or the
// plain core-matrix layout for Bq = 8), so the copy shift is a uniform row-group stride: nothing
// is loaded twice. Each CTA accumulates up to 512/N tap groups; all groups of a K-step use the
// same B (dY) and differ only in A's start address (the tap offset). The X window arrives by a
// 4-D TMA box straight into the q-chunk-major layout.
namespace {

struct W2Plan {
    int cp, t, kpw, p, bq, n;
    uint32_t swz;            // UMMA layout type for the dY operand
    int taps_per_group, groups_total, gpc, roles;
    int role_groups[64];
    int role_cta_begin[65];
    int ks, stage_q, x_chunks, nbox;
    uint32_t box_bytes, x_bytes, y_bytes, stage_bytes;
    int stages;
    size_t smem_bytes;
    int grid;
    // X ring (q-chunk-major, chunks of 8 columns x CP channels): `span` chunks of tap overlap
    // carried between consecutive stages, `kch` new chunks per stage, `xb` mirrored chunks
    int xb, span, kch, ring;
    uint32_t chunk_bytes, ring_bytes;
    int copies;  // accumulator copies per group (power of two)
    // Expanded rows (d = 1, 2, 4): X arrives as the row tensor E (rows of 8 elements at every
    // d-column start, launch_expand_rows). A ring "chunk" is then one E row per channel, i.e. a
    // column step of d: a tap is one chunk for every d, and 8 columns are ph = 8/d chunks (the
    // K-group stride). dY copies are off (P = 1): their Bq-column shift would need sub-16-B boxes.
    int ph;
    // inline expansion (d = 1, 2, 4): the loaders stage natural x columns in `raw` (raw_cols per
    // channel, 16-B cp.async pieces) and write the ring's rows themselves (no row tensor in HBM)
    int xin, raw_cols;
    uint32_t raw_bytes;
    // Channel-octet streams (xt, d = 1, 2, 4): X arrives as XT[n][c/8][w][8] (launch_to_octets), 8
    // channels x one column = one 16-B row. Each stage holds its own X window (no ring): 16
    // streams (M groups) of xt_rows rows, stream j = t*(CP/8) + o = channel octet o of copy t,
    // shifted by t*d columns (the T taps of a group stacked on M), each copy loaded by ONE 3-D TMA
    // box (256 elements x xt_nb blocks x CP/8 octets, through an overlapping view whose block
    // stride is 512 B) that lands the octets xt_rows*16 B apart. A is MN-major: K rows (columns)
    // 16 B apart, K groups 128 B apart, M groups one stream apart, so ANY column shift is a
    // start-address offset: tap group g of K-step k starts at row 16k + g*T*d. No expansion, no
    // dY copies, and the loader warps stay idle.
    int xt;
    int xt_nb;                    // 256-element blocks per stream and stage (xt_rows = 32 * xt_nb)
    uint32_t xt_x_bytes;          // X bytes per stage (16 streams)
    uint32_t stream_bytes;        // xt: stream stride in a stage (xt_rows x 16 B)
    uint32_t a_lbo, a_sbo, a_mn;  // A descriptor
    uint32_t a_ks_bytes, a_g_bytes;  // A advance per K-step / per tap group
};

bool make_w2plan(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, W2Plan* out, bool xin = false,
                 bool xt = false, int gpc_cap = 8) {
    if (q % 8 != 0 || q < 16) return false;
    if (xt ? (d < 1 || d > 64) : (d != 8 && d != 1 && d != 2 && d != 4)) return false;
    if (xin && d == 8) return false;
    if (xin && xt) return false;
    if (c > 128 || k > 128) return false;
    if (n * c >= (int64_t{1} << 31) || n * k >= (int64_t{1} << 31)) return false;
    W2Plan p{};
    p.xt = xt ? 1 : 0;
    p.ph = xt ? 1 : static_cast<int>(8 / d);  // (xt: any d)
    p.cp = 16;
    while (p.cp < c) p.cp *= 2;
    p.t = 128 / p.cp;
    p.kpw = 16;
    while (p.kpw < k) p.kpw *= 2;
    // dY copies (P > 1) shift by Bq = 8T columns, so their boxes are 8T columns wide; at T = 1 that is a
    // 16-B box, which TMA moves at ~16 B/clk (too slow to feed the MMAs: C = 128 ran 63% data-starved),
    // so T = 1 and the expanded rows run without copies and with wide dY boxes
    p.p = (d == 8 && !xt && p.t > 1) ? std::min<int>(256 / p.kpw, static_cast<int>(ceil_div(s, p.t))) : 1;
    p.n = p.p * p.kpw;
    p.bq = 8 * p.t;  // with P = 1 re-chosen per stage size below (64 / 32 / 16 columns)
    if (p.bq > 64) return false;
    p.taps_per_group = p.t * p.p;
    p.groups_total = static_cast<int>(ceil_div(s, p.taps_per_group));
    p.gpc = std::max(1, static_cast<int>(kTmemCols) / p.n);
    if (p.gpc > gpc_cap) p.gpc = gpc_cap;
    if (p.n > static_cast<int>(kTmemCols)) return false;
    if (p.gpc > p.groups_total) p.gpc = p.groups_total;
    p.roles = static_cast<int>(ceil_div(p.groups_total, p.gpc));
    if (p.roles > 64) return false;
    const int sms = num_sms();
    if (p.roles > sms) return false;
    int assigned = 0;
    for (int r = 0; r < p.roles; ++r) p.role_groups[r] = std::min(p.gpc, p.groups_total - p.gpc * r);
    p.role_cta_begin[0] = 0;
    // CTAs are split evenly across roles: every role streams the same X/dY data per K-step, and a
    // weighted split (fewer CTAs for the 1-group role) measured slower on B200.
    for (int r = 0; r < p.roles; ++r) {
        const int64_t want = static_cast<int64_t>(sms) * (r + 1) / p.roles;
        int end = static_cast<int>(std::max<int64_t>(want, assigned + 1));
        if (r == p.roles - 1) end = std::max(sms, assigned + 1);
        p.role_cta_begin[r + 1] = end;
        assigned = end;
    }
    p.grid = assigned;
    if (p.grid > kW2MaxGrid) return false;
    p.box_bytes = static_cast<uint32_t>(p.kpw * 2 * p.bq);
    // Accumulator copies (consecutive K-steps rotating over R accumulators, summed by the drain) were
    // added against a supposed ~128-cycle same-accumulator chain; that was the issuing thread, and
    // with straight-line issue one accumulator runs as fast (C = K = 15, batch 64: copies 4 / 2 / 1
    // = 106.5 / 105.5 / 104.5 us, the drain 9.2k -> 6.7k cycles), so the default is one copy.
    static const int copies_cap = [] {  // C1D_W2_COPIES: dev override of the copy cap
        const char* e = getenv("C1D_W2_COPIES");
        const int v = e ? atoi(e) : 1;
        return v == 1 || v == 2 || v == 4 ? v : 1;
    }();
    p.copies = 1;
    while (p.copies < copies_cap && p.gpc * p.n * p.copies < 256 &&
           p.gpc * p.n * p.copies * 2 <= static_cast<int>(kTmemCols))
        p.copies *= 2;
    // X lives in a ring: every stage loads only its new chunks; the window's tap span is reused.
    // Safety (a stage slot is refilled only after that slot's MMAs completed):
    //   ring >= 2*span + stages*kch   (the window a stage reads, the stages-1 stages the
    //   loaders may run ahead, and one extra fresh window when an item boundary falls in there)
    // Ring positions [0, xb) are mirrored past the end, xb = the furthest chunk one stage's MMAs
    // reach beyond the stage's first chunk, so a stage never wraps. Expanded rows take ph chunks
    // per 8 columns, so their stages shrink (fewer K-steps) until the ring fits.
    p.chunk_bytes = xt ? 16u : static_cast<uint32_t>(p.cp * 16);
    // xt: a stage's window is its 16*ks rows plus the reach of the other tap groups, (gpc-1)*T*d
    p.span = xt ? static_cast<int>(ceil_div(static_cast<int64_t>(p.gpc - 1) * p.t * d + 1, 4) * 4)
                : static_cast<int>(ceil_div(p.gpc * p.taps_per_group + p.t + p.ph, 4) * 4);
    static const int max_stages = [] {  // C1D_W2_STAGES: dev override of the stage cap
        const char* e = getenv("C1D_W2_STAGES");
        const int v = e ? atoi(e) : kW2MaxStages;
        return v >= 3 && v <= kW2MaxStages ? v : kW2MaxStages;
    }();
    bool ok = false;
    // narrow plans (one tap group per CTA) take 32-K-step stages: half the per-stage overhead (barrier
    // waits, commits, ring bookkeeping) and fewer re-loaded dY history boxes per new column
    static const int ks_env = [] {  // C1D_W2_KS: dev override of the K-steps per stage
        const char* e = getenv("C1D_W2_KS");
        return e ? atoi(e) : 0;
    }();
    const int ks_max = ks_env > 0 ? std::min(ks_env, 32) : (p.gpc == 1 && p.p > 1 ? 32 : kW2Ks);
    for (int ks = ks_max; ks >= 1 && !ok; --ks) {
        if (p.p == 1) p.bq = (16 * ks) % 64 == 0 ? 64 : ((16 * ks) % 32 == 0 ? 32 : 16);
        const int ks_unit = std::max(1, p.bq / 16);  // K-steps per dY box
        if (ks % ks_unit || (2 * ks * p.ph) % 4) continue;
        p.swz = p.bq == 64 ? kLayoutSw128 : (p.bq == 32 ? kLayoutSw64 : (p.bq == 16 ? kLayoutSw32 : kLayoutNone));
        p.box_bytes = static_cast<uint32_t>(p.kpw * 2 * p.bq);
        p.ks = ks;
        p.stage_q = 16 * p.ks;
        p.kch = xt ? 16 * p.ks : 2 * p.ks * p.ph;
        p.xb = xt ? 0 : 2 * p.ph * (p.ks - 1) + (p.gpc - 1) * p.taps_per_group + p.t + p.ph;
        p.x_chunks = p.kch + p.span;
        p.nbox = p.stage_q / p.bq + p.p - 1 + (p.bq == 8 ? 1 : 0);
        p.y_bytes = (static_cast<uint32_t>(p.nbox) * p.box_bytes + 1023) & ~1023u;
        p.stage_bytes = p.y_bytes;
        if (xt) {  // the stage's X window: 16 K-step rows x ks plus the other groups' reach
            p.xt_nb = static_cast<int>(ceil_div(p.kch + p.span, 32));
            p.stream_bytes = static_cast<uint32_t>(p.xt_nb) * 512u;
            p.xt_x_bytes = 16u * p.stream_bytes;
            p.stage_bytes = p.y_bytes + p.xt_x_bytes;
        }
        p.xin = xin ? 1 : 0;
        p.raw_cols = xin ? static_cast<int>(ceil_div(static_cast<int64_t>(d) * (p.span + p.kch) + 40, 8) * 8) : 0;
        p.raw_bytes = xin ? ((static_cast<uint32_t>(p.cp * p.raw_cols * 2) + 1023) & ~1023u) : 0u;  // one of two
        for (int st = max_stages; st >= 3; --st) {
            p.stages = st;
            p.ring = xt ? 0 : static_cast<int>(ceil_div(2 * p.span + st * p.kch, 4) * 4);
            p.ring_bytes = xt ? 0u : (((static_cast<uint32_t>(p.ring + p.xb) * p.chunk_bytes) + 1023) & ~1023u);
            if (p.ring_bytes + static_cast<uint32_t>(st) * p.stage_bytes + 2 * p.raw_bytes <= kW2SmemBudget) {
                ok = true;
                break;
            }
        }
    }
    if (!ok) return false;
    if (xt && (p.stream_bytes >= (1u << 18) || p.xt_nb > 256)) return false;  // descriptor stride / box dims
    if (xt) {
        p.a_mn = 1;
        p.a_lbo = 128;                // K groups (8 columns) are consecutive 128-B core matrices
        p.a_sbo = p.stream_bytes;     // M groups (8 rows of D) are streams
        p.a_ks_bytes = 16u * 16u;     // a K-step = 16 rows
        p.a_g_bytes = static_cast<uint32_t>(p.t * d) * 16u;
    } else {
        p.a_mn = 0;
        p.a_lbo = static_cast<uint32_t>(p.ph * p.cp * 16);
        p.a_sbo = 128;
        p.a_ks_bytes = 2u * static_cast<uint32_t>(p.ph) * p.chunk_bytes;
        p.a_g_bytes = static_cast<uint32_t>(p.taps_per_group) * p.chunk_bytes;
    }
    p.x_bytes = p.ring_bytes;
    p.smem_bytes = p.ring_bytes + static_cast<size_t>(p.stages) * p.stage_bytes + 2 * p.raw_bytes + 1024;
    *out = p;
    return true;
}

// xt plans: the widest tap-group count per CTA whose stage window (16 K-step rows plus the other
// groups' reach, (gpc-1)*T*d rows) still leaves >= 3 pipeline stages; long reaches (large T*d)
// trade roles (each re-reading X and dY) for window size
bool make_w2plan_xt(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, W2Plan* out) {
    for (int cap = 8; cap >= 1; --cap)
        if (make_w2plan(n, c, k, s, d, q, out, false, true, cap)) return true;
    return false;
}

struct W2Params {
    int64_t n_items, c, k, s, q, w_in;
    int64_t dil;
    int64_t steps_per_item, total_steps;
    int64_t seg;  // K-steps per accumulation segment (0: the whole split is one chain)
    int64_t slot_elems;  // floats per slot: K x (the role's taps) x C
    int max_segs;        // slots per CTA
    int* nseg;           // [cta]: slots this CTA wrote
    W2Plan pl;
    const uint16_t* x;  // [n][c][w_in] bf16
    float* part;        // [cta][k][c][s]
    unsigned long long* prof;
};

// One stage of MMAs: K-step ks (accumulator copy (k0 + ks) mod R) x G tap groups. Descriptors
// advance by running adds (units of 16 B) so the per-stage prologue stays a handful of uniform
// instructions; with G >= 2 the tensor pipe hides the per-K-step loop overhead.
struct W2Issue {
    uint32_t idesc, a_ks, a_g, b_k, b_box, copy_stride, cmask;
    int per_box, n, copies;
    uint32_t b_off[9];  // B descriptor offset (16-B units) of K-step ks of an 8-step block (8: the next block)
};
template <int G>
__device__ __forceinline__ void w2_issue_stage(const W2Issue& w, uint32_t tmem, uint64_t a, uint64_t b, int k0,
                                               int nks, int g_count) {
    if (G > 0 && nks % 8 == 0) {
        // full stage, straight line: every K-step's descriptors come from the stage base with
        // independent adds (no loop-carried chain), so the issuing thread keeps up with the
        // tensor pipe; a rolled loop's dependent uniform-datapath chain cost ~90-130 cycles per
        // K-step (tools/probe_mma_layouts.cu: STRAIGHT vs loop rows)
#pragma unroll 1
        for (int blk = 0; blk < nks; blk += 8) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const uint32_t kk = static_cast<uint32_t>(k0 + blk + ks);
            const uint32_t d0 = tmem + (kk & w.cmask) * w.copy_stride;
            const uint32_t acc = kk >= static_cast<uint32_t>(w.copies) ? 1u : 0u;
            const uint64_t ak = a + static_cast<uint64_t>(static_cast<uint32_t>(ks) * w.a_ks);
            const uint64_t bk = b + static_cast<uint64_t>(w.b_off[ks]);
#pragma unroll
            for (int g = 0; g < (G > 0 ? G : 1); ++g)
                mma_bf16_ss(d0 + static_cast<uint32_t>(g * w.n), ak + static_cast<uint64_t>(g * w.a_g), bk, w.idesc, acc);
        }
        a += static_cast<uint64_t>(8u * w.a_ks);
        b += static_cast<uint64_t>(w.b_off[8]);
        }
        return;
    }
    int inbox = 0;
#pragma unroll 1
    for (int ks = 0; ks < nks; ++ks) {
        const int kk = k0 + ks;
        const uint32_t d0 = tmem + (static_cast<uint32_t>(kk) & w.cmask) * w.copy_stride;
        const uint32_t acc = kk >= w.copies ? 1u : 0u;
        if (G > 0) {
#pragma unroll
            for (int g = 0; g < G; ++g)
                mma_bf16_ss(d0 + static_cast<uint32_t>(g * w.n), a + static_cast<uint64_t>(g * w.a_g), b, w.idesc, acc);
        } else {
#pragma unroll 1
            for (int g = 0; g < g_count; ++g)
                mma_bf16_ss(d0 + static_cast<uint32_t>(g * w.n), a + static_cast<uint64_t>(g * w.a_g), b, w.idesc, acc);
        }
        a += w.a_ks;
        if (++inbox == w.per_box) {
            inbox = 0;
            b += w.b_box;
        } else {
            b += w.b_k;
        }
    }
}

// Inline rows for the X ring: positions p0 .. p0+RG-1 of channel c (position p = natural columns
// D*p .. D*p+7 past the stage's first column; raw element K0 + D*(p - p0) of the loaded words).
template <int D, int K0>
__device__ __forceinline__ void w2_expand_group(uint32_t rc, int p0, int npos, uint32_t ring_s, int v_pos, int ring,
                                                int xb, uint32_t chunk_bytes, uint32_t mirror_bytes, int c) {
    constexpr int RG = D == 4 ? 4 : 8;
    constexpr int NW = ((K0 + D * (RG - 1) + 8 + 7) / 8) * 4;
    const uint32_t src = rc + static_cast<uint32_t>(D * p0 * 2);
    uint32_t w[NW];
#pragma unroll
    for (int i = 0; i < NW; i += 4)
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[i]), "=r"(w[i + 1]), "=r"(w[i + 2]), "=r"(w[i + 3])
                     : "r"(src + static_cast<uint32_t>(i * 4)));
#pragma unroll
    for (int j = 0; j < RG; ++j) {
        if (p0 + j >= npos) break;
        const int o = K0 + D * j;
        uint32_t v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            v[i] = (o & 1) ? __funnelshift_r(w[(o >> 1) + i], w[(o >> 1) + i + 1], 16) : w[(o >> 1) + i];
        int slot = v_pos + p0 + j;
        if (slot >= ring) slot -= ring;
        const uint32_t dst = ring_s + static_cast<uint32_t>(slot) * chunk_bytes + static_cast<uint32_t>(c) * 16u;
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
                     : "memory");
        if (slot < xb)
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + mirror_bytes), "r"(v[0]), "r"(v[1]),
                         "r"(v[2]), "r"(v[3])
                         : "memory");
    }
}

template <int D>
__device__ __forceinline__ void w2_expand_d(int off, uint32_t rc, int p0, int npos, uint32_t ring_s, int v_pos, int ring,
                                            int xb, uint32_t chunk_bytes, uint32_t mirror_bytes, int c) {
#define W2X(K) w2_expand_group<D, K>(rc, p0, npos, ring_s, v_pos, ring, xb, chunk_bytes, mirror_bytes, c)
    switch (off) {
        case 0: W2X(0); break;
        case 1: W2X(1); break;
        case 2: W2X(2); break;
        case 3: W2X(3); break;
        case 4: W2X(4); break;
        case 5: W2X(5); break;
        case 6: W2X(6); break;
        default: W2X(7); break;
    }
#undef W2X
}

template <int kLean>
__global__ void __launch_bounds__(kW2Threads, 1)
    tc_wgrad2_kernel(const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap xmap,
                     const W2Params p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[kW2MaxStages], empty[kW2MaxStages];
    __shared__ uint64_t acc_full, acc_empty;
    __shared__ uint32_t tmem_base_s;

    const W2Plan& pl = p.pl;
    // kLean: the dilation-8 natural ring plan (no channel-octet streams, no inline expansion, one
    // accumulator copy); folding those plan fields drops the other feeds' code from the hot loops
    const int pl_xt = kLean ? 0 : pl.xt, pl_xin = kLean ? 0 : pl.xin, pl_ph = kLean ? 1 : pl.ph;
    const int pl_copies = kLean ? 1 : pl.copies, pl_raw_cols = kLean ? 0 : pl.raw_cols;
    const uint32_t pl_a_mn = kLean ? 0u : pl.a_mn, pl_raw_bytes = kLean ? 0u : pl.raw_bytes;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    int role = 0;
    while (role + 1 < pl.roles && static_cast<int>(blockIdx.x) >= pl.role_cta_begin[role + 1]) ++role;
    const int split = blockIdx.x - pl.role_cta_begin[role];
    const int splits = pl.role_cta_begin[role + 1] - pl.role_cta_begin[role];
    const int g_count = pl.role_groups[role];
    const int tap0 = pl.gpc * role * pl.taps_per_group;
    const int64_t kb = p.total_steps * split / splits;
    const int64_t ke = p.total_steps * (split + 1) / splits;

    if (threadIdx.x == 0) {
        for (int s = 0; s < pl.stages; ++s) {
            mbar_init(&full[s], pl_xt ? 1 : 1 + kLoaderThreads);  // dY (+ xt: X) TMA tx bytes + every X loader thread
            mbar_init(&empty[s], 1);
        }
        mbar_init(&acc_full, 1);
        mbar_init(&acc_empty, 4);  // one arrival per drain warp
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<kTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    // PDL: everything above overlapped the previous kernel; global memory only from here on (no
    // early trigger: the reduce's many small CTAs would sit on the SMs beside this kernel)
    pdl_wait();
    const int64_t back = static_cast<int64_t>(pl.p - 1) * pl.bq;  // dY history columns per stage

    if (warp == 0) {
        if (lane == 0) {
            prefetch_tmap(&ymap);
            if (pl_xt) prefetch_tmap(&xmap);
            const int octets = static_cast<int>((p.c + 7) / 8);
            long long tw_sum = 0;
            const long long tb = clock64();
            int stage = 0;
            uint32_t phase = 0;
            int64_t cur = kb;
            while (cur < ke) {
                const int64_t item = cur / p.steps_per_item;
                const int64_t seg_end = imin(ke, (item + 1) * p.steps_per_item);
                for (int64_t st = cur; st < seg_end; st += pl.ks) {
                    const int64_t q0 = (st - item * p.steps_per_item) * 16;
                    const long long tw = clock64();
                    mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    tw_sum += clock64() - tw;
                    const uint32_t fb = smem_u32(&full[stage]);
                    mbar_arrive_expect_tx(fb, static_cast<uint32_t>(pl.nbox) * pl.box_bytes + (pl_xt ? pl.xt_x_bytes : 0u));
                    uint8_t* sbase = smem + pl.ring_bytes + static_cast<size_t>(stage) * pl.stage_bytes;
                    for (int b = 0; b < pl.nbox; ++b)
                        tma_load_3d(smem_u32(sbase + static_cast<uint32_t>(b) * pl.box_bytes), &ymap,
                                    static_cast<int32_t>(q0 - back + static_cast<int64_t>(b) * pl.bq), 0,
                                    static_cast<int32_t>(item), fb);
                    if (pl_xt) {
                        // copy t: columns q0 + tap0*d + t*d .. of every octet, one box
                        const int64_t col0 = q0 + static_cast<int64_t>(tap0) * p.dil;
                        const uint32_t xs = smem_u32(sbase + pl.y_bytes);
                        for (int t = 0; t < pl.t; ++t)
                            tma_load_3d(xs + static_cast<uint32_t>(t * (pl.cp / 8)) * pl.stream_bytes, &xmap,
                                        static_cast<int32_t>(8 * (col0 + static_cast<int64_t>(t) * p.dil)), 0,
                                        static_cast<int32_t>(item * octets), fb);
                    }
                    if (++stage == pl.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                cur = seg_end;
            }
            if (p.prof) {
                p.prof[blockIdx.x * 8 + 0] = tw_sum;
                p.prof[blockIdx.x * 8 + 1] = clock64() - tb;
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = make_idesc(128, static_cast<uint32_t>(pl.n), kFmtBF16, pl_a_mn, 0);
        // B (dY) descriptor: swizzled K-major rows of 2*Bq bytes (8-row atoms), or for Bq = 8 the
        // plain core-matrix layout with K-chunks one box apart.
        const uint32_t b_sbo = pl.bq == 8 ? 128u : 16u * static_cast<uint32_t>(pl.bq);
        const uint32_t b_lbo = pl.bq == 8 ? pl.box_bytes : 16u;
        long long tf_sum = 0, ti_sum = 0, tc_sum = 0, te_sum = 0;
        const long long tb = clock64();
        int stage = 0;
        uint32_t phase = 0;
        // descriptor steps in units of 16 B. B (dY): Bq = 8 -> a K-step spans two boxes; else
        // 16/Bq K-steps (32 B each) per box
        W2Issue wi;
        wi.idesc = idesc;
        wi.a_ks = pl.a_ks_bytes >> 4;
        wi.a_g = pl.a_g_bytes >> 4;
        if (pl.bq == 8) {
            wi.per_box = 1;
            wi.b_box = (2u * pl.box_bytes) >> 4;
            wi.b_k = 0;
        } else {
            wi.per_box = pl.bq / 16;
            wi.b_k = 32u >> 4;
            wi.b_box = (pl.box_bytes - static_cast<uint32_t>(wi.per_box - 1) * 32u) >> 4;
        }
        wi.copy_stride = static_cast<uint32_t>(pl.gpc * pl.n);
        wi.cmask = static_cast<uint32_t>(pl_copies - 1);
        wi.n = pl.n;
        wi.copies = pl_copies;
#pragma unroll
        for (int ks = 0; ks < 9; ++ks)
            wi.b_off[ks] = static_cast<uint32_t>(ks / wi.per_box) * (wi.b_box + static_cast<uint32_t>(wi.per_box - 1) * wi.b_k) +
                           static_cast<uint32_t>(ks % wi.per_box) * wi.b_k;
        int kdone = 0;  // K-steps issued so far
        int seg_base = 0;  // kdone at the start of the current accumulation segment
        int nseg_mma = 0;
        uint32_t eph = 0;
        // ring bookkeeping mirrors the loaders': a segment (item) starts a fresh window of
        // span + kch chunks at v_pos; each later stage appends kch chunks and the window start
        // moves by kch
        int v_pos = 0, cur_pos = 0;
        int64_t cur = kb;
        while (cur < ke) {
            const int64_t item = cur / p.steps_per_item;
            const int64_t seg_end = imin(ke, (item + 1) * p.steps_per_item);
            bool seg_first = true;
            for (int64_t st = cur; st < seg_end; st += pl.ks) {
                const int nks = static_cast<int>(imin(pl.ks, seg_end - st));
                if (seg_first) {
                    cur_pos = v_pos;
                    v_pos += pl.span + pl.kch;
                    seg_first = false;
                } else {
                    cur_pos += pl.kch;
                    if (cur_pos >= pl.ring) cur_pos -= pl.ring;
                    v_pos += pl.kch;
                }
                if (v_pos >= pl.ring) v_pos -= pl.ring;
                if (p.seg > 0 && kdone - seg_base >= w2_seg_len(p.seg, nseg_mma, blockIdx.x, pl.ks)) {
                    // segment boundary: hand the accumulators to the drain warps, restart the chain
                    if (elect_one()) mma_commit(smem_u32(&acc_full));
                    __syncwarp();
                    const long long te = clock64();
                    mbar_wait(smem_u32(&acc_empty), eph);
                    te_sum += clock64() - te;
                    eph ^= 1;
                    tc_fence_after();
                    seg_base = kdone;
                    ++nseg_mma;
                }
                const long long tf = clock64();
                mbar_wait(smem_u32(&full[stage]), phase);
                tf_sum += clock64() - tf;
                tc_fence_after();
                uint8_t* sbase = smem + pl.ring_bytes + static_cast<size_t>(stage) * pl.stage_bytes;
                // A (X) of K-step ks, group g starts at chunk lo + 2ks + g*tpg: ring position
                const int stage_pos = cur_pos;  // ring position of chunk `lo`
                const uint64_t ax0 = make_smem_desc(smem_u32(smem), pl.a_lbo, pl.a_sbo, kLayoutNone);
                const uint64_t by0 = make_smem_desc(smem_u32(sbase), b_lbo, b_sbo, pl.swz);
                // One elected lane issues the whole stage. The ring mirror keeps every address of
                // the stage wrap-free, so a full stage is a straight-line run of MMAs.
                const long long ti = clock64();
                if (elect_one()) {
                    // xt: the stage's own window (rows from its first column); else the ring
                    const uint64_t a_st = pl_xt ? make_smem_desc(smem_u32(sbase + pl.y_bytes), pl.a_lbo, pl.a_sbo, kLayoutNone)
                                                : desc_advance(ax0, static_cast<uint32_t>(stage_pos) * pl.chunk_bytes);
                    const int k0 = kdone - seg_base;  // K-step within the segment (copy rotation, init)
                    switch (g_count) {
                        case 1: w2_issue_stage<1>(wi, tmem, a_st, by0, k0, nks, 1); break;
                        case 2: w2_issue_stage<2>(wi, tmem, a_st, by0, k0, nks, 2); break;
                        case 3: w2_issue_stage<3>(wi, tmem, a_st, by0, k0, nks, 3); break;
                        case 4: w2_issue_stage<4>(wi, tmem, a_st, by0, k0, nks, 4); break;
                        default: w2_issue_stage<0>(wi, tmem, a_st, by0, k0, nks, g_count);
                    }
                }
                kdone += nks;
                __syncwarp();
                const long long tc = clock64();
                ti_sum += tc - ti;
                if (elect_one()) mma_commit(smem_u32(&empty[stage]));
                __syncwarp();
                tc_sum += clock64() - tc;
                if (++stage == pl.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            cur = seg_end;
        }
        if (elect_one()) mma_commit(smem_u32(&acc_full));  // the last segment
        __syncwarp();
        if (p.prof && lane == 0) {
            p.prof[blockIdx.x * 8 + 2] = tf_sum;
            p.prof[blockIdx.x * 8 + 3] = ti_sum;
            p.prof[blockIdx.x * 8 + 5] = tc_sum;
            p.prof[blockIdx.x * 8 + 4] = clock64() - tb;
            p.prof[blockIdx.x * 8 + 6] = te_sum;
        }
    }
    if ((warp == 2 || warp == 3 || warp == 6 || warp == 7) && pl_xt) {
        // xt: the producer's TMA boxes bring X; nothing to load here
    } else if ((warp == 2 || warp == 3 || warp == 6 || warp == 7) && pl_xin) {
        // ---- X loaders, inline expanded rows: the natural columns of a stage's positions land in
        // one of two `raw` buffers (16-B cp.async pieces, issued one stage ahead), then the loaders
        // write the ring rows (position p = the 8 elements at column D*p), proxy fence, arrive
        const int lt = (warp < 4 ? warp - 2 : warp - 4) * 32 + lane;  // 0..127
        const int d = 8 / pl_ph;
        const int cshift = __ffs(pl.cp) - 1;
        const uint32_t ring_s = smem_u32(smem);
        const uint32_t raw_s0 = ring_s + pl.ring_bytes + static_cast<uint32_t>(pl.stages) * pl.stage_bytes;
        const uint32_t mirror_bytes = static_cast<uint32_t>(pl.ring) * pl.chunk_bytes;
        const int pieces_per_c = pl_raw_cols / 8;
        const int rg = d == 4 ? 4 : 8;
        // the loaders' stage sequence: (item, first position, positions) per stage
        struct XStage {
            int64_t item, first;
            int n;
        };
        int64_t it_cur = kb, it_st = kb, it_seg_end = kb, it_next = 0;
        bool it_seg_first = true;
        auto next_stage = [&](XStage* xs) -> bool {
            if (it_st >= it_seg_end) {  // next item segment
                it_cur = it_seg_end;
                if (it_cur >= ke) return false;
                const int64_t item = it_cur / p.steps_per_item;
                it_seg_end = imin(ke, (item + 1) * p.steps_per_item);
                it_st = it_cur;
                it_seg_first = true;
            }
            const int64_t item = it_st / p.steps_per_item;
            const int64_t q0 = (it_st - item * p.steps_per_item) * 16;
            xs->item = item;
            xs->first = it_seg_first ? q0 * pl_ph / 8 + tap0 : it_next;
            xs->n = it_seg_first ? pl.span + pl.kch : pl.kch;
            it_seg_first = false;
            it_next = xs->first + xs->n;
            it_st += pl.ks;
            return true;
        };
        auto load_raw = [&](const XStage& xs, uint32_t raw_s) {
            const uint16_t* xi = p.x + xs.item * p.c * p.w_in;
            const int64_t col0 = (static_cast<int64_t>(d) * xs.first) & ~int64_t{7};
            for (int i = lt; i < pl.cp * pieces_per_c; i += kLoaderThreads) {
                const int c = i & (pl.cp - 1), j = i >> cshift;
                const int64_t col = col0 + 8 * j;
                const bool valid = c < p.c && col < p.w_in;
                cp_async16_zfill(raw_s + static_cast<uint32_t>((c * pl_raw_cols + 8 * j) * 2),
                                 valid ? xi + static_cast<int64_t>(c) * p.w_in + col : p.x, valid);
            }
            cp_async_commit();
        };
        it_seg_end = kb;
        it_st = kb;
        XStage cur_s, nxt_s;
        bool have = next_stage(&cur_s);
        if (have) load_raw(cur_s, raw_s0);
        int stage = 0, rb = 0;
        uint32_t phase = 0;
        int v_pos = 0;
        while (have) {
            const bool have_next = next_stage(&nxt_s);
            if (have_next) load_raw(nxt_s, raw_s0 + static_cast<uint32_t>(rb ^ 1) * pl_raw_bytes);
            mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
            if (have_next)
                cp_async_wait_group<1>();  // this stage's raw has landed (the next one may be in flight)
            else
                cp_async_wait_group<0>();
            asm volatile("bar.sync 3, 128;" ::: "memory");
            const uint32_t raw_s = raw_s0 + static_cast<uint32_t>(rb) * pl_raw_bytes;
            const int64_t cfirst = static_cast<int64_t>(d) * cur_s.first;
            const int off = static_cast<int>(cfirst & 7);
            const int ngroups = (cur_s.n + rg - 1) / rg;
            for (int i = lt; i < pl.cp * ngroups; i += kLoaderThreads) {
                const int c = i & (pl.cp - 1), g = i >> cshift;
                const uint32_t rc = raw_s + static_cast<uint32_t>(c * pl_raw_cols * 2);
                if (d == 1)
                    w2_expand_d<1>(off, rc, g * rg, cur_s.n, ring_s, v_pos, pl.ring, pl.xb, pl.chunk_bytes, mirror_bytes, c);
                else if (d == 2)
                    w2_expand_d<2>(off, rc, g * rg, cur_s.n, ring_s, v_pos, pl.ring, pl.xb, pl.chunk_bytes, mirror_bytes, c);
                else
                    w2_expand_d<4>(off, rc, g * rg, cur_s.n, ring_s, v_pos, pl.ring, pl.xb, pl.chunk_bytes, mirror_bytes, c);
            }
            fence_async_smem();  // generic-proxy ring rows -> the tensor core
            mbar_arrive(smem_u32(&full[stage]));
            asm volatile("bar.sync 3, 128;" ::: "memory");  // raw buffer rb is free again
            v_pos += cur_s.n;
            if (v_pos >= pl.ring) v_pos -= pl.ring;
            if (++stage == pl.stages) {
                stage = 0;
                phase ^= 1;
            }
            rb ^= 1;
            cur_s = nxt_s;
            have = have_next;
        }
    } else if (warp == 2 || warp == 3 || warp == 6 || warp == 7) {
        // ---- X loaders (warps 2, 3, 6, 7: the sub-partitions of the TMA and MMA warps stay free
        // of their issue load): 16-byte cp.async pieces straight from the [n][c][w] rows into the
        // q-chunk-major ring. One warp instruction moves 8 channels x 4 chunks: 64 contiguous bytes
        // per channel row in global, one 128-byte smem row per chunk. (TMA moves 16-byte-wide boxes
        // at ~16 B/clk/SM, below what the MMAs consume.)
        const int wl = warp < 4 ? warp - 2 : warp - 4;  // 0..3
        const int c_lo = lane & 7, j_lo = (lane >> 3) & 3;
        const int cshift = __ffs(pl.cp / 8) - 1;  // CP/8 channel groups (power of two)
        const int cmask_g = pl.cp / 8 - 1;
        const uint32_t ring_s = smem_u32(smem);
        const uint32_t mirror_bytes = static_cast<uint32_t>(pl.ring) * pl.chunk_bytes;
        const int64_t w_chunks = p.w_in / 8;
        int stage = 0;
        uint32_t phase = 0;
        int v_pos = 0;  // ring position of the next chunk loaded
        int64_t cur = kb;
        while (cur < ke) {
            const int64_t item = cur / p.steps_per_item;
            const int64_t seg_end = imin(ke, (item + 1) * p.steps_per_item);
            const uint16_t* xi = p.x + item * p.c * p.w_in;
            bool seg_first = true;
            int64_t next_chunk = 0;
            for (int64_t st = cur; st < seg_end; st += pl.ks) {
                const int64_t q0 = (st - item * p.steps_per_item) * 16;
                mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                const int64_t first_chunk = seg_first ? q0 * pl_ph / 8 + tap0 : next_chunk;
                const int nchunks = seg_first ? pl.span + pl.kch : pl.kch;
                seg_first = false;
                next_chunk = first_chunk + nchunks;
                const int64_t lim = w_chunks - first_chunk;  // chunks jl < lim exist
                const uint16_t* src0 = xi + first_chunk * 8;
                const int rows = (nchunks * pl.cp) >> 5;
                for (int r = wl; r < rows; r += 4) {
                    const int c = ((r & cmask_g) << 3) + c_lo;
                    const int jl = ((r >> cshift) << 2) + j_lo;
                    int pos = v_pos + jl;
                    if (pos >= pl.ring) pos -= pl.ring;
                    const bool valid = c < p.c && jl < lim;
                    const uint16_t* src = valid ? src0 + static_cast<int64_t>(c) * p.w_in + jl * 8 : p.x;
                    const uint32_t dst = ring_s + static_cast<uint32_t>(pos) * pl.chunk_bytes + static_cast<uint32_t>(c) * 16u;
                    cp_async16_zfill(dst, src, valid);
                    if (pos < pl.xb) cp_async16_zfill(dst + mirror_bytes, src, valid);
                }
                // the stage's full barrier counts this thread's arrival once its pieces have landed
                cp_async_mbar_arrive_noinc(smem_u32(&full[stage]));
                v_pos += nchunks;
                if (v_pos >= pl.ring) v_pos -= pl.ring;
                if (++stage == pl.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            cur = seg_end;
        }
        cp_async_wait_group<0>();
    }
    if (warp == 4 || warp == 5 || warp == 10 || warp == 11) {
        // ---- drains: D rows (t, c) x columns (p', k) -> slot[cta][j][k][tap - tap0][c] (c fastest:
        // a warp's 32 lanes are consecutive channels, so every store is one coalesced 128-B line)
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int t = row / pl.cp, c = row % pl.cp;
        const int role_taps = pl.gpc * pl.taps_per_group;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const int kshift = __ffs(pl.kpw) - 1;  // KPw is a power of two >= 16: a 16-column chunk is
        const int64_t kstride = static_cast<int64_t>(role_taps) * p.c;  // one (copy, filter run)
        long long td_sum = 0;
        // store 16 drained columns starting at col0 of group g
        auto put16 = [&](float* dst, int g, int col0, const uint32_t (&v)[16]) {
            if (c >= p.c) return;
            const int pp = col0 >> kshift, kk0 = col0 & (pl.kpw - 1);
            const int tap = g * pl.taps_per_group + t + pl.t * (pl.p - 1 - pp);
            if (tap0 + tap >= p.s || kk0 >= p.k) return;
            float* base = dst + (static_cast<int64_t>(kk0) * role_taps + tap) * p.c + c;
            const int kn = static_cast<int>(imin(16, p.k - kk0));
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < kn) base[j * kstride] = __uint_as_float(v[j]);
        };
        auto drain = [&](int64_t seg_k, int jslot, uint32_t parity) {
            float* dst = p.part + (static_cast<int64_t>(blockIdx.x) * p.max_segs + jslot) * p.slot_elems;
            mbar_wait_sleep(smem_u32(&acc_full), parity, 128);
            tc_fence_after();
            const long long td = clock64();
            // copies this segment wrote (a short segment leaves the rest stale); order 0 + 1 + ...
            const int used = static_cast<int>(imin(pl_copies, seg_k));
            for (int g = 0; g < g_count; ++g) {
                int col0 = 0;
                if (used == 1) {  // four TMEM loads in flight per wait
                    for (; col0 + 64 <= pl.n; col0 += 64) {
                        uint32_t v0[16], v1[16], v2[16], v3[16];
                        const uint32_t a0 = lane_base + static_cast<uint32_t>(g * pl.n + col0);
                        tmem_ld16(a0, v0);
                        tmem_ld16(a0 + 16, v1);
                        tmem_ld16(a0 + 32, v2);
                        tmem_ld16(a0 + 48, v3);
                        tmem_ld_wait();
                        put16(dst, g, col0, v0);
                        put16(dst, g, col0 + 16, v1);
                        put16(dst, g, col0 + 32, v2);
                        put16(dst, g, col0 + 48, v3);
                    }
                }
                for (; col0 < pl.n; col0 += 16) {
                    uint32_t v[16];
                    tmem_ld16(lane_base + static_cast<uint32_t>(g * pl.n + col0), v);
                    tmem_ld_wait();
                    for (int r = 1; r < used; ++r) {
                        uint32_t u[16];
                        tmem_ld16(lane_base + static_cast<uint32_t>((r * pl.gpc + g) * pl.n + col0), u);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(u[j]));
                    }
                    put16(dst, g, col0, v);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&acc_empty));
            td_sum += clock64() - td;
        };
        int nseg = 0;
        if (kb < ke) {
            // the MMA warp's segmentation, replayed
            int64_t kd = 0, sb = 0;
            for (int64_t cur = kb; cur < ke;) {
                const int64_t item = cur / p.steps_per_item;
                const int64_t seg_end = imin(ke, (item + 1) * p.steps_per_item);
                for (int64_t st = cur; st < seg_end; st += pl.ks) {
                    if (p.seg > 0 && kd - sb >= w2_seg_len(p.seg, nseg, blockIdx.x, pl.ks)) {
                        drain(kd - sb, nseg, static_cast<uint32_t>(nseg & 1));
                        ++nseg;
                        sb = kd;
                    }
                    kd += imin(pl.ks, seg_end - st);
                }
                cur = seg_end;
            }
            drain(kd - sb, nseg, static_cast<uint32_t>(nseg & 1));
            ++nseg;
        }
        if (kb >= ke && c < p.c) {  // no work: a zero slot 0 (the one-slot reduce reads every CTA's)
            float* dst = p.part + static_cast<int64_t>(blockIdx.x) * p.max_segs * p.slot_elems;
            for (int g = 0; g < g_count; ++g)
                for (int col0 = 0; col0 < pl.n; col0 += 16) {
                    const uint32_t z[16] = {0};
                    put16(dst, g, col0, z);
                }
        }
        if (warp == 4 && lane == 0) {
            p.nseg[blockIdx.x] = nseg;  // 0: no work (slot 0 holds zeros)
            if (p.prof) p.prof[blockIdx.x * 8 + 7] = td_sum;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<kTmemCols>(tmem);
}

// dw = the fixed-order sum over the role's CTAs (ascending) and each CTA's segment slots (ascending)
// of slot[cta][j][k][tap - tap0][c]; the sum lands at dw[(k*C + c)*S + s] (KCS). Entries are taken
// in (k, s, c) order so a warp reads consecutive channels (coalesced). A block covers 64 outputs x
// 4 CTA quarters: each thread sums its quarter in order (eight loads in flight), then the four
// quarter sums are added in order (fixed shape, deterministic).
__global__ void __launch_bounds__(256) wgrad2_reduce_kernel(const float* __restrict__ part, const int* __restrict__ nseg,
                                                            float* __restrict__ dw, int64_t K, int64_t C, int64_t S,
                                                            int max_segs, int64_t slot_elems, const W2Plan pl) {
    __shared__ float red[4][64];
    __shared__ int ns_s[kW2MaxGrid];
    pdl_trigger();
    pdl_wait();
    if (max_segs > 1)
        for (int i = threadIdx.x; i < pl.grid; i += blockDim.x) ns_s[i] = __ldg(nseg + i);
    __syncthreads();
    // 32-bit index math (K*C*S < 2^31): 64-bit divisions made this kernel issue-bound (~100 us at
    // config 1's 148 CTA partials)
    const uint32_t count = static_cast<uint32_t>(K * C * S);
    const uint32_t cc = static_cast<uint32_t>(C), ss = static_cast<uint32_t>(S);
    const uint32_t e = blockIdx.x * 64u + (threadIdx.x % 64u);
    const int quarter = threadIdx.x / 64;
    const uint32_t role_taps = static_cast<uint32_t>(pl.gpc * pl.taps_per_group);
    float v = 0.0f;
    uint32_t c = 0, s = 0, k = 0;
    if (e < count) {
        c = e % cc;
        const uint32_t ks = e / cc;
        s = ks % ss;
        k = ks / ss;
        const uint32_t role = s / role_taps;
        const int64_t idx = static_cast<int64_t>((k * role_taps + (s - role * role_taps)) * cc + c);
        const int b0 = pl.role_cta_begin[role], b1 = pl.role_cta_begin[role + 1];
        const int n = b1 - b0;
        const int lo = b0 + n * quarter / 4, hi = b0 + n * (quarter + 1) / 4;
        if (max_segs == 1) {  // one slot per CTA, always written (zeros for a CTA without work)
            for (int bb = lo; bb < hi; bb += 16) {
                float t[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) t[j] = bb + j < hi ? __ldg(part + static_cast<int64_t>(bb + j) * slot_elems + idx) : 0.0f;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (bb + j < hi) v += t[j];
            }
        } else {
            // the (CTA, segment) slots in order, 16 loads in flight: the segment counts come from
            // shared memory (a dependent global load of each CTA's count before its slots made this
            // loop latency-bound: ~55 us at config 1 in FP32)
            int bb = lo, j = 0;
            while (bb < hi && ns_s[bb] == 0) ++bb;
            while (bb < hi) {
                float t[16];
                int cnt = 0;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    t[u] = 0.0f;
                    if (bb < hi) {
                        t[u] = __ldg(part + (static_cast<int64_t>(bb) * max_segs + j) * slot_elems + idx);
                        ++cnt;
                        if (++j == ns_s[bb]) {
                            j = 0;
                            ++bb;
                            while (bb < hi && ns_s[bb] == 0) ++bb;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    if (u < cnt) v += t[u];
            }
        }
    }
    red[quarter][threadIdx.x % 64] = v;
    __syncthreads();
    if (threadIdx.x < 64 && e < count)
        dw[(static_cast<int64_t>(k) * C + c) * S + s] =
            ((red[0][threadIdx.x] + red[1][threadIdx.x]) + red[2][threadIdx.x]) + red[3][threadIdx.x];
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

}  // namespace

namespace {
// Segment bookkeeping of a v3 launch (shared by the workspace sizing and the launch).
struct W2Seg {
    int64_t steps_per_item, total_steps, seg, slot_elems;
    int max_segs;
    size_t part_bytes, nseg_bytes;
};
W2Seg w2_segments(const W2Plan& pl, int64_t n, int64_t c, int64_t k, int64_t q) {
    W2Seg r{};
    // reduction columns q in [0, Q + (P-1)*Bq): copy p' reaches (P-1-p')*Bq columns back
    r.steps_per_item = ceil_div(q + static_cast<int64_t>(pl.p - 1) * pl.bq, 16);
    r.total_steps = n * r.steps_per_item;
    static const int64_t seg_env = [] {  // C1D_W2_SEG: dev override of kW2SegChain (0 = off)
        const char* e = getenv("C1D_W2_SEG");
        return e ? static_cast<int64_t>(atoll(e)) : int64_t{-1};
    }();
    // segmented chains only in the exact-accumulation mode (FP32, or C1D_FLAG_EXACT_ACCUM)
    const int64_t seg_chain = !exact_accum() ? 0 : (seg_env >= 0 ? seg_env : static_cast<int64_t>(kW2SegChain));
    // segment length in K-steps: kW2SegChain per accumulator copy, rounded up to whole stages
    r.seg = seg_chain > 0 ? ceil_div(seg_chain * pl.copies, pl.ks) * pl.ks : 0;
    int64_t longest = 0;  // the longest CTA split (K-steps)
    for (int ro = 0; ro < pl.roles; ++ro)
        longest = std::max<int64_t>(longest, ceil_div(r.total_steps, pl.role_cta_begin[ro + 1] - pl.role_cta_begin[ro]));
    // segments of >= seg K-steps after a first one of >= seg/2: at most (longest - seg/2)/seg + 2
    r.max_segs = r.seg > 0 ? static_cast<int>(std::max<int64_t>(0, longest - r.seg / 2) / r.seg + 2) : 1;
    r.slot_elems = k * c * static_cast<int64_t>(pl.gpc) * pl.taps_per_group;
    r.part_bytes = (sizeof(float) * static_cast<size_t>(pl.grid) * r.max_segs * r.slot_elems + 255) & ~size_t{255};
    r.nseg_bytes = sizeof(int) * static_cast<size_t>(pl.grid);
    return r;
}

cudaError_t launch_v2(const uint16_t* x_bf16, const uint16_t* dy_bf16, float* dw_kcs, void* workspace, int64_t n,
                      int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, const W2Plan& pl, cudaStream_t stream,
                      int64_t x_w) {
    auto encode = encode_fn();
    if (!encode) return cudaErrorNotSupported;
    const int64_t w_in = x_w > 0 ? x_w : q + d * (s - 1);
    CUtensorMap ymap;
    if ((reinterpret_cast<uintptr_t>(x_bf16) & 15u) || (!pl.xt && w_in % 8)) return cudaErrorInvalidValue;
    {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(q), static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(n)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(q) * 2, static_cast<cuuint64_t>(k * q) * 2};
        const cuuint32_t box[3] = {static_cast<cuuint32_t>(pl.bq), static_cast<cuuint32_t>(pl.kpw), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUtensorMapSwizzle sw =
            pl.bq == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                        : (pl.bq == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : (pl.bq == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                                                   : CU_TENSOR_MAP_SWIZZLE_NONE));
        if (encode(&ymap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(dy_bf16), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    CUtensorMap xmap = ymap;  // unused unless xt
    if (pl.xt) {
        // XT[n][o][u][8] as (element e of the stream, 256-element block j, stream n*octets + o): element
        // (e, j, r) at r*rows*16 + j*512 + e*2 -- an overlapping view, so a box of 256 x nb x CP/8 is
        // nb*256 consecutive elements of CP/8 consecutive streams (OOB past the stream: zeros)
        const int64_t octets = (c + 7) / 8;
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w_in) * 8, static_cast<cuuint64_t>(ceil_div(w_in * 8, 256)),
                                    static_cast<cuuint64_t>(n * octets)};
        const cuuint64_t strides[2] = {512, static_cast<cuuint64_t>(w_in) * 16};
        const cuuint32_t box[3] = {256, static_cast<cuuint32_t>(pl.xt_nb), static_cast<cuuint32_t>(pl.cp / 8)};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(x_bf16), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    static const bool no_lean = getenv("C1D_NO_LEAN") != nullptr;  // dev A/B switch
    auto kernel = (!pl.xt && !pl.xin && pl.ph == 1 && pl.copies == 1 && !pl.a_mn && !no_lean) ? tc_wgrad2_kernel<1>
                                                                                              : tc_wgrad2_kernel<0>;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(pl.smem_bytes));
    if (e != cudaSuccess) return e;
    W2Params wp{};
    wp.n_items = n;
    wp.c = c;
    wp.k = k;
    wp.s = s;
    wp.q = q;
    wp.w_in = w_in;  // xt: rows per octet stream
    wp.dil = d;
    const W2Seg sg = w2_segments(pl, n, c, k, q);
    wp.steps_per_item = sg.steps_per_item;
    wp.total_steps = sg.total_steps;
    wp.seg = sg.seg;
    wp.slot_elems = sg.slot_elems;
    wp.max_segs = sg.max_segs;
    wp.pl = pl;
    wp.x = x_bf16;
    wp.part = static_cast<float*>(workspace);
    wp.nseg = reinterpret_cast<int*>(static_cast<char*>(workspace) + sg.part_bytes);
    static const bool profile = getenv("C1D_PROFILE") != nullptr;
    if (profile) {
        cudaMalloc(&wp.prof, sizeof(unsigned long long) * 8 * pl.grid);
        cudaMemset(wp.prof, 0, sizeof(unsigned long long) * 8 * pl.grid);
    }
    e = launch_pdl(kernel, dim3(pl.grid), dim3(kW2Threads), pl.smem_bytes, stream, ymap, xmap, wp);
    note_launch();
    if (e != cudaSuccess) return e;
    if (profile) {
        std::vector<unsigned long long> h(8 * pl.grid);
        cudaMemcpy(h.data(), wp.prof, h.size() * 8, cudaMemcpyDeviceToHost);
        double acc[8] = {0};
        for (int bb = 0; bb < pl.grid; ++bb)
            for (int i2 = 0; i2 < 8; ++i2) acc[i2] += static_cast<double>(h[bb * 8 + i2]) / pl.grid;
        fprintf(stderr, "[tc_wgrad3 prof] T=%d P=%d N=%d gpc=%d roles=%d ks=%d stages=%d span=%d ring=%d nbox=%d copies=%d xb=%d | "
                "producer wait_empty %.0f / total %.0f | mma wait_full %.0f issue %.0f commit %.0f wait_drain %.0f total %.0f | drain %.0f\n",
                pl.t, pl.p, pl.n, pl.gpc, pl.roles, pl.ks, pl.stages, pl.span, pl.ring, pl.nbox, pl.copies, pl.xb, acc[0], acc[1], acc[2], acc[3], acc[5], acc[6], acc[4], acc[7]);
        for (int r = 0; r < pl.roles; ++r) {
            unsigned long long mx = 0, wf = 0;
            for (int bb = pl.role_cta_begin[r]; bb < pl.role_cta_begin[r + 1]; ++bb) {
                mx = std::max(mx, h[bb * 8 + 4]);
                wf = std::max(wf, h[bb * 8 + 2]);
            }
            fprintf(stderr, "   role %d: ctas %d groups %d  max total %llu  max wait_full %llu\n", r,
                    pl.role_cta_begin[r + 1] - pl.role_cta_begin[r], pl.role_groups[r], mx, wf);
        }
        cudaFree(wp.prof);
    }
    const int64_t count = k * c * s;
    note_launch();
    return launch_pdl(wgrad2_reduce_kernel, dim3(static_cast<unsigned>(ceil_div(count, 64))), dim3(256), 0, stream,
                      static_cast<const float*>(wp.part), static_cast<const int*>(wp.nseg), dw_kcs,
                      static_cast<int64_t>(k), static_cast<int64_t>(c), static_cast<int64_t>(s), sg.max_segs,
                      sg.slot_elems, pl);
}
}  // namespace

bool tc_wgrad_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    WPlan p;
    W2Plan p2;
    return make_w2plan(n, c, k, s, d, q, &p2) || make_wplan(n, c, k, s, d, q, &p);
}

size_t tc_wgrad_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    W2Plan p2;
    if (make_w2plan(n, c, k, s, d, q, &p2)) {
        const W2Seg sg = w2_segments(p2, n, c, k, q);
        return sg.part_bytes + sg.nseg_bytes;
    }
    WPlan p;
    if (!make_wplan(n, c, k, s, d, q, &p)) return 0;
    return sizeof(float) * static_cast<size_t>(p.roles) * p.splits * static_cast<size_t>(k * c * s);
}

bool tc_wgrad_xin_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    W2Plan p2;
    return make_w2plan(n, c, k, s, d, q, &p2, true);
}

size_t tc_wgrad_xin_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    W2Plan p2;
    if (!make_w2plan(n, c, k, s, d, q, &p2, true)) return 0;
    const W2Seg sg = w2_segments(p2, n, c, k, q);
    return sg.part_bytes + sg.nseg_bytes;
}

cudaError_t launch_tc_wgrad_xin(const uint16_t* x_bf16, int64_t x_w, const uint16_t* dy_bf16, float* dw_kcs,
                                void* workspace, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q,
                                cudaStream_t stream) {
    W2Plan p2;
    if (!make_w2plan(n, c, k, s, d, q, &p2, true)) return cudaErrorNotSupported;
    return launch_v2(x_bf16, dy_bf16, dw_kcs, workspace, n, c, k, s, d, q, p2, stream, x_w);
}

bool tc_wgrad_xt_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    W2Plan p2;
    return make_w2plan_xt(n, c, k, s, d, q, &p2);
}

int64_t tc_wgrad_xt_pad_rows(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    W2Plan p2;
    if (!make_w2plan_xt(n, c, k, s, d, q, &p2)) return 0;
    return 32 * static_cast<int64_t>(p2.xt_nb) + 16;
}

size_t tc_wgrad_xt_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    W2Plan p2;
    if (!make_w2plan_xt(n, c, k, s, d, q, &p2)) return 0;
    const W2Seg sg = w2_segments(p2, n, c, k, q);
    return sg.part_bytes + sg.nseg_bytes;
}

cudaError_t launch_tc_wgrad_xt(const uint16_t* xt, int64_t rows, const uint16_t* dy_bf16, float* dw_kcs,
                               void* workspace, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q,
                               cudaStream_t stream) {
    W2Plan p2;
    if (!make_w2plan_xt(n, c, k, s, d, q, &p2)) return cudaErrorNotSupported;
    return launch_v2(xt, dy_bf16, dw_kcs, workspace, n, c, k, s, d, q, p2, stream, rows);
}

bool tc_wgrad_v3_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    W2Plan p2;
    return make_w2plan(n, c, k, s, d, q, &p2);
}

cudaError_t launch_tc_wgrad(const uint16_t* x_bf16, const uint16_t* dy_bf16, float* dw_kcs, void* workspace,
                            int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, cudaStream_t stream,
                            int64_t x_w) {
    {
        W2Plan p2;
        if (make_w2plan(n, c, k, s, d, q, &p2))
            return launch_v2(x_bf16, dy_bf16, dw_kcs, workspace, n, c, k, s, d, q, p2, stream, x_w);
    }
    WPlan pl;
    if (!make_wplan(n, c, k, s, d, q, &pl)) return cudaErrorNotSupported;
    auto encode = encode_fn();
    if (!encode) return cudaErrorNotSupported;
    const int64_t w_in = x_w > 0 ? x_w : q + d * (s - 1);  // row pitch of x
    if (w_in % 8) return cudaErrorInvalidValue;
    CUtensorMap xmap, ymap;
    {
        // X as (qi=8, c, q-chunk, n): element (qi, c, qc, n) at n*C*W + c*W + qc*8 + qi
        const cuuint64_t dims[4] = {8, static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w_in / 8),
                                    static_cast<cuuint64_t>(n)};
        const cuuint64_t strides[3] = {static_cast<cuuint64_t>(w_in) * 2, 16,
                                       static_cast<cuuint64_t>(c * w_in) * 2};
        const cuuint32_t box[4] = {8, static_cast<cuuint32_t>(pl.cp), static_cast<cuuint32_t>(pl.x_chunks), 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(x_bf16), dims, strides,
                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(q), static_cast<cuuint64_t>(k),
                                    static_cast<cuuint64_t>(n)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(q) * 2, static_cast<cuuint64_t>(k * q) * 2};
        const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(pl.kp), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode(&ymap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(dy_bf16), dims, strides,
                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaFuncSetAttribute(tc_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(pl.smem_bytes));
    if (e != cudaSuccess) return e;
    WParams wp{};
    wp.n_items = n;
    wp.c = c;
    wp.k = k;
    wp.s = s;
    wp.q = q;
    wp.w_in = w_in;
    wp.steps_per_item = ceil_div(q, 16);
    wp.total_steps = n * wp.steps_per_item;
    wp.pl = pl;
    wp.part = static_cast<float*>(workspace);
    const int grid = pl.roles * pl.splits;
    static const bool profile = getenv("C1D_PROFILE") != nullptr;
    if (profile) {
        cudaMalloc(&wp.prof, sizeof(unsigned long long) * 8 * grid);
        cudaMemset(wp.prof, 0, sizeof(unsigned long long) * 8 * grid);
    }
    tc_wgrad_kernel<<<grid, kThreads, pl.smem_bytes, stream>>>(xmap, ymap, wp);
    note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (profile) {
        std::vector<unsigned long long> h(8 * grid);
        cudaMemcpy(h.data(), wp.prof, h.size() * 8, cudaMemcpyDeviceToHost);
        double a[8] = {0};
        for (int b = 0; b < grid; ++b)
            for (int i = 0; i < 8; ++i) a[i] += static_cast<double>(h[b * 8 + i]) / grid;
        fprintf(stderr, "[tc_wgrad prof] ks=%d stages=%d x_chunks=%d | producer wait_empty %.0f / total %.0f | mma wait_full %.0f total %.0f\n",
                pl.ks, pl.stages, pl.x_chunks, a[0], a[1], a[2], a[4]);
        cudaFree(wp.prof);
    }
    const int64_t count = k * c * s;
    wgrad_reduce_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 256), 4096)), 256, 0, stream>>>(
        wp.part, dw_kcs, k, c, s, pl.t, pl.gmax, pl.splits);
    note_launch();
    return cudaGetLastError();
}

}  // namespace c1d
