// mlp_tc.cuh -- fused MLP forward on the 5th-generation tensor cores (tcgen05),
// for the PPO rollout's policy / value networks (
// reference ppo.py:109-141 _mlp / MLPPolicy / MLPValue: Linear + Swish layers).
//
// y = W_out . silu(... silu(W_1 . silu(W_0 x + b_0) + b_1) ...) + b_out for a
// batch of rows, one CTA per 128-row tile (M = 128), 16 warps: warp w serves
// TMEM lanes / rows 32 (w % 4) .. 32 (w % 4) + 31 and the column quarter w / 4:
//   * layer 0 (d_in -> H, d_in small) on the CUDA cores in float32;
//   * the H x H hidden layers on tcgen05.mma kind::f16 with float32 accumulators in
//     TMEM, operands split BF16x3: x = x_hi + x_lo (bf16 each), x.w ~ x_hi w_hi +
//     x_hi w_lo + x_lo w_hi -- ~16 significant bits per product, float32 sums;
//   * the output layer (H -> n_out, n_out small) on the CUDA cores in float32
//     straight from the last hidden layer's float32 activations.
// Activations stay in shared memory between layers (K-major canonical layout,
// SWIZZLE_NONE: 8-row x 16-byte core matrices, LBO = core-matrix stride along K,
// SBO = along M); weights are pre-split and pre-packed in the same layout in HBM
// (pack_weights_kernel) and streamed per 32-column K chunk by 1-D bulk copies
// (cp.async.bulk, the TMA engine) by a loader warp into a 2-4 stage ring (as
// deep as shared memory allows); one thread of another warp issues the MMAs and
// commits them to mbarriers; in the epilogue each warp reads its 32
// TMEM lanes x its column quarter (tcgen05.ld 32x32b): bias, SiLU, split, store;
// the output layer's four partial sums per row are added in quarter order.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace dk {
namespace mlp {

constexpr int M = 128;          // rows per CTA (= TMEM lanes)
constexpr int EPI_WARPS = 16;   // warp w < 16 -> TMEM lanes 32 (w % 4), column quarter w / 4
constexpr int THREADS = 32 * (EPI_WARPS + 2);  // + warp 16: MMA issue, warp 17: weight copies
constexpr int MAXNS = 4;        // weight ring stages (runtime: as many as fit, >= 2)
constexpr int MAXCH = 8;        // K chunks of a hidden layer (H / KC)
constexpr int MAXOUT = 16;      // output-layer width
constexpr int MAXDIN = 128;     // input width (> 16: layer 0 on the tensor cores)
// layer 0's padded input width: 4, 8 or 16 columns
__host__ __device__ constexpr int din_pad(int d_in) { return d_in <= 4 ? 4 : (d_in <= 8 ? 8 : 16); }
// d_in > 16: layer 0 is a tensor-core layer over K0 = d_in rounded up to 32
__host__ __device__ constexpr bool tc_layer0(int d_in) { return d_in > 16; }
constexpr int KC = 32;          // K columns per chunk
constexpr int MAXH = 256;
__host__ __device__ constexpr int k0_pad(int d_in) { return (d_in + KC - 1) / KC * KC; }

struct MlpArgs {
    const float *x;        // [rows][x_stride], first d_in columns used
    int64_t rows, x_stride;
    int d_in, H, n_tc, n_out;
    const float *w0, *b0;             // [H][d_in], [H]
    const __nv_bfloat16 *whi, *wlo;   // packed hidden weights [n_tc][H*H]
    const float *bh;                  // [n_tc][H]
    const float *wout, *bout;         // [n_out][H], [n_out]
    const __nv_bfloat16 *w0hi, *w0lo; // d_in > 16: layer 0 packed [H][K0] (K0 = d_in rounded
                                      // up to 32), run on the tensor cores like the rest
    float *y;                         // [rows][y_stride]
    int64_t y_stride;
    int desc_swap;                    // debug: swap LBO / SBO
    const int64_t *rows_dev;          // nullable: the row count, read on the device
                                      // (<= rows; tiles past it exit at once)
    int ns;                           // weight ring stages (2..MAXNS, mlp_stages)
};

// ------------------------------------------------------------------ PTX glue

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor): start >> 4 at
// [0,14), LBO >> 4 at [16,30), SBO >> 4 at [32,46), version 1 at [46,48),
// base offset 0, layout type 0 = SWIZZLE_NONE at [61,64)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// UMMA instruction descriptor (cute::UMMA::InstrDescriptor): D f32 (bits 4-5 = 1),
// A bf16 (bits 7-9 = 1), B bf16 (bits 10-12 = 1), both K-major, N >> 3 at
// [17,23), M >> 4 at [24,29)
__host__ __device__ constexpr uint32_t instr_desc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *mbar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// 32 consecutive f32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
        "[%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// x * sigmoid(x) = x / (1 + 2^(-x log2 e)): MUFU.EX2 and MUFU.RCP without the
// range fix-ups of __expf / __fdividef (x -> -inf: e = inf, rcp = 0, -0; x -> +inf:
// e = 0, x; NaN propagates)
__device__ __forceinline__ float silu(float x) {
#ifdef DK_MLP_EXP_NOSILU
    return x;
#endif
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
    return x * r;
}

// element (row r, column k) of a K-major canonical operand made of 32-column
// chunks: chunk k / 32 at chunk_bytes * (k / 32); inside a chunk, core matrix
// (r / 8, (k % 32) / 8) at (r / 8) * 512 + ((k % 32) / 8) * 128; inside it, row
// r % 8 at 16 * (r % 8), element k % 8 at 2 * (k % 8)
__host__ __device__ __forceinline__ uint32_t op_offset(int r, int k, int rows_total) {
    const uint32_t chunk_bytes = (uint32_t)rows_total * KC * 2;
    return (uint32_t)(k / KC) * chunk_bytes + (uint32_t)(r / 8) * 512 + (uint32_t)((k % KC) / 8) * 128 +
           (uint32_t)(r % 8) * 16 + (uint32_t)(k % 8) * 2;
}

// store 8 consecutive float activations (row r, columns k..k+7) split into bf16
// hi / lo (x = hi + lo, both rounded to nearest), two values per conversion
__device__ __forceinline__ void store_split8(unsigned char *ahi, unsigned char *alo, int r, int k,
                                             const float *v) {
    uint4 h4, l4;
    uint32_t *hp = &h4.x, *lp = &l4.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        const float2 hf = __bfloat1622float2(h);
        const __nv_bfloat162 l = __floats2bfloat162_rn(v[2 * i] - hf.x, v[2 * i + 1] - hf.y);
        hp[i] = *reinterpret_cast<const uint32_t *>(&h);
        lp[i] = *reinterpret_cast<const uint32_t *>(&l);
    }
    const uint32_t off = op_offset(r, k, M);
    *reinterpret_cast<uint4 *>(ahi + off) = h4;
    *reinterpret_cast<uint4 *>(alo + off) = l4;
}

// fp32 W [N][K] (torch Linear weight: out x in, K contiguous) -> packed bf16 hi / lo
__global__ void pack_weights_kernel(const float *w, int N, int K, __nv_bfloat16 *hi,
                                    __nv_bfloat16 *lo) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * K) return;
    const int n = i / K, k = i % K;
    const float v = w[i];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
    const uint32_t e = op_offset(n, k, N) / 2;
    hi[e] = h;
    lo[e] = l;
}

// Warp-specialised and pipelined across layers: warp 17 streams the weights,
// warp 16 issues the MMAs; warps 0-15 run layer 0 and the epilogues.  Two TMEM
// accumulators alternate between layers, and the activations of layer l + 1
// are handed to the MMA warp K-chunk by K-chunk (an mbarrier per 32-column
// chunk): layer l + 1's MMAs start on the first chunks while layer l's
// epilogue is still producing the rest, and the first hidden layer's MMAs
// overlap layer 0.  (The serial MMA -> epilogue -> MMA chain was most of a
// call: r02 A/B.)
//
// One launch may evaluate two networks (e.g. the PPO policy on this step's
// observations and the value function on the same observations): CTAs
// [0, tiles0) take network a0, the rest a1 -- the two calls' latency-bound
// tiles then share the GPU instead of running back to back.
// MO: output-layer accumulators per thread (4, or MAXOUT for wider heads)
template <int MO>
__global__ void __launch_bounds__(THREADS, 1) mlp_tc_kernel(MlpArgs a0, MlpArgs a1,
                                                            int64_t tiles0) {
    extern __shared__ __align__(1024) unsigned char smem[];
    // programmatic dependent launch (capi_mlp.cu): nothing of the previous
    // kernel's (inputs, row count, outputs) is touched before this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool second = (int64_t)blockIdx.x >= tiles0;
    MlpArgs a = second ? a1 : a0;
    const int64_t tile = second ? (int64_t)blockIdx.x - tiles0 : (int64_t)blockIdx.x;
    if (a.rows_dev) {  // a device-side row count (e.g. the compacted bootstrap rows)
        const int64_t rd = *a.rows_dev;
        a.rows = rd < a.rows ? rd : a.rows;
        if (tile * M >= a.rows) return;  // the whole CTA: uniform
    }
    const int H = a.H, din = a.d_in, nout = a.n_out;
    const int nch = H / KC;
    const uint32_t a_bytes = (uint32_t)M * H * 2;           // one of A_hi / A_lo
    const uint32_t b_chunk = (uint32_t)H * KC * 2;          // one B chunk (hi or lo)
    unsigned char *A_hi = smem;
    unsigned char *A_lo = smem + a_bytes;
    const int ns = a.ns;
    unsigned char *Bst = smem + 2 * a_bytes;                // [ns stages][hi, lo][b_chunk]
    // full[ns] empty[ns] (weight ring), done[2] (accumulator of layer l: done[l & 1]),
    // achunk[MAXCH] (K chunk c of the current layer's input written), w0free (a
    // CUDA-core layer 0 has read its weights)
    uint64_t *bars = reinterpret_cast<uint64_t *>(Bst + 2 * ns * b_chunk);
    uint64_t *full = bars, *empty = bars + MAXNS, *done = bars + 2 * MAXNS,
             *achunk = bars + 2 * MAXNS + 2;
    uint64_t *w0free = bars + 2 * MAXNS + 2 + MAXCH;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * MAXNS + 3 + MAXCH);
    // the float32 parameters used on the CUDA cores, staged once; layer 0's weight
    // rows (CUDA-core layer 0 only) padded to DP columns (zeros past d_in) for
    // 16-byte loads, in the ring's last stage (the loader fills that stage once
    // layer 0 is done).  (Biases are read from global memory: L1-resident.)
    const bool tc0 = tc_layer0(din);
    const int DP = tc0 ? 0 : din_pad(din);
    const int NO = nout <= 4 ? 4 : MAXOUT;                   // partial-sum slots per row
    float *s_w0 = reinterpret_cast<float *>(Bst + 2 * (ns - 1) * b_chunk);  // [H][DP]
    float *s_wo = reinterpret_cast<float *>(bars + 2 * MAXNS + 4 + MAXCH);  // [nout][H]
    // [4 quarters][M][NO] partial outputs: written after the last layer's MMAs
    // completed, so they reuse the activation buffer
    float *s_red = reinterpret_cast<float *>(A_hi);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q = warp & 3, quarter = warp >> 2;            // TMEM lane group, column quarter
    const int row = 32 * q + lane;
    const int64_t r_glob = tile * M + row;
    const int HQ = H / 4;                                    // columns per thread (32 or 64)
    const uint32_t tcols = 2u * (uint32_t)H;                 // two accumulators

    for (int i = tid; i < H * DP; i += THREADS) {
        const int j = i / DP, k = i - j * DP;
        s_w0[i] = k < din ? a.w0[j * din + k] : 0.0f;
    }
    for (int i = tid; i < nout * H; i += THREADS) s_wo[i] = a.wout[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int i = 0; i < 2 * MAXNS + 2; ++i) mbar_init(&bars[i], 1);
        for (int c = 0; c < MAXCH; ++c) mbar_init(&achunk[c], 4);  // the 4 warps of a quarter
        mbar_init(w0free, EPI_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // K chunks are consumed in the order the epilogue finishes them: each column
    // quarter writes its chunks in turn, so the first of every quarter comes first
    // (a tensor-core layer 0 reads x, staged one 32-column chunk per quarter)
    const int cpq = nch / 4;                                 // chunks per quarter (1 or 2)
    auto kchunk = [&](int i) { return (i % 4) * cpq + i / 4; };
    const int nl = a.n_tc + (tc0 ? 1 : 0);                   // tensor-core layers
    const int nch0 = tc0 ? k0_pad(din) / KC : nch;           // K chunks of layer 0
    auto layer_chunks = [&](int l) { return l == 0 ? nch0 : nch; };

    const uint32_t total = (uint32_t)(nch0 + (nl - 1) * nch);  // weight chunks
    if (warp == EPI_WARPS + 1) {
        // ---------------------------------------------- weight loader: runs ahead
        // of the MMAs by up to ns chunks (its own warp: it never waits on the
        // activations)
        if (lane == 0) {
            for (uint32_t gg = 0; gg < total; ++gg) {
                const int s = (int)(gg % (uint32_t)ns);
                if (gg >= (uint32_t)ns) mbar_wait(&empty[s], ((gg / ns) - 1) & 1);  // stage free
                else if (!tc0 && gg + 1 == (uint32_t)ns) mbar_wait(w0free, 0);  // holds W0
                int ll, i;
                if (gg < (uint32_t)nch0) {
                    ll = 0;
                    i = (int)gg;
                } else {
                    ll = 1 + (int)((gg - nch0) / nch);
                    i = (int)((gg - nch0) % nch);
                }
#ifdef DK_MLP_EXP_NOLOAD
                mbar_expect_tx(&full[s], 0);
                continue;
#endif
                mbar_expect_tx(&full[s], 2 * b_chunk);
                const __nv_bfloat16 *hi, *lo;
                if (tc0 && ll == 0) {
                    hi = a.w0hi + (size_t)i * H * KC;
                    lo = a.w0lo + (size_t)i * H * KC;
                } else {
                    const int c = kchunk(i);
                    const size_t off = (size_t)(ll - (tc0 ? 1 : 0)) * H * H + (size_t)c * H * KC;
                    hi = a.whi + off;
                    lo = a.wlo + off;
                }
                bulk_g2s(Bst + (2 * s) * b_chunk, hi, b_chunk, &full[s]);
                bulk_g2s(Bst + (2 * s + 1) * b_chunk, lo, b_chunk, &full[s]);
            }
        }
        __syncwarp();
    } else if (warp == EPI_WARPS) {
        // ---------------------------------------------- MMA issue
        if (lane == 0) {
            const uint32_t idesc = instr_desc_bf16(M, H);
            const uint32_t lbo = a.desc_swap ? 512u : 128u, sbo = a.desc_swap ? 128u : 512u;
            uint32_t gbase = 0;
            for (int l = 0; l < nl; ++l) {
                const uint32_t tacc = tmem + (uint32_t)((l & 1) * H);
                const int lch = layer_chunks(l);
                for (int i = 0; i < lch; ++i) {
                    const int c = (tc0 && l == 0) ? i : kchunk(i);
                    const uint32_t gc = gbase + (uint32_t)i;
                    const int s = (int)(gc % (uint32_t)ns);
                    // this layer's input, K chunk c: its barrier completed once per
                    // earlier layer whose input had chunk c (a tensor-core layer 0
                    // reads only x's nch0 chunks)
                    const int ph = (tc0 && l > 0 && c >= nch0) ? l - 1 : l;
                    mbar_wait(&achunk[c], ph & 1);
                    mbar_wait(&full[s], (gc / ns) & 1);  // its weights
                    tc_fence_after();
                    const uint32_t a_hi = smem_u32(A_hi) + c * (M * KC * 2);
                    const uint32_t a_lo = smem_u32(A_lo) + c * (M * KC * 2);
                    const uint32_t b_hi = smem_u32(Bst + (2 * s) * b_chunk);
                    const uint32_t b_lo = smem_u32(Bst + (2 * s + 1) * b_chunk);
#pragma unroll
                    for (int ks = 0; ks < KC / 16; ++ks) {
                        const uint32_t o = ks * 256;  // two core matrices along K
                        const uint64_t dah = smem_desc(a_hi + o, lbo, sbo);
                        const uint64_t dal = smem_desc(a_lo + o, lbo, sbo);
                        const uint64_t dbh = smem_desc(b_hi + o, lbo, sbo);
                        const uint64_t dbl = smem_desc(b_lo + o, lbo, sbo);
#ifndef DK_MLP_EXP_NOMMA
                        mma_bf16(tacc, dah, dbh, idesc, (i | ks) != 0);
                        mma_bf16(tacc, dah, dbl, idesc, 1);
                        mma_bf16(tacc, dal, dbh, idesc, 1);
#else
                        (void)dah; (void)dal; (void)dbh; (void)dbl;
#endif
                    }
                    mma_commit(&empty[s]);  // stage s free once these MMAs complete
                    if (i + 1 == lch) mma_commit(&done[l & 1]);  // layer l's accumulator final
                }
                gbase += (uint32_t)lch;
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ layer 0 and epilogues
        // hand K chunk c of the next layer's input to the MMA warp: stores
        // visible to the tensor core (async proxy), TMEM reads ordered before
        auto publish = [&](int c) {
#ifndef DK_MLP_EXP_NOFENCE
            fence_async_smem();
#endif
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(
                                            smem_u32(&achunk[c]))
                                        : "memory");
        };
        // layer 0 on the CUDA cores (float32): this thread's row, its column quarter;
        // padded weight rows read 16 bytes at a time (the padding adds exact zeros)
        auto layer0 = [&](auto dp_c) {
            constexpr int DPC = decltype(dp_c)::value;
            float x[DPC];
#pragma unroll
            for (int i = 0; i < DPC; ++i)
                x[i] = (i < din && r_glob < a.rows) ? a.x[r_glob * a.x_stride + i] : 0.0f;
            for (int j0 = quarter * HQ; j0 < (quarter + 1) * HQ; j0 += 8) {
                float v[8];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int j = j0 + jj;
                    float s = __ldg(a.b0 + j);
                    const float4 *w = reinterpret_cast<const float4 *>(s_w0 + j * DPC);
#pragma unroll
                    for (int i4 = 0; i4 < DPC / 4; ++i4) {
                        const float4 q4 = w[i4];
                        s = fmaf(q4.x, x[4 * i4], s);
                        s = fmaf(q4.y, x[4 * i4 + 1], s);
                        s = fmaf(q4.z, x[4 * i4 + 2], s);
                        s = fmaf(q4.w, x[4 * i4 + 3], s);
                    }
                    v[jj] = r_glob < a.rows ? silu(s) : 0.0f;
                }
                store_split8(A_hi, A_lo, row, j0, v);
                if ((j0 + 8) % KC == 0) publish(j0 / KC);
            }
        };
        if (tc0) {
            // stage x (K0 columns, zeros past d_in) as the first layer's operand:
            // quarter c splits chunk c of its 32 rows
            if (quarter < nch0) {
                for (int k8 = 0; k8 < KC; k8 += 8) {
                    float v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int col = quarter * KC + k8 + i;
                        v[i] = (col < din && r_glob < a.rows) ? a.x[r_glob * a.x_stride + col]
                                                              : 0.0f;
                    }
                    store_split8(A_hi, A_lo, row, quarter * KC + k8, v);
                }
                publish(quarter);
            }
        } else {
            if (DP == 4) layer0(std::integral_constant<int, 4>{});
            else if (DP == 8) layer0(std::integral_constant<int, 8>{});
            else layer0(std::integral_constant<int, 16>{});
            // the weight ring's last stage (W0's home) may now be filled
            fence_async_smem();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(
                                            smem_u32(w0free))
                                        : "memory");
        }
        float out_acc[MO];
#pragma unroll
        for (int o = 0; o < MO; ++o) out_acc[o] = 0.f;
        for (int l = 0; l < nl; ++l) {
            mbar_wait(&done[l & 1], (l >> 1) & 1);
            tc_fence_after();
            // ---- epilogue (this thread's row and column quarter): bias, SiLU; split
            // into the next layer's input, or partial output-layer dot products
            const bool last = l + 1 == nl;
            const float *bias = (tc0 && l == 0) ? a.b0 : a.bh + (size_t)(l - (tc0 ? 1 : 0)) * H;
            const uint32_t tacc = tmem + (uint32_t)((l & 1) * H);
            // one 32-column chunk of this thread's row, loaded from TMEM: bias, SiLU,
            // then the next layer's input (split, stored, published) or the output
            // layer's partial dot products
            auto chunk = [&](int cc, float *v) {
                const float4 *b4 = reinterpret_cast<const float4 *>(bias + cc * 32);  // 16 B aligned
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {
                    const float4 bb = b4[i4];
                    v[4 * i4] = silu(v[4 * i4] + bb.x);
                    v[4 * i4 + 1] = silu(v[4 * i4 + 1] + bb.y);
                    v[4 * i4 + 2] = silu(v[4 * i4 + 2] + bb.z);
                    v[4 * i4 + 3] = silu(v[4 * i4 + 3] + bb.w);
                }
                if (last) {
#pragma unroll
                    for (int o = 0; o < MO; ++o) {
                        if (o < nout) {
                            const float4 *w4 = reinterpret_cast<const float4 *>(s_wo + (size_t)o * H + cc * 32);
                            float s = out_acc[o];
#pragma unroll
                            for (int i4 = 0; i4 < 8; ++i4) {
                                const float4 ww = w4[i4];
                                s = fmaf(ww.x, v[4 * i4], s);
                                s = fmaf(ww.y, v[4 * i4 + 1], s);
                                s = fmaf(ww.z, v[4 * i4 + 2], s);
                                s = fmaf(ww.w, v[4 * i4 + 3], s);
                            }
                            out_acc[o] = s;
                        }
                    }
                } else {
#ifndef DK_MLP_EXP_NOSTORE
#pragma unroll
                    for (int k8 = 0; k8 < 4; ++k8)
                        store_split8(A_hi, A_lo, row, cc * 32 + k8 * 8, v + 8 * k8);
#else
                    if (v[0] == 1234.5f) store_split8(A_hi, A_lo, row, cc * 32, v);
#endif
                    publish(cc);
                }
            };
            const uint32_t trow = tacc + ((uint32_t)(q * 32) << 16);
            for (int cc = quarter * HQ / 32; cc < (quarter + 1) * HQ / 32; ++cc) {
                float v[32];
#ifndef DK_MLP_EXP_NOLD
                tmem_ld32(trow + cc * 32, v);
#else
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = (float)(i + row) * 0.01f;
#endif
                chunk(cc, v);
            }
        }
        // output layer: the four column quarters' partial sums, in quarter order
#pragma unroll
        for (int o = 0; o < MO; ++o)
            if (o < nout) s_red[(quarter * M + row) * NO + o] = out_acc[o];
    }
    tc_fence_before();
    __syncthreads();
    if (warp < EPI_WARPS && quarter == 0 && r_glob < a.rows)
        for (int o = 0; o < nout; ++o) {
            const float s = ((s_red[(0 * M + row) * NO + o] + s_red[(1 * M + row) * NO + o]) +
                             (s_red[(2 * M + row) * NO + o] + s_red[(3 * M + row) * NO + o]));
            a.y[r_glob * a.y_stride + o] = s + a.bout[o];
        }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                     "r"(tcols));
}

// dynamic shared memory of a call with an ns-stage weight ring
inline size_t mlp_smem_bytes(int H, int d_in, int n_out, int ns) {
    (void)d_in;  // a CUDA-core layer 0's weights live in the ring's last stage
    return 2 * (size_t)M * H * 2 + 2 * (size_t)ns * H * KC * 2 + 8 * (2 * MAXNS + 4 + MAXCH) +
           4 * (size_t)n_out * H;
}

// the deepest weight ring (<= MAXNS stages) that fits in 227 KB; 0 if none (>= 2)
inline int mlp_stages(int H, int d_in, int n_out) {
#ifdef DK_MLP_EXP_NS
    for (int ns = DK_MLP_EXP_NS; ns >= 2; --ns)  // A/B: a shallower ring
#else
    for (int ns = MAXNS; ns >= 2; --ns)
#endif
        if (mlp_smem_bytes(H, d_in, n_out, ns) <= 227 * 1024) return ns;
    return 0;
}

}  // namespace mlp
}  // namespace dk
