// envstep_kernels.cuh -- fused batched env step / rollout kernels.
//
// One thread owns one world for the whole launch: the state is read from HBM
// once, advanced K control steps in registers (dynamics -> reward -> obs ->
// truncation -> Philox autoreset, the whole of Environment.step +
// BatchEnv.step's autoreset, envkit.py:526-552, 630-635), and written back
// once.  Per step the only HBM traffic is the algorithmic I/O: the action in,
// obs / reward / done / trunc (and optionally the info terms) out.
//
//  - Warp-specialised: a producer warp runs the serial dynamics chain of 32
//    worlds, consumer warps turn its ring of states into outputs (below).
//  - Actions are prefetched CH steps ahead into registers (double-buffered
//    chunks), so the dependent chain of the dynamics never waits on HBM.
//  - Row outputs ([.., N, O] obs, [.., N, I] info) are transposed through a
//    per-warp shared-memory tile so every global store is a full, coalesced
//    128-byte line instead of a 4-byte strided scatter.
//  - Validation is fused and batch-atomic: each world checks its own actions
//    as it consumes them (and knows up front at which step it would need a
//    reset); the first error in reference order (step-major, then world) is
//    kept in a sticky key, and the state buffers are double-buffered so the
//    launch commits only when the whole batch was valid.
#pragma once
#include "tasks.cuh"

namespace dk {

constexpr unsigned long long kNoError = ~0ULL;
constexpr int kErrUsage = 1;    // UsageError: world must be reset (envkit.py:527-528)
constexpr int kErrInvalid = 2;  // InvalidInputError: non-finite action (envkit.py:530-531)

// SoA world bookkeeping in HBM, double-buffered: a launch reads buffer
// `*cur` and writes buffer `1 - *cur`; the last block to finish flips `*cur`
// only if the launch saw no error, so an invalid batch leaves every world
// exactly as it was (batch-atomic) without a separate validation pass.
template <typename T>
struct Worlds {
    T *state[2];              // [NS, N] each
    int32_t *steps[2];        // [N]   Environment.steps
    uint32_t *episode[2];     // [N]   Environment._episode mod 2^32 (-1 == 0xffffffff)
    uint8_t *needs_reset[2];  // [N]   Environment._needs_reset
    int32_t *cur;             // which buffer is live
    uint32_t *blocks_done;    // last-block counter (returns to 0 after each launch)
};

template <typename T>
struct StepOut {
    T *obs;                 // [K, N, O]
    T *reward;              // [K, N]
    uint8_t *done;          // [K, N]
    uint8_t *trunc;         // [K, N]
    T *term_obs;            // [K, N, O] sparse, may be null
    uint8_t *term_mask;     // [K, N], may be null
    T *info;                // [K, N, I], may be null
};

struct EnvScalars {
    uint64_t seed;
    int64_t n;              // worlds on this device
    int64_t env_offset;     // global index of world 0
    int32_t episode_length;
    int32_t action_repeat;
    int32_t wide_init;
    int32_t autoreset;
};

// ---------------------------------------------------------------------------
// Warp-cooperative store of one R-wide row per lane into out[row0 + lane][R]
// (rows beyond `nrows` are skipped).  tile: this warp's 32*R slots of smem.

template <typename T, int R>
__device__ __forceinline__ void warp_store_rows(T *__restrict__ out, int64_t row0, int64_t nrows,
                                                const T (&v)[R], T *tile, int lane) {
#pragma unroll
    for (int j = 0; j < R; ++j) tile[lane * R + j] = v[j];
    __syncwarp();
    const int64_t valid = nrows - row0 < 32 ? (nrows - row0) * R : 32 * R;
    T *dst = out + row0 * R;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int e = j * 32 + lane;
        if (e < valid) dst[e] = tile[e];
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// Last block of a launch: commit the written state buffer if the batch was valid.

__device__ __forceinline__ void finish_launch(int32_t *cur, uint32_t *blocks_done,
                                              const unsigned long long *err, bool commit_ok) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(blocks_done, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence();
            const unsigned long long e = *(volatile const unsigned long long *)err;
            if (commit_ok && e == kNoError) *cur = 1 - *cur;
            *blocks_done = 0u;
        }
    }
}

static __device__ __noinline__ void record_error(unsigned long long *err, int64_t k, int64_t n,
                                          int64_t i, int code) {
    const unsigned long long key = ((unsigned long long)(k * n + i) << 2) | (unsigned long long)code;
    atomicMin(err, key);
}

// ---------------------------------------------------------------------------
// mbarrier helpers (shared::cta, generic proxy only)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// cp.async (LDGSTS): per-lane async global->shared copy of one action row.
template <int BYTES>
__device__ __forceinline__ void cp_async_ca(void *smem_dst, const void *gsrc, bool valid) {
    static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
    const int src_size = valid ? BYTES : 0;  // 0: zero-fill, no global read
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(smem_dst)),
                 "l"(gsrc), "n"(BYTES), "r"(src_size)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// Fused K-step rollout (K == 1 is BatchEnv.step), warp-specialised.
//
// A block owns a tile of 32 worlds.  With only 8192 worlds per GPU there are
// fewer warps than the 592 SM sub-partitions, so a monolithic thread-per-world
// step is bound by the latency of one serial instruction stream.  The work is
// therefore split by dependency:
//   warp 0 (producer):   the serial chain only -- action clip/validation,
//                        dynamics (+ trig refresh), step counter, Philox
//                        autoreset; writes each post-step world state into a
//                        D-deep shared-memory ring (slot layout [field][lane],
//                        conflict-free) and arrives on full[slot].
//   warps 1..M (consumers): control step k is handled by consumer k % M:
//                        wait full[slot], pull the state into registers,
//                        release empty[slot], then reward + info terms,
//                        observation, flags and all global stores (rows
//                        transposed through a per-warp tile so every store is
//                        a coalesced 128 B line).
// Rewards of the first action_repeat-1 substeps are summed by the producer in
// the reference's order (reward = 0.0; reward += r, envkit.py:533-540), the
// consumer adds the last one, so the arithmetic is unchanged.

template <class Task, typename T>
struct RolloutShape {
    static constexpr int WF = (int)(sizeof(typename Task::W) / sizeof(T));  // floats per world
    static constexpr int SLOT_BYTES = 32 * WF * (int)sizeof(T);
    static constexpr int D = SLOT_BYTES <= 1024 ? 16 : 8;                    // ring depth
    static constexpr int M = 4;                                              // consumer warps
    static constexpr int R = Task::O > Task::I ? Task::O : Task::I;
    static constexpr int THREADS = 32 * (1 + M);
    static constexpr int P = 16;                                             // action prefetch depth
    // shared memory carve-up
    static constexpr size_t OFF_BAR = 0;                                     // full[D], empty[D]
    static constexpr size_t OFF_RING = 16 * D;
    static constexpr size_t OFF_POST = OFF_RING + (size_t)D * WF * 32 * sizeof(T);
    static constexpr size_t OFF_RPART = OFF_POST + (size_t)D * WF * 32 * sizeof(T);
    static constexpr size_t OFF_FLAGS = OFF_RPART + (size_t)D * 32 * sizeof(T);
    static constexpr size_t OFF_TILE = (OFF_FLAGS + (size_t)D * 32 + 15) / 16 * 16;
    static constexpr size_t OFF_ACT = OFF_TILE + (size_t)M * 32 * R * sizeof(T);  // [P][32][A]
    static constexpr size_t OFF_CTRL = OFF_ACT + (size_t)P * 32 * Task::A * sizeof(T);
    static constexpr size_t SMEM = OFF_CTRL + 16;
};

template <class Task, typename T>
__device__ __forceinline__ void world_to_slot(const typename Task::W &w, T *slot, int lane);

// Environment.reset (envkit.py:502-519) of one world inside a rollout: the
// next Philox stream of (seed, env, episode) -> sample_initial.  Out of line:
// taken once per episode_length steps.
template <class Task, typename T>
__device__ __noinline__ typename Task::W autoreset_world(uint64_t seed, uint64_t gidx,
                                                         uint32_t episode, Params<T> p, int wide,
                                                         T *post_slot, int lane) {
    typename Task::W wd;
    Philox4x64 rng;
    rng.init(seed, gidx, episode, 0);
    Task::sample(wd, rng, p, wide != 0);
    world_to_slot<Task, T>(wd, post_slot, lane);
    return wd;
}

template <class Task, typename T>
__device__ __forceinline__ void world_to_slot(const typename Task::W &w, T *slot, int lane) {
    constexpr int WF = RolloutShape<Task, T>::WF;
    const T *f = reinterpret_cast<const T *>(&w);
#pragma unroll
    for (int j = 0; j < WF; ++j) slot[j * 32 + lane] = f[j];
}

template <class Task, typename T>
__device__ __forceinline__ void slot_to_world(typename Task::W &w, const T *slot, int lane) {
    constexpr int WF = RolloutShape<Task, T>::WF;
    T *f = reinterpret_cast<T *>(&w);
#pragma unroll
    for (int j = 0; j < WF; ++j) f[j] = slot[j * 32 + lane];
}

template <class Task, typename T, bool R1>
__global__ void __launch_bounds__(RolloutShape<Task, T>::THREADS)
rollout_kernel(const T *__restrict__ actions, int64_t K, EnvScalars sc, Params<T> p, Worlds<T> w,
               StepOut<T> out, unsigned long long *err) {
    using S = RolloutShape<Task, T>;
    constexpr int A = Task::A, O = Task::O, I = Task::I, WF = S::WF, D = S::D, M = S::M;
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::OFF_BAR);
    uint64_t *empty = full + D;
    T *ring = reinterpret_cast<T *>(smem + S::OFF_RING);    // [D][WF][32]
    T *post = reinterpret_cast<T *>(smem + S::OFF_POST);    // [D][WF][32] post-reset state
    T *rpart = reinterpret_cast<T *>(smem + S::OFF_RPART);  // [D][32]
    uint8_t *flags = smem + S::OFF_FLAGS;                   // [D][32] bit0 trunc, bit1 reset
    int *ctrl = reinterpret_cast<int *>(smem + S::OFF_CTRL);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n = sc.n;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    const int64_t row0 = (int64_t)blockIdx.x * 32;
    const bool in_range = i < n;

    if (threadIdx.x == 0) {
        // a pending (sticky) error from an earlier call: the batch is not
        // stepped.  Read once so the whole block takes the same branch.
        ctrl[0] = *(volatile const unsigned long long *)err != kNoError;
        ctrl[1] = *w.cur;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            mbar_init(&full[d], 32);
            mbar_init(&empty[d], 32);  // consumer warp 0 pre-arms every slot once (below)
        }
    }
    __syncthreads();
    const bool blocked = ctrl[0] != 0;
    const int src = ctrl[1];

    if (!blocked && warp == 0) {
        // ------------------------------------------------------------ producer
        // buffer selection by ternary: runtime-indexing the by-value param
        // arrays would spill the whole struct to local memory
        const T *st_src = src ? w.state[1] : w.state[0];
        T *st_dst = src ? w.state[0] : w.state[1];
        const int32_t *steps_src = src ? w.steps[1] : w.steps[0];
        int32_t *steps_dst = src ? w.steps[0] : w.steps[1];
        const uint32_t *ep_src = src ? w.episode[1] : w.episode[0];
        uint32_t *ep_dst = src ? w.episode[0] : w.episode[1];
        const uint8_t *nr_src = src ? w.needs_reset[1] : w.needs_reset[0];
        uint8_t *nr_dst = src ? w.needs_reset[0] : w.needs_reset[1];

        typename Task::W wd;
        int32_t steps = 0;
        uint32_t episode = 0;
        int64_t k_usage = K;  // step at which this world would need a reset (UsageError)
        if (in_range) {
            Task::load(wd, st_src, i, n);
            steps = steps_src[i];
            episode = ep_src[i];
            if (nr_src[i]) {
                k_usage = 0;
            } else if (!sc.autoreset && (int64_t)sc.episode_length - steps < K) {
                k_usage = (int64_t)sc.episode_length - steps;
            }
            if (k_usage < K) record_error(err, k_usage, n, i, kErrUsage);
        } else {
            Task::zero(wd);
        }
        Task::refresh(wd);
        const uint64_t gidx = (uint64_t)(sc.env_offset + i);
        bool ok = true;

        // actions stream through a P-deep shared-memory ring filled by
        // cp.async P steps ahead: the loop body stays one step long (small
        // I-cache footprint) and the dependent chain never waits on HBM
        constexpr int P = S::P;
        T *aring = reinterpret_cast<T *>(smem + S::OFF_ACT);  // [P][32][A]
        const int K32 = (int)K;  // host guarantees K < 2^31
        const T *aptr = actions + (in_range ? i * A : 0);
        const int64_t astep = in_range ? n * A : 0;
#pragma unroll 1
        for (int k = 0; k < P; ++k) {
            cp_async_ca<A * sizeof(T)>(aring + (k * 32 + lane) * A, aptr + k * astep,
                                       in_range && k < K32);
            cp_async_commit();
        }
        const T *anext = aptr + P * astep;
        const int ku = k_usage < K ? (int)k_usage : K32;
        uint32_t phase_bits = 0;  // bit d: parity of the next empty[d] completion to wait for

#pragma unroll 1
        for (int k = 0; k < K32; ++k) {
            const int slot = k & (D - 1);
            const int ar = k & (P - 1);
            cp_async_wait<P - 1>();  // this lane's copy for step k has landed
            T a[A];
            bool fin = true;
#pragma unroll
            for (int j = 0; j < A; ++j) {  // min(max(float(a), -1.0), 1.0)  (envkit.py:532)
                T v = aring[(ar * 32 + lane) * A + j];
                fin &= RealOps<T>::finite_(v);
                a[j] = fmin(fmax(v, T(-1)), T(1));
            }
            cp_async_ca<A * sizeof(T)>(aring + (ar * 32 + lane) * A, anext,
                                       in_range && k + P < K32);
            cp_async_commit();
            anext += astep;
            if (__builtin_expect(!fin && ok && in_range && k < ku, 0)) {  // envkit.py:529-531
                ok = false;
                record_error(err, k, n, i, kErrInvalid);
            }
            T rp = T(0);
            Task::step(wd, a, p);
            if (!R1) {
                for (int rep = 1; rep < sc.action_repeat; ++rep) {
                    T inf[I];
                    rp += Task::reward(wd, p, inf);
                    Task::step(wd, a, p);
                }
            }
            steps += 1;
            const bool truncated = steps >= sc.episode_length;
            const bool reset = truncated && sc.autoreset && in_range;
            mbar_wait(&empty[slot], (phase_bits >> slot) & 1u);
            phase_bits ^= 1u << slot;
            world_to_slot<Task, T>(wd, ring + (size_t)slot * WF * 32, lane);
            if (!R1) rpart[slot * 32 + lane] = rp;
            flags[slot * 32 + lane] = (uint8_t)((truncated ? 1 : 0) | (reset ? 2 : 0));
            if (__builtin_expect(reset, 0)) {
                episode += 1;
                steps = 0;
                wd = autoreset_world<Task, T>(sc.seed, gidx, episode, p, sc.wide_init,
                                              post + (size_t)slot * WF * 32, lane);
            }
            mbar_arrive(&full[slot]);
        }
        cp_async_wait<0>();
        if (in_range) {
            Task::store(wd, st_dst, i, n);
            steps_dst[i] = steps;
            ep_dst[i] = episode;
            // without autoreset a world that truncated in this window needs a reset
            nr_dst[i] = (!sc.autoreset && steps >= sc.episode_length) ? 1 : 0;
        }
    } else if (!blocked) {
        // ------------------------------------------------------------ consumers
        const int c = warp - 1;
        T *tile = reinterpret_cast<T *>(smem + S::OFF_TILE) + (size_t)c * 32 * S::R;
        const T inv_rep = T(sc.action_repeat);
        if (c == 0) {
#pragma unroll
            for (int d = 0; d < D; ++d) mbar_arrive(&empty[d]);  // slots start free
        }
        for (int64_t k = c; k < K; k += M) {
            const int slot = (int)(k % D);
            mbar_wait(&full[slot], (uint32_t)(k / D) & 1u);
            typename Task::W wd, wp;
            slot_to_world<Task, T>(wd, ring + (size_t)slot * WF * 32, lane);
            const T rp = R1 ? T(0) : rpart[slot * 32 + lane];
            const uint8_t fl = flags[slot * 32 + lane];
            const bool reset = (fl & 2) != 0;
            if (reset) slot_to_world<Task, T>(wp, post + (size_t)slot * WF * 32, lane);
            mbar_arrive(&empty[slot]);

            T info[I];
            const T r = R1 ? (T(0) + Task::reward(wd, p, info))
                           : (rp + Task::reward(wd, p, info)) / inv_rep;
            T o[O];
            Task::obs(wd, p, o);
            const int64_t ko = k * n;
            if (reset) {
                if (out.term_obs) {
#pragma unroll
                    for (int j = 0; j < O; ++j) out.term_obs[(ko + i) * O + j] = o[j];
                }
                Task::obs(wp, p, o);
            }
            warp_store_rows<T, O>(out.obs + ko * O, row0, n, o, tile, lane);
            if (out.info) warp_store_rows<T, I>(out.info + ko * I, row0, n, info, tile, lane);
            if (in_range) {
                out.reward[ko + i] = r;
                out.done[ko + i] = 0;
                out.trunc[ko + i] = fl & 1;
                if (out.term_mask) out.term_mask[ko + i] = reset ? 1 : 0;
            }
        }
    }
    finish_launch(w.cur, w.blocks_done, err, !blocked);
}

// ---------------------------------------------------------------------------
// BatchEnv.reset (envkit.py:616-623): rewind -> episode := -1 first.  Writes
// the live buffer in place (a reset cannot fail).

template <class Task, typename T>
__global__ void reset_kernel(EnvScalars sc, Params<T> p, Worlds<T> w, int rewind, T *obs_out) {
    constexpr int O = Task::O;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tile = reinterpret_cast<T *>(smem_raw) + (threadIdx.x / 32) * 32 * O;
    const int lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = i < sc.n;
    const int c = *w.cur;
    T o[O];
    if (live) {
        const uint32_t ep = rewind ? 0u : w.episode[c][i] + 1u;
        typename Task::W wd;
        Philox4x64 rng;
        rng.init(sc.seed, (uint64_t)(sc.env_offset + i), ep, 0);
        Task::sample(wd, rng, p, sc.wide_init != 0);
        Task::store(wd, w.state[c], i, sc.n);
        Task::obs(wd, p, o);
        w.steps[c][i] = 0;
        w.episode[c][i] = ep;
        w.needs_reset[c][i] = 0;
    } else {
#pragma unroll
        for (int j = 0; j < O; ++j) o[j] = T(0);
    }
    if (obs_out) warp_store_rows<T, O>(obs_out, i - lane, sc.n, o, tile, lane);
}

// Live state <-> float64 [N,4] / [N,2] (diagnostics, tests, Environment views).
template <class Task, typename T>
__global__ void get_state_kernel(EnvScalars sc, Worlds<T> w, double *s4, double *t2) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= sc.n) return;
    typename Task::W wd;
    Task::load(wd, w.state[*w.cur], i, sc.n);
    Task::to_f64(wd, s4 + 4 * i, t2 + 2 * i);
}

template <class Task, typename T>
__global__ void set_state_kernel(EnvScalars sc, Worlds<T> w, const double *s4, const double *t2) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= sc.n) return;
    typename Task::W wd;
    memset(&wd, 0, sizeof(wd));
    const int c = *w.cur;
    Task::load(wd, w.state[c], i, sc.n);
    Task::from_f64(wd, s4 + 4 * i, t2 + 2 * i);
    Task::store(wd, w.state[c], i, sc.n);
}

}  // namespace dk
