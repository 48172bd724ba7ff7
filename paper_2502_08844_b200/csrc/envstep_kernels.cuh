// envstep_kernels.cuh -- fused batched env step / rollout kernels.
//
// One thread owns one world for the whole launch: the state is read from HBM
// once, advanced K control steps in registers (dynamics -> reward -> obs ->
// truncation -> Philox autoreset, the whole of Environment.step +
// BatchEnv.step's autoreset, envkit.py:526-552, 630-635), and written back
// once.  Per step the only HBM traffic is the algorithmic I/O: the action in,
// obs / reward / done / trunc (and optionally the info terms) out.
//
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

__device__ __forceinline__ void record_error(unsigned long long *err, int64_t k, int64_t n,
                                             int64_t i, int code) {
    const unsigned long long key = ((unsigned long long)(k * n + i) << 2) | (unsigned long long)code;
    atomicMin(err, key);
}

// ---------------------------------------------------------------------------
// Fused K-step rollout (K == 1 is BatchEnv.step).

template <class Task, typename T, int CH>
__global__ void __launch_bounds__(256)
rollout_kernel(const T *__restrict__ actions, int64_t K, EnvScalars sc, Params<T> p, Worlds<T> w,
               StepOut<T> out, unsigned long long *err) {
    constexpr int A = Task::A, O = Task::O, I = Task::I;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tile = reinterpret_cast<T *>(smem_raw) + (threadIdx.x / 32) * 32 * (O > I ? O : I);

    // a pending (sticky) error from an earlier call: the batch is not stepped
    const bool blocked = *(volatile const unsigned long long *)err != kNoError;
    const int src = *w.cur;
    // select buffers with ternaries: runtime-indexing the by-value param
    // arrays would spill the whole struct to local memory
    T *const st_src = src ? w.state[1] : w.state[0];
    T *const st_dst = src ? w.state[0] : w.state[1];
    int32_t *const steps_src = src ? w.steps[1] : w.steps[0];
    int32_t *const steps_dst = src ? w.steps[0] : w.steps[1];
    uint32_t *const ep_src = src ? w.episode[1] : w.episode[0];
    uint32_t *const ep_dst = src ? w.episode[0] : w.episode[1];
    const uint8_t *const nr_src = src ? w.needs_reset[1] : w.needs_reset[0];
    uint8_t *const nr_dst = src ? w.needs_reset[0] : w.needs_reset[1];

    const int lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t row0 = i - lane;  // first world of this warp
    const bool live = i < sc.n && !blocked;
    const int64_t n = sc.n;

    typename Task::W wd;
    int32_t steps = 0;
    uint32_t episode = 0;
    int64_t k_usage = K;  // step at which this world would need a reset (UsageError)
    if (live) {
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
    bool ok = true;  // no non-finite action seen yet by this world

    if (!blocked) {
        // double-buffered action prefetch (CH steps per chunk)
        T abuf[2][CH][A];
        auto load_chunk = [&](int b, int64_t k0) {
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int j = 0; j < A; ++j)
                    abuf[b][c][j] = (live && k0 + c < K)
                                        ? __ldg(actions + ((k0 + c) * n + i) * A + j)
                                        : T(0);
        };

        auto run_chunk = [&](int b, int64_t k0) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int64_t k = k0 + c;
                if (k >= K) break;
                T a[A];
                bool fin = true;
#pragma unroll
                for (int j = 0; j < A; ++j) {  // min(max(float(a), -1.0), 1.0)  (envkit.py:532)
                    T v = abuf[b][c][j];
                    fin &= RealOps<T>::finite_(v);
                    if (T(-1) > v) v = T(-1);
                    if (T(1) < v) v = T(1);
                    a[j] = v;
                }
                if (!fin && ok && live && k < k_usage) {  // (envkit.py:529-531)
                    ok = false;
                    record_error(err, k, n, i, kErrInvalid);
                }
                T r = T(0);
                T info[I];
                for (int rep = 0; rep < sc.action_repeat; ++rep) {
                    Task::step(wd, a, p);
                    r += Task::reward(wd, p, info);
                }
                r /= T(sc.action_repeat);
                steps += 1;
                const bool truncated = steps >= sc.episode_length;
                T o[O];
                Task::obs(wd, p, o);
                const int64_t ko = k * n;
                if (truncated && live && sc.autoreset) {
                    if (out.term_obs) {
#pragma unroll
                        for (int j = 0; j < O; ++j) out.term_obs[(ko + i) * O + j] = o[j];
                    }
                    episode += 1;  // Environment.reset (envkit.py:502-519)
                    Philox4x64 rng;
                    rng.init(sc.seed, gidx, episode, 0);
                    Task::sample(wd, rng, p, sc.wide_init != 0);
                    steps = 0;
                    Task::obs(wd, p, o);
                }
                warp_store_rows<T, O>(out.obs + ko * O, row0, n, o, tile, lane);
                if (out.info) warp_store_rows<T, I>(out.info + ko * I, row0, n, info, tile, lane);
                if (live) {
                    out.reward[ko + i] = r;
                    out.done[ko + i] = 0;
                    out.trunc[ko + i] = truncated ? 1 : 0;
                    if (out.term_mask)
                        out.term_mask[ko + i] = (truncated && sc.autoreset) ? 1 : 0;
                }
            }
        };

        load_chunk(0, 0);
        for (int64_t k0 = 0; k0 < K; k0 += 2 * CH) {
            load_chunk(1, k0 + CH);
            run_chunk(0, k0);
            if (k0 + CH >= K) break;
            load_chunk(0, k0 + 2 * CH);
            run_chunk(1, k0 + CH);
        }

        if (live) {
            Task::store(wd, st_dst, i, n);
            steps_dst[i] = steps;
            ep_dst[i] = episode;
            // without autoreset a world that truncated in this window needs a reset
            nr_dst[i] = (!sc.autoreset && steps >= sc.episode_length) ? 1 : 0;
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
