// envstep_kernels.cuh -- fused batched env step / rollout kernels.
//
// One CTA owns a tile of 32 worlds for the whole launch: the state is read
// from HBM once, advanced K control steps on chip (dynamics -> reward -> obs ->
// truncation -> Philox autoreset, the whole of Environment.step +
// BatchEnv.step's autoreset, envkit.py:526-552, 630-635), and written back
// once.  Per step the only HBM traffic is the algorithmic I/O: the action in,
// obs / reward / done / trunc (and optionally the info terms) out.
//
//  - Warp-specialised (rollout_kernel below): a stager warp streams and
//    validates actions through a cp.async ring, a producer warp runs only the
//    serial dynamics chain of the 32 worlds, consumer warps turn its ring of
//    post-step states into rewards, observations and every global store.
//  - Validation is fused and batch-atomic: the stager checks each action as it
//    stages it (and knows up front at which step a world would need a reset);
//    the first error in reference order (step-major, then world) is kept in a
//    sticky key, and the state buffers are double-buffered so the launch
//    commits only when the whole batch was valid.
//
// Development hooks (off in the product build; tools/exp_variants.sh builds
// them as separate libraries): DK_EXP_CLOCK (%globaltimer / %clock64 timeline
// printed per launch), DK_EXP_NO_STAGER / DK_EXP_NO_CONSUMER (drop a role's
// work to measure its share), DK_EXP_EARLY_TRIGGER (PDL trigger at kernel start).
#pragma once
#include <type_traits>
#include <cstdio>

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
    int32_t solo_sm;        // rollout launcher: 1 = one CTA per SM (grid <= SM count)
    int32_t reserved1;
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

#ifdef DK_EXP_CLOCK
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

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
// fewer warps than the 592 SM sub-partitions, so the step rate is set by the
// latency of one world's serial dependency chain.  The block's warps split the
// work by dependency so that the chain runs alone in its warp:
//   stager   (1 warp): streams the actions of G-step groups into a
//            shared-memory ring (coalesced loads issued a group at a time),
//            validates them (non-finite -> sticky error, envkit.py:529-531)
//            and clips them to [-1, 1] (envkit.py:532).
//   producer (1 warp): the serial chain only -- dynamics + trig refresh,
//            step counter / truncation, Philox autoreset (out of line; it
//            also writes the post-reset observation row itself).  Each
//            post-step state goes into a group ring in shared memory
//            (layout [field][lane], conflict-free).
//   consumers (M warps): group g is handled by consumer g % M: reward + info
//            terms, observation, flags and every global store.
// Hand-offs are mbarrier phases, one per G-step group, so the chain pays
// for synchronisation once per group.  Rewards of the first action_repeat-1
// substeps are summed by the producer in the reference's order
// (reward = 0.0; reward += r, envkit.py:533-540) and the consumer adds the last.

// Publication word for stager -> producer hand-off: a release store after the
// whole warp's slot writes (bar.warp.sync orders them before lane 0's store)
// and an acquire load, which for shared::cta compiles to a plain LDS -- so the
// producer can issue it a group ahead and only consume it at the next group's
// head, instead of blocking its serial chain on an mbarrier try_wait
// (SYNCS.PHASECHK, ~250 cycles per group measured on the chain).
__device__ __forceinline__ void st_release_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void mbar_arrive_u32(uint32_t addr) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ bool mbar_test_u32(uint32_t addr, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t addr, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!done);
}

template <class Task, typename T, int TL>
struct RolloutShape {
    static constexpr int A = Task::A, O = Task::O, I = Task::I;
    static constexpr int WF = (int)(sizeof(typename Task::W) / sizeof(T));  // reals per world
    static constexpr int WPC = 32 * TL;                                      // worlds per CTA
    // steps per group: as many as keep two CTAs per SM (<= 113 KB of smem);
    // each group boundary costs the serial chain ~300 cycles (16 steps per group
    // measured 8% faster than 8 for cartpole f32)
    static constexpr int WB = WF * (int)sizeof(T);                           // bytes per world-step
    static constexpr int G = WB <= 24 ? 16 : WB <= 48 ? 8 : 4;
    static constexpr int M = 4;                                              // consumer warps
    static constexpr int NG = M + 2;                                         // state ring (groups)
    static constexpr int NA = 4;                                             // action ring (groups)
    static constexpr int NR = 8;                                             // raw action ring (groups)
    static constexpr int R = O > I ? O : I;
    static constexpr int THREADS = 32 * (M + 2);  // stager + M consumers + producer
    // shared memory carve-up
    static constexpr int NBAR = 2 * NG + NA;
    static constexpr size_t OFF_BAR = 0;  // full[NG] empty[NG] aempty[NA]
    static constexpr size_t OFF_RING = (8 * NBAR + 127) / 128 * 128;
    static constexpr size_t RING_G = (size_t)G * WF * WPC * sizeof(T);      // bytes per group
    static constexpr size_t OFF_RPART = OFF_RING + NG * RING_G;
    static constexpr size_t OFF_ACT = OFF_RPART + (size_t)NG * G * WPC * sizeof(T);
    static constexpr size_t ACT_G = (size_t)G * A * WPC * sizeof(T);
    static constexpr size_t OFF_RAW = (OFF_ACT + NA * ACT_G + 127) / 128 * 128;  // [NR][G][WPC][A]
    static constexpr size_t OFF_FLAGS = OFF_RAW + NR * ACT_G;
    static constexpr size_t OFF_GFLAG = OFF_FLAGS + (size_t)NG * G * WPC;  // [NG] u8: fast group
    static constexpr size_t OFF_CTRL = (OFF_GFLAG + NG + 15) / 16 * 16;
    static constexpr size_t SMEM = OFF_CTRL + 16;
    static_assert(SMEM <= 113 * 1024, "rollout CTA must leave room for a second CTA per SM");
};

// One world's registers <-> its column of a [field][worlds] ring slot.  Only
// the fields the consumers read (Task::SLOT_FIELDS: reward + observation) are
// passed; e.g. cartpole's raw angle is not (obs and reward use its sin/cos).
template <class Task, typename T, int STRIDE>
__device__ __forceinline__ void world_to_slot(const typename Task::W &w, T *slot, int col) {
    constexpr int WF = (int)(sizeof(typename Task::W) / sizeof(T));
    const T *f = reinterpret_cast<const T *>(&w);
#pragma unroll
    for (int j = 0; j < WF; ++j)
        if ((Task::SLOT_FIELDS >> j) & 1u) slot[j * STRIDE + col] = f[j];
}

template <class Task, typename T, int STRIDE>
__device__ __forceinline__ void slot_to_world(typename Task::W &w, const T *slot, int col) {
    constexpr int WF = (int)(sizeof(typename Task::W) / sizeof(T));
    T *f = reinterpret_cast<T *>(&w);
#pragma unroll
    for (int j = 0; j < WF; ++j) f[j] = ((Task::SLOT_FIELDS >> j) & 1u) ? slot[j * STRIDE + col] : T(0);
}

// Environment.reset (envkit.py:502-519) of one world inside a rollout: the
// next Philox stream of (seed, env, episode) -> sample_initial; writes the
// post-reset observation row (the step's returned obs, envkit.py:634).  Out of
// line: taken once per episode_length steps.
template <class Task, typename T>
__device__ __noinline__ typename Task::W autoreset_world(uint64_t seed, uint64_t gidx,
                                                         uint32_t episode, Params<T> p, int wide,
                                                         T *obs_row) {
    typename Task::W wd;
    Philox4x64 rng;
    rng.init(seed, gidx, episode, 0);
    Task::sample(wd, rng, p, wide != 0);
    T o[Task::O];
    Task::obs(wd, p, o);
#pragma unroll
    for (int j = 0; j < Task::O; ++j) obs_row[j] = o[j];
    return wd;
}

// TL = 32-world tiles per CTA (the launcher uses TL = 1: interleaving two
// worlds' chains in one producer lane, TL = 2 on 64-world CTAs, was measured
// 1.7x slower per world at 8192 worlds -- the chains did not overlap and 20 of
// 148 SMs sat idle -- profiles/r01_ncu_summary.md).
template <class Task, typename T, bool R1, int TL>
__global__ void __launch_bounds__(RolloutShape<Task, T, TL>::THREADS)
rollout_kernel(const T *__restrict__ actions, int64_t K, EnvScalars sc, Params<T> p, Worlds<T> w,
               StepOut<T> out, unsigned long long *err) {
    using S = RolloutShape<Task, T, TL>;
    constexpr int A = Task::A, O = Task::O, I = Task::I, WF = S::WF, G = S::G, M = S::M;
    constexpr int NG = S::NG, NA = S::NA, WPC = S::WPC;
    extern __shared__ __align__(16) unsigned char smem[];
    T *ring = reinterpret_cast<T *>(smem + S::OFF_RING);    // [NG][G][WF][WPC]
    T *rpart = reinterpret_cast<T *>(smem + S::OFF_RPART);  // [NG][G][WPC]
    T *aring = reinterpret_cast<T *>(smem + S::OFF_ACT);    // [NA][G][A][WPC]
    uint8_t *flags = smem + S::OFF_FLAGS;                   // [NG][G][WPC] bit0 trunc, bit1 reset
    uint8_t *gflag = smem + S::OFF_GFLAG;                   // [NG] 1: no world truncated in the group
    int *ctrl = reinterpret_cast<int *>(smem + S::OFF_CTRL);
    const uint32_t bar = smem_u32(smem + S::OFF_BAR);
    const uint32_t full_b = bar, empty_b = bar + 8 * NG, aempty_b = bar + 16 * NG;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef DK_EXP_CLOCK
    const unsigned long long g_entry = gtimer();
    unsigned long long g_loop0 = 0, g_loop1 = 0, g_first = 0;
#endif
    const int64_t n = sc.n;
    const int64_t cta0 = (int64_t)blockIdx.x * WPC;  // first world of this CTA
    const int K32 = (int)K;  // host guarantees K < 2^31
    const int ngroups = (K32 + G - 1) / G;

    // programmatic dependent launch: everything below may read what the
    // previous grid on the stream wrote (error word, live buffer index, state)
#ifdef DK_EXP_EARLY_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef DK_EXP_CLOCK
    const unsigned long long g_dep = gtimer();
#endif
    if (threadIdx.x == 0) {
        // a pending (sticky) error from an earlier call: the batch is not
        // stepped.  Read once so the whole block takes the same branch.
        ctrl[0] = *(volatile const unsigned long long *)err != kNoError;
        ctrl[1] = *w.cur;
        ctrl[3] = 0;  // groups published by the stager
        unsigned slot0;  // hardware warp slot of warp 0 (slot % 4 = SM sub-partition)
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(slot0));
        ctrl[2] = (int)slot0;
        uint64_t *b = reinterpret_cast<uint64_t *>(smem + S::OFF_BAR);
#pragma unroll
        for (int d = 0; d < S::NBAR; ++d) mbar_init(&b[d], 32);
    }
    __syncthreads();
    const bool blocked = ctrl[0] != 0;
    const int src = ctrl[1];
    // warp roles: 0 stager, 1..M consumers, M+1 producer
    // Warp roles (0 stager, 1..M consumers, M+1 producer), placed by the warp
    // slots the CTA actually got: warp slot s runs on SM sub-partition s % 4
    // and the arbiter prefers the highest slot (B300 microarchitecture notes;
    // tools/micro/warpmap.cu shows a co-resident second CTA takes slots 6-11).
    //   first CTA of an SM  (slots 0-5, SMSPs 0 1 2 3 0 1): producer = warp 5
    //     on SMSP 1, stager = warp 0 on SMSP 0;
    //   second CTA (slots 6-11, SMSPs 2 3 0 1 2 3): producer = warp 4, the top
    //     slot of SMSP 2, stager = warp 1 on SMSP 3.
    // Each producer then shares its sub-partition with two consumers only
    // (busiest SMSP 113 instead of 121 issue slots per step); 10% faster at
    // 8192 worlds than a fixed warp-4 producer (measured).  The mapping is a
    // permutation for any slot base, so it only affects speed.
    int role;
    if ((ctrl[2] & 3) == 2) {
        role = warp == 4 ? M + 1 : warp == 1 ? 0 : warp == 0 ? 1 : warp == 5 ? 4 : warp;
    } else {
        // one CTA per SM (few worlds): the producer alone on sub-partition 3 and
        // the stager alone on 2, the consumers on 0 / 1 (1024 worlds: 6% faster;
        // with a second CTA on the SM this placement was 5% slower)
        if (sc.solo_sm)
            role = warp == 3 ? M + 1 : warp == 2 ? 0 : warp == 0 ? 1 : warp == 1 ? 2 : warp == 4 ? 3 : 4;
        else
            role = warp == 5 ? M + 1 : warp;
    }
    // buffer selection by ternary: runtime-indexing the by-value param arrays
    // would spill the whole struct to local memory
    const int32_t *steps_src = src ? w.steps[1] : w.steps[0];
    const uint8_t *nr_src = src ? w.needs_reset[1] : w.needs_reset[0];

    // step at which world i would need a reset (UsageError, envkit.py:527-528)
    auto usage_step = [&](int64_t i, int32_t steps) -> int {
        if (i >= n) return K32;
        if (nr_src[i]) return 0;
        if (!sc.autoreset && (int64_t)sc.episode_length - steps < K)
            return (int)((int64_t)sc.episode_length - steps);
        return K32;
    };

    if (blocked) {
        // nothing
    } else if (role == M + 1) {
        // ------------------------------------------------------------ producer
        const T *st_src = src ? w.state[1] : w.state[0];
        T *st_dst = src ? w.state[0] : w.state[1];
        int32_t *steps_dst = src ? w.steps[0] : w.steps[1];
        const uint32_t *ep_src = src ? w.episode[1] : w.episode[0];
        uint32_t *ep_dst = src ? w.episode[0] : w.episode[1];
        uint8_t *nr_dst = src ? w.needs_reset[0] : w.needs_reset[1];

        typename Task::W wd[TL];
        int32_t steps[TL];
        uint32_t episode[TL];
        bool live[TL], can_reset[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            const int64_t i = cta0 + t * 32 + lane;
            live[t] = i < n;
            steps[t] = 0;
            episode[t] = 0;
            if (live[t]) {
                Task::load(wd[t], st_src, i, n);
                steps[t] = steps_src[i];
                episode[t] = ep_src[i];
            } else {
                Task::zero(wd[t]);
            }
            const int ku = usage_step(i, steps[t]);
            if (ku < K32) record_error(err, ku, n, i, kErrUsage);
            Task::refresh(wd[t]);
            can_reset[t] = sc.autoreset && live[t];
        }

        auto step_body = [&](int t, int s, int k, T *ring_g, T *rp_g, uint8_t *fl_g, const T *u) {
            const int col = t * 32 + lane;
            T rp = T(0);
            Task::step_u(wd[t], u, p);
            if (!R1) {
                for (int rep = 1; rep < sc.action_repeat; ++rep) {
                    T inf[I];
                    rp += Task::reward(wd[t], p, inf);
                    Task::step_u(wd[t], u, p);
                }
            }
            steps[t] += 1;
            const bool truncated = steps[t] >= sc.episode_length;
            const bool reset = truncated && can_reset[t];
            world_to_slot<Task, T, WPC>(wd[t], ring_g + s * WF * WPC, col);
            if (!R1) rp_g[s * WPC + col] = rp;
            fl_g[s * WPC + col] = (uint8_t)((truncated ? 1 : 0) | (reset ? 2 : 0));
            if (__builtin_expect(reset, 0)) {
                episode[t] += 1;
                steps[t] = 0;
                const int64_t i = cta0 + col;
                wd[t] = autoreset_world<Task, T>(sc.seed, (uint64_t)(sc.env_offset + i),
                                                 episode[t], p, sc.wide_init,
                                                 out.obs + ((int64_t)k * n + i) * O);
            }
        };

        // Group loop.  Everything the next group's head needs (its fast/slow
        // decision, the stager's publication count, ring indices) is computed
        // inside the current group's body, where it schedules under the chain's
        // latency; the head itself is one branch on a ready predicate.  (A
        // head with a constant load -> compare -> vote -> branch sequence cost
        // ~200 cycles per group of the serial chain, measured.)
        //
        // fast group: no world of this warp reaches episode_length inside it
        // (124 of 125 groups at episode_length 1000), so the chain carries no
        // step counting, flags or reset branch.
        auto group_is_fast = [&](int gg) -> bool {
            bool near_end = false;
#pragma unroll
            for (int t = 0; t < TL; ++t) near_end |= live[t] && steps[t] + G >= sc.episode_length;
            return (gg * G + G <= K32) && !__any_sync(0xffffffffu, near_end);
        };
        // groups published by the stager (acquire-loaded one group ahead)
        const uint32_t staged_a = smem_u32(&ctrl[3]);
#ifdef DK_EXP_CLOCK
        g_loop0 = gtimer();
#endif
        uint32_t avail = ld_acquire_u32(staged_a);
        while (avail < 1u) avail = ld_acquire_u32(staged_a);
#ifdef DK_EXP_CLOCK
        g_first = gtimer();
#endif
        bool fast = group_is_fast(0);
        int sb = 0, ab = 0;
        // group g's hand-off arrives (release: they wait for the group's ring
        // stores to drain, stalling in-order issue) are issued after the first
        // step of group g + 1, by when the stores have drained (+1.3%, measured)
        int pend_sb = -1, pend_ab = 0;
        auto flush_arrive = [&]() {
            if (pend_sb >= 0) {
                mbar_arrive_u32(aempty_b + 8 * pend_ab);
                mbar_arrive_u32(full_b + 8 * pend_sb);
                pend_sb = -1;
            }
        };
#pragma unroll 1
        for (int g = 0; g < ngroups; ++g) {
            const uint32_t avail_next = ld_acquire_u32(staged_a);  // consumed at the next head
            T *ring_g = ring + (size_t)sb * G * WF * WPC;
            T *rp_g = rpart + (size_t)sb * G * WPC;
            uint8_t *fl_g = flags + sb * G * WPC;
            const T *act_g = aring + (size_t)ab * G * A * WPC;
            const int k0 = g * G;
            bool fast_next;
            if (fast) {
                T u[G][TL][A];  // the whole group's controls, loaded ahead of the chains
#pragma unroll
                for (int s = 0; s < G; ++s)
#pragma unroll
                    for (int t = 0; t < TL; ++t)
#pragma unroll
                        for (int j = 0; j < A; ++j)
                            u[s][t][j] = act_g[(s * A + j) * WPC + t * 32 + lane];
#pragma unroll
                for (int t = 0; t < TL; ++t) steps[t] += G;
                fast_next = group_is_fast(g + 1);
#pragma unroll
                for (int s = 0; s < G; ++s) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) {  // independent chains interleave here
                        T rp = T(0);
                        Task::step_u(wd[t], u[s][t], p);
                        if (!R1) {
                            for (int rep = 1; rep < sc.action_repeat; ++rep) {
                                T inf[I];
                                rp += Task::reward(wd[t], p, inf);
                                Task::step_u(wd[t], u[s][t], p);
                            }
                            rp_g[s * WPC + t * 32 + lane] = rp;
                        }
                        world_to_slot<Task, T, WPC>(wd[t], ring_g + s * WF * WPC, t * 32 + lane);
                    }
                    if (s == 0) flush_arrive();
                }
            } else {
                flush_arrive();
#pragma unroll 1
                for (int s = 0; s < min(G, K32 - k0); ++s) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) {
                        T u[A];
#pragma unroll
                        for (int j = 0; j < A; ++j) u[j] = act_g[(s * A + j) * WPC + t * 32 + lane];
                        step_body(t, s, k0 + s, ring_g, rp_g, fl_g, u);
                    }
                }
                fast_next = group_is_fast(g + 1);
            }
            if (lane == 0) gflag[sb] = fast ? 1 : 0;
            pend_sb = sb;
            pend_ab = ab;
            sb = sb + 1 == NG ? 0 : sb + 1;
            ab = ab + 1 == NA ? 0 : ab + 1;
            avail = avail_next;
            // the stager publishes group g+1 once its actions are staged AND its
            // state-ring slot is free (it waits on empty for us); normally it
            // already has, and this loop is not entered
            while (avail < (uint32_t)(g + 2) && g + 1 < ngroups) avail = ld_acquire_u32(staged_a);
            fast = fast_next;
        }
        flush_arrive();
#ifdef DK_EXP_CLOCK
        g_loop1 = gtimer();
#endif
        // this CTA's chain is done: the next rollout on the stream may start
        // launching (it still waits for this grid to finish before reading)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            const int64_t i = cta0 + t * 32 + lane;
            if (live[t]) {
                Task::store(wd[t], st_dst, i, n);
                steps_dst[i] = steps[t];
                ep_dst[i] = episode[t];
                // without autoreset a world that truncated in this window needs a reset
                nr_dst[i] = (!sc.autoreset && steps[t] >= sc.episode_length) ? 1 : 0;
            }
        }
    } else if (role == 0) {
        // ------------------------------------------------------------ stager
        // raw actions stream into an NR-group shared-memory ring through
        // cp.async (each lane copies its own worlds' values), NR-1 groups ahead
        // of the group being validated.  (1-D TMA bulk copies of the 128 B
        // rows were measured 24% slower end to end: eight tiny bulk ops per
        // group serialise in the copy engine and the producer starved.)
        constexpr int NR = S::NR;
        constexpr int ROWV = WPC * A;  // values per row slot
        T *raw = reinterpret_cast<T *>(smem + S::OFF_RAW);  // [NR][G][WPC][A]
        int ku[TL];
        bool ok[TL], live[TL];
        const T *arow[TL];
        int64_t astep[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            const int64_t i = cta0 + t * 32 + lane;
            live[t] = i < n;
            ku[t] = usage_step(i, live[t] ? steps_src[i] : 0);
            ok[t] = true;
            arow[t] = actions + (live[t] ? i * A : 0);
            astep[t] = live[t] ? n * A : 0;
        }
        auto issue = [&](int g) {
            T *dst = raw + (size_t)(g % NR) * G * ROWV;
            const int k0 = g * G;
#pragma unroll
            for (int s = 0; s < G; ++s)
#pragma unroll
                for (int t = 0; t < TL; ++t) {
                    const bool v = live[t] && k0 + s < K32;
#pragma unroll
                    for (int j = 0; j < A; ++j)
                        cp_async_ca<sizeof(T)>(dst + s * ROWV + (t * 32 + lane) * A + j,
                                               v ? arow[t] + (int64_t)(k0 + s) * astep[t] + j
                                                 : actions,
                                               v);
                }
            cp_async_commit();  // one group per call (empty groups past K keep the count)
        };
        // Vectorised staging (full 32-world tile, 16-byte aligned action rows):
        // each lane owns one 16-byte chunk of a row -- the same worlds in every
        // row -- so a group is G * ROWV / VW / 32 cp.async.16 per lane instead of
        // G * A scalar copies, and validation / control / staging run on
        // 16-byte smem loads (pendulum: the stager was 23% of the step).
        constexpr int VW = 16 / (int)sizeof(T);   // values per chunk
        constexpr int CPR = ROWV / VW;            // chunks per row
        constexpr int WPK = VW / A;               // worlds per chunk
        constexpr bool VEC_SHAPE = TL == 1 && (ROWV % VW) == 0 && (VW % A) == 0 &&
                                   CPR <= 32 && (32 % CPR) == 0 && ((G * CPR) % 32) == 0;
        const bool vec = VEC_SHAPE && cta0 + WPC <= n &&
                         ((reinterpret_cast<uintptr_t>(actions + cta0 * A) |
                           (uintptr_t)(n * A * (int64_t)sizeof(T))) & 15) == 0;
        if constexpr (VEC_SHAPE) {
            if (vec) {
                const int c = lane % CPR, r0 = lane / CPR;  // chunk of the row; first row
                constexpr int RSTEP = 32 / CPR, ITER = G / RSTEP;
                int kuv[WPK];
#pragma unroll
                for (int k = 0; k < WPK; ++k) {
                    const int64_t i = cta0 + c * WPK + k;
                    kuv[k] = usage_step(i, steps_src[i]);
                }
                const T *abase = actions + (cta0 * A + c * VW);
                const int64_t rowstride = n * A;
                auto issue_v = [&](int g) {
                    T *dst = raw + (size_t)(g % NR) * G * ROWV;
                    const int k0 = g * G;
#pragma unroll
                    for (int m = 0; m < ITER; ++m) {
                        const int srow = r0 + m * RSTEP;
                        const bool v = k0 + srow < K32;
                        cp_async_ca<16>(dst + srow * ROWV + c * VW,
                                        v ? abase + (int64_t)(k0 + srow) * rowstride : actions, v);
                    }
                    cp_async_commit();
                };
#pragma unroll 1
                for (int g = 0; g < NR - 1; ++g) issue_v(g);
#pragma unroll 1
                for (int g = 0; g < ngroups; ++g) {
                    issue_v(g + NR - 1);
                    cp_async_wait<NR - 1>();
                    __syncwarp();  // every lane's copies landed (each lane reads its own chunks)
                    const int ab = g % NA;
                    const int k0 = g * G;
                    const T *src_g = raw + (size_t)(g % NR) * G * ROWV;
                    if (g >= NA) mbar_wait_u32(aempty_b + 8 * ab, (uint32_t)(g / NA - 1) & 1u);
                    T *act_g = aring + (size_t)ab * G * A * WPC;
#pragma unroll
                    for (int m = 0; m < ITER; ++m) {
                        const int srow = r0 + m * RSTEP;
                        T vals[VW];
                        if constexpr (sizeof(T) == 4) {
                            const float4 x = *reinterpret_cast<const float4 *>(
                                src_g + srow * ROWV + c * VW);
                            vals[0] = x.x; vals[1] = x.y; vals[2] = x.z; vals[3] = x.w;
                        } else {
                            const double2 x = *reinterpret_cast<const double2 *>(
                                src_g + srow * ROWV + c * VW);
                            vals[0] = x.x; vals[1] = x.y;
                        }
                        T us[WPK][A];
#pragma unroll
                        for (int k = 0; k < WPK; ++k) {
                            bool fin = true;
                            T a[A];
#pragma unroll
                            for (int j = 0; j < A; ++j) {
                                fin &= RealOps<T>::finite_(vals[k * A + j]);
                                a[j] = fmin(fmax(vals[k * A + j], T(-1)), T(1));  // envkit.py:532
                            }
                            Task::control(a, p, us[k]);
                            if (__builtin_expect(!fin && k0 + srow < kuv[k] && k0 + srow < K32, 0))
                                record_error(err, k0 + srow, n, cta0 + c * WPK + k, kErrInvalid);
                        }
                        if constexpr (A == 1 && sizeof(T) == 4) {
                            *reinterpret_cast<float4 *>(act_g + srow * WPC + c * WPK) =
                                make_float4(us[0][0], us[1][0], us[2][0], us[3][0]);
                        } else {
#pragma unroll
                            for (int k = 0; k < WPK; ++k)
#pragma unroll
                                for (int j = 0; j < A; ++j)
                                    act_g[(srow * A + j) * WPC + c * WPK + k] = us[k][j];
                        }
                    }
                    mbar_wait_u32(empty_b + 8 * (g % NG), (uint32_t)(g / NG) & 1u);
                    __syncwarp();
                    if (lane == 0) st_release_u32(smem_u32(&ctrl[3]), (uint32_t)(g + 1));
                }
                cp_async_wait<0>();
            }
        }
#pragma unroll 1
        for (int g = 0; g < NR - 1 && !vec; ++g) issue(g);
#pragma unroll 1
        for (int g = 0; g < ngroups && !vec; ++g) {
#ifdef DK_EXP_NO_STAGER
            {
                const int ab = g % NA;
                if (g >= NA) mbar_wait_u32(aempty_b + 8 * ab, (uint32_t)(g / NA - 1) & 1u);
                mbar_wait_u32(empty_b + 8 * (g % NG), (uint32_t)(g / NG) & 1u);
                __syncwarp();
                if (lane == 0) st_release_u32(smem_u32(&ctrl[3]), (uint32_t)(g + 1));
                continue;
            }
#endif
            issue(g + NR - 1);        // into the slot read in the previous iteration
            cp_async_wait<NR - 1>();  // this lane's copies of group g have landed
            const int ab = g % NA;
            const int k0 = g * G;
            const T *src_g = raw + (size_t)(g % NR) * G * ROWV;
            T v[G][TL][A];
#pragma unroll
            for (int s = 0; s < G; ++s)
#pragma unroll
                for (int t = 0; t < TL; ++t)
#pragma unroll
                    for (int j = 0; j < A; ++j)
                        v[s][t][j] = src_g[s * ROWV + (t * 32 + lane) * A + j];
            if (g >= NA) mbar_wait_u32(aempty_b + 8 * ab, (uint32_t)(g / NA - 1) & 1u);
            T *act_g = aring + (size_t)ab * G * A * WPC;
#pragma unroll
            for (int s = 0; s < G; ++s)
#pragma unroll
                for (int t = 0; t < TL; ++t) {
                    bool fin = true;
                    T a[A], u[A];
#pragma unroll
                    for (int j = 0; j < A; ++j) {
                        fin &= RealOps<T>::finite_(v[s][t][j]);
                        a[j] = fmin(fmax(v[s][t][j], T(-1)), T(1));  // envkit.py:532
                    }
                    // the force / torque clip of step_dynamics, off the producer's chain
                    Task::control(a, p, u);
#pragma unroll
                    for (int j = 0; j < A; ++j) act_g[(s * A + j) * WPC + t * 32 + lane] = u[j];
                    if (__builtin_expect(
                            !fin && ok[t] && live[t] && k0 + s < ku[t] && k0 + s < K32, 0)) {
                        ok[t] = false;  // envkit.py:529-531
                        record_error(err, k0 + s, n, cta0 + t * 32 + lane, kErrInvalid);
                    }
                }
            // the producer's state-ring slot for this group must be free too
            // (phase 0 pre-armed by consumer 0)
            mbar_wait_u32(empty_b + 8 * (g % NG), (uint32_t)(g / NG) & 1u);
            __syncwarp();
            if (lane == 0) st_release_u32(smem_u32(&ctrl[3]), (uint32_t)(g + 1));
        }
        cp_async_wait<0>();
    } else if (role > 0) {
        // ------------------------------------------------------------ consumers
        const int c = role - 1;  // consumer index 0..M-1
        const T inv_rep = T(sc.action_repeat);
        const bool has_info = out.info != nullptr, has_mask = out.term_mask != nullptr;
        if (c == 0) {
#pragma unroll 1
            for (int d = 0; d < NG; ++d) mbar_arrive_u32(empty_b + 8 * d);  // slots start free
        }
        // FULL: all 32 rows of the tile exist -> no per-element bounds checks
        // FAST (no world of the group truncates, no reset): no flag loads, no
        // terminal-observation branch, the three flag bytes are constant zeros
        // per-step strides, hoisted (the compiler otherwise re-derives the
        // 64-bit products from the constant bank every step)
        const int64_t step_obs = n * O, step_info = n * I;
        const bool idx32 = (int64_t)K32 * n * (O > I ? O : I) < (int64_t)1 << 31;
        auto run_tile = [&](auto full_c, auto fast_c, int t, int g, const T *ring_g,
                            const T *rp_g, const uint8_t *fl_g) {
            constexpr bool FULL = decltype(full_c)::value;
            constexpr bool FAST = decltype(fast_c)::value;
            const int col = t * 32 + lane;
            const int64_t row0 = cta0 + t * 32;
            const int64_t i = row0 + lane;
            const bool in_range = i < n;
            const int kend = min(G, K32 - g * G);
            const int64_t kb = (int64_t)g * G * n;  // element row of step g*G
            // fast full tiles of the wider-observation tasks: a 32-bit element
            // index with each store address one IMAD.WIDE, instead of six 64-bit
            // pointer streams (+2-3% for cartpole / acrobot / reacher; the
            // 3-value pendulum row measured 3% slower, so it keeps the pointers)
            if constexpr (FAST && FULL && O >= 5) {
                if (idx32) {
                    uint32_t e = (uint32_t)(kb + i);
#pragma unroll 1
                    for (int s = 0; s < kend; ++s) {
                        typename Task::W wd;
                        slot_to_world<Task, T, WPC>(wd, ring_g + s * WF * WPC, col);
                        T info[I];
                        const T r = R1 ? (T(0) + Task::reward(wd, p, info))
                                       : (rp_g[s * WPC + col] + Task::reward(wd, p, info)) / inv_rep;
                        T o[O];
                        Task::obs(wd, p, o);
                        T *ob = out.obs + (uint64_t)e * O;
#pragma unroll
                        for (int j = 0; j < O; ++j) ob[j] = o[j];
                        if (has_info) {
                            T *ib = out.info + (uint64_t)e * I;
#pragma unroll
                            for (int j = 0; j < I; ++j) ib[j] = info[j];
                        }
                        out.reward[e] = r;
                        out.done[e] = 0;
                        out.trunc[e] = 0;
                        if (has_mask) out.term_mask[e] = 0;
                        e += (uint32_t)n;
                    }
                    return;
                }
            }
            T *obs_p = out.obs + (kb + row0) * O;
            T *info_p = has_info ? out.info + (kb + row0) * I : nullptr;
            T *rew_p = out.reward + kb + i;
            uint8_t *done_p = out.done + kb + i, *trunc_p = out.trunc + kb + i;
            uint8_t *mask_p = has_mask ? out.term_mask + kb + i : nullptr;
#pragma unroll 1
            for (int s = 0; s < kend; ++s) {
                typename Task::W wd;
                slot_to_world<Task, T, WPC>(wd, ring_g + s * WF * WPC, col);
                const uint8_t fl = FAST ? 0 : fl_g[s * WPC + col];
                const bool reset = !FAST && (fl & 2) != 0;
                T info[I];
                const T r = R1 ? (T(0) + Task::reward(wd, p, info))
                               : (rp_g[s * WPC + col] + Task::reward(wd, p, info)) / inv_rep;
                T o[O];
                Task::obs(wd, p, o);
                if (!FAST && __builtin_expect(reset, 0) && out.term_obs) {
                    T *tt = out.term_obs + (kb + (int64_t)s * n + i) * O;
#pragma unroll
                    for (int j = 0; j < O; ++j) tt[j] = o[j];
                }
                // (the producer wrote the post-reset observation of reset worlds)
                // Row stores straight from registers: each instruction spans the
                // warp's contiguous 32-row block and the L2 merges the partial
                // sectors, so no DRAM traffic is wasted -- and it costs 1 issue
                // slot per value instead of 3 for a shared-memory transpose
                // (issue slots, not bandwidth, bound this kernel at 8K worlds).
                if (FULL || in_range) {
                    if (!reset) {
#pragma unroll
                        for (int j = 0; j < O; ++j) obs_p[lane * O + j] = o[j];
                    }
                    if (has_info) {
#pragma unroll
                        for (int j = 0; j < I; ++j) info_p[lane * I + j] = info[j];
                    }
                }
                if (FULL || in_range) {
                    *rew_p = r;
                    *done_p = 0;
                    *trunc_p = FAST ? 0 : fl & 1;
                    if (has_mask) *mask_p = FAST ? 0 : (reset ? 1 : 0);
                }
                obs_p += step_obs;
                info_p += step_info;
                rew_p += n;
                done_p += n;
                trunc_p += n;
                mask_p += n;
            }
        };
#pragma unroll 1
        for (int g = c; g < ngroups; g += M) {
            const int sb = g % NG;
            mbar_wait_u32(full_b + 8 * sb, (uint32_t)(g / NG) & 1u);
            const T *ring_g = ring + (size_t)sb * G * WF * WPC;
            const T *rp_g = rpart + (size_t)sb * G * WPC;
            const uint8_t *fl_g = flags + sb * G * WPC;
            const bool fast = gflag[sb] != 0;
#ifndef DK_EXP_NO_CONSUMER
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                if (cta0 + t * 32 + 32 <= n) {
                    if (fast)
                        run_tile(std::true_type{}, std::true_type{}, t, g, ring_g, rp_g, fl_g);
                    else
                        run_tile(std::true_type{}, std::false_type{}, t, g, ring_g, rp_g, fl_g);
                } else if (cta0 + t * 32 < n) {  // (fast groups write no flags)
                    if (fast)
                        run_tile(std::false_type{}, std::true_type{}, t, g, ring_g, rp_g, fl_g);
                    else
                        run_tile(std::false_type{}, std::false_type{}, t, g, ring_g, rp_g, fl_g);
                }
            }
#endif
            mbar_arrive_u32(empty_b + 8 * sb);
        }
    }
    finish_launch(w.cur, w.blocks_done, err, !blocked);
#ifdef DK_EXP_CLOCK
    const unsigned long long g_exit = gtimer();
    if (role == M + 1 && lane == 0 && (blockIdx.x == 0 || blockIdx.x == 200))
        printf("gt cta %d: dep-wait %llu, to loop %llu, first group %llu, loop %llu, drain %llu ns\n",
               (int)blockIdx.x, g_dep - g_entry, g_loop0 - g_dep, g_first - g_loop0,
               g_loop1 - g_first, g_exit - g_loop1);
#endif
}

// ---------------------------------------------------------------------------
// One control step (K = 1: BatchEnv.step, the PPO rollout's per-step env call)
// without the rollout kernel's staging ring: its fixed cost (action staging, the
// producer / consumer hand-off, the drain: ~6 us at 8192 worlds) is most of a
// single step.  One thread per world does what the stager, the producer and a
// consumer do for that world in rollout_kernel, in the same order and with the
// same arithmetic: validate / clip / control the action (envkit.py:529-532),
// step (action_repeat loop, reward averaged), count, truncate, reward /
// observation / info of the post-step state, terminal observation and Philox
// auto-reset, state into the other buffer; the last block commits the buffer
// flip unless an error was recorded (batch-atomic, as rollout_kernel).
template <class Task, typename T, bool R1>
__global__ void __launch_bounds__(64)
step1_kernel(const T *__restrict__ actions, EnvScalars sc, Params<T> p, Worlds<T> w,
             StepOut<T> out, unsigned long long *err) {
    constexpr int A = Task::A, O = Task::O, I = Task::I;
    __shared__ int ctrl[2];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        ctrl[0] = *(volatile const unsigned long long *)err != kNoError;
        ctrl[1] = *w.cur;
    }
    __syncthreads();
    const bool blocked = ctrl[0] != 0;
    const int src = ctrl[1];
    const int64_t n = sc.n;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (!blocked && i < n) {
        const T *st_src = src ? w.state[1] : w.state[0];
        T *st_dst = src ? w.state[0] : w.state[1];
        const int32_t *steps_src = src ? w.steps[1] : w.steps[0];
        int32_t *steps_dst = src ? w.steps[0] : w.steps[1];
        const uint32_t *ep_src = src ? w.episode[1] : w.episode[0];
        uint32_t *ep_dst = src ? w.episode[0] : w.episode[1];
        const uint8_t *nr_src = src ? w.needs_reset[1] : w.needs_reset[0];
        uint8_t *nr_dst = src ? w.needs_reset[0] : w.needs_reset[1];
        typename Task::W wd;
        Task::load(wd, st_src, i, n);
        int32_t steps = steps_src[i];
        uint32_t episode = ep_src[i];
        // step at which the world would need a reset (UsageError, envkit.py:527-528)
        int ku = 1;
        if (nr_src[i]) ku = 0;
        else if (!sc.autoreset && (int64_t)sc.episode_length - steps < 1)
            ku = (int)((int64_t)sc.episode_length - steps);
        if (ku < 1) record_error(err, ku, n, i, kErrUsage);
        Task::refresh(wd);
        // the stager's validation, clip and control
        bool fin = true;
        T a[A], u[A];
#pragma unroll
        for (int j = 0; j < A; ++j) {
            const T v = actions[i * A + j];
            fin &= RealOps<T>::finite_(v);
            a[j] = fmin(fmax(v, T(-1)), T(1));  // envkit.py:532
        }
        Task::control(a, p, u);
        if (!fin && 0 < ku) record_error(err, 0, n, i, kErrInvalid);  // envkit.py:529-531
        // the producer's step
        T rp = T(0);
        Task::step_u(wd, u, p);
        if (!R1) {
            for (int rep = 1; rep < sc.action_repeat; ++rep) {
                T inf[I];
                rp += Task::reward(wd, p, inf);
                Task::step_u(wd, u, p);
            }
        }
        steps += 1;
        const bool truncated = steps >= sc.episode_length;
        const bool reset = truncated && sc.autoreset;
        // the consumer's outputs of the post-step state
        T info[I];
        const T r = R1 ? (T(0) + Task::reward(wd, p, info))
                       : (rp + Task::reward(wd, p, info)) / T(sc.action_repeat);
        T o[O];
        Task::obs(wd, p, o);
        if (reset && out.term_obs) {
#pragma unroll
            for (int j = 0; j < O; ++j) out.term_obs[i * O + j] = o[j];
        }
        if (!reset) {
#pragma unroll
            for (int j = 0; j < O; ++j) out.obs[i * O + j] = o[j];
        }
        if (out.info) {
#pragma unroll
            for (int j = 0; j < I; ++j) out.info[i * I + j] = info[j];
        }
        out.reward[i] = r;
        out.done[i] = 0;
        out.trunc[i] = truncated ? 1 : 0;
        if (out.term_mask) out.term_mask[i] = reset ? 1 : 0;
        if (__builtin_expect(reset, 0)) {
            episode += 1;
            steps = 0;
            wd = autoreset_world<Task, T>(sc.seed, (uint64_t)(sc.env_offset + i), episode, p,
                                          sc.wide_init, out.obs + i * O);
        }
        Task::store(wd, st_dst, i, n);
        steps_dst[i] = steps;
        ep_dst[i] = episode;
        nr_dst[i] = (!sc.autoreset && steps >= sc.episode_length) ? 1 : 0;
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
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
