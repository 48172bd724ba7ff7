// pixels.cuh -- the cartpole pixel observation path on device (SURVEY.md §8f
// rank 2): the software rasteriser, brightness post-process, ITU-R 601 luma
// and the three-frame grayscale stack of `cartpole-balance-pixels`.
//
//   batch_render            pixelrender.py:73-131
//   randomize_visuals       pixelrender.py:134-153 (+ envkit.py:515-518 keying)
//   brightness_postprocess  pixelrender.py:156-161
//   rgb_to_gray             pixelrender.py:184-186
//   FrameStack              pixelrender.py:164-181 / Environment._observe envkit.py:555-577
//
// Design: a frame is a function of (cart x, cos th, sin th, visuals) only, so a
// world's stacked observation is rendered from its last three states instead of
// being read back from HBM: the kernel writes the [H, W, 3] stack once and reads
// nothing per pixel (write-only HBM traffic).  Each pixel is one of three
// colours, so a world's three gray levels are computed once per frame.
// float64 arithmetic follows the reference's NumPy expression order with one
// rounding per operation (_rn intrinsics).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "envmath.cuh"

namespace dk {

// VisualParams packed as 12 doubles: background rgb, cart rgb, pole rgb,
// camera offset x, y, zoom; + brightness = 13.
constexpr int kVis = 13;

struct PixFrame {  // one state to draw: cart x and the pole direction
    double x, c, s;
};

// Classify pixel (row, col) of a w x h view: 0 background, 1 cart, 2 pole.
__device__ __forceinline__ int pix_class(const double *vis, double pole_len, int w, int h, int row,
                                         int col, const PixFrame &f) {
    const double px = __dsub_rn(__dadd_rn((double)col, 0.5), __ddiv_rn((double)w, 2.0));
    const double py = __dsub_rn(__ddiv_rn((double)h, 2.0), __dadd_rn((double)row, 0.5));
    // _world_to_pixel_scale: w / (2.0 * _VIEW_HALF_WIDTH) * zoom
    const double scale = __dmul_rn(__ddiv_rn((double)w, __dmul_rn(2.0, 2.4)), vis[11]);
    const double wx = __dadd_rn(__ddiv_rn(px, scale), vis[9]);
    const double wy = __dadd_rn(__ddiv_rn(py, scale), vis[10]);
    int cls = 0;
    if (fabs(__dsub_rn(wx, f.x)) <= 0.36 / 2 && fabs(__dsub_rn(wy, 0.0)) <= 0.22 / 2) cls = 1;
    // pole segment from the pivot (cart top) to pivot + l (sin th, cos th)
    const double p0 = f.x, p1 = __dadd_rn(0.0, 0.22 / 2);
    const double d0 = __dsub_rn(__dadd_rn(p0, __dmul_rn(pole_len, f.s)), p0);
    const double d1 = __dsub_rn(__dadd_rn(p1, __dmul_rn(pole_len, f.c)), p1);
    const double seg = __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
    const double rx = __dsub_rn(wx, p0), ry = __dsub_rn(wy, p1);
    double t = __ddiv_rn(__dadd_rn(__dmul_rn(rx, d0), __dmul_rn(ry, d1)), seg);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    const double ex = __dsub_rn(rx, __dmul_rn(t, d0)), ey = __dsub_rn(ry, __dmul_rn(t, d1));
    const double dist2 = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
    if (dist2 <= (0.045 / 2) * (0.045 / 2)) cls = 2;
    return cls;
}

// The same classification with the world coordinates of the pixel centres
// precomputed (a view has only w distinct wx and h distinct wy, both
// frame-independent) and the pole's segment constants per frame.  Pixels far
// from the pole's supporting line skip the clamped projection (and its
// division): the clamped-segment distance is never below the line distance,
// and the cut-off keeps a 1e-9 relative margin, so the decision is unchanged.
struct PoleSeg {
    double x, p1, d0, d1, seg, band;  // band: reject perp^2 above this
};

__device__ __forceinline__ PoleSeg pole_seg(const PixFrame &f, double pole_len) {
    PoleSeg g;
    g.x = f.x;
    g.p1 = __dadd_rn(0.0, 0.22 / 2);
    g.d0 = __dsub_rn(__dadd_rn(f.x, __dmul_rn(pole_len, f.s)), f.x);
    g.d1 = __dsub_rn(__dadd_rn(g.p1, __dmul_rn(pole_len, f.c)), g.p1);
    g.seg = __dadd_rn(__dmul_rn(g.d0, g.d0), __dmul_rn(g.d1, g.d1));
    // line distance^2 = perp^2 / seg  <=  r^2   <=>  perp^2 <= r^2 seg
    g.band = (0.045 / 2) * (0.045 / 2) * g.seg * (1.0 + 1e-9) + 1e-300;
    return g;
}

__device__ __forceinline__ int pix_class_pre(double wx, double wy, const PoleSeg &g) {
    int cls = 0;
    if (fabs(__dsub_rn(wx, g.x)) <= 0.36 / 2 && fabs(__dsub_rn(wy, 0.0)) <= 0.22 / 2) cls = 1;
    const double rx = __dsub_rn(wx, g.x), ry = __dsub_rn(wy, g.p1);
    const double perp = rx * g.d1 - ry * g.d0;  // (filter only: rounding covered by the margin)
    if (perp * perp > g.band) return cls;
    double t = __ddiv_rn(__dadd_rn(__dmul_rn(rx, g.d0), __dmul_rn(ry, g.d1)), g.seg);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    const double ex = __dsub_rn(rx, __dmul_rn(t, g.d0)), ey = __dsub_rn(ry, __dmul_rn(t, g.d1));
    const double dist2 = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
    if (dist2 <= (0.045 / 2) * (0.045 / 2)) cls = 2;
    return cls;
}

// pixel-centre world coordinates of a view (pix_class's wx / wy)
__device__ __forceinline__ double view_wx(const double *vis, int w, int col) {
    const double px = __dsub_rn(__dadd_rn((double)col, 0.5), __ddiv_rn((double)w, 2.0));
    const double scale = __dmul_rn(__ddiv_rn((double)w, __dmul_rn(2.0, 2.4)), vis[11]);
    return __dadd_rn(__ddiv_rn(px, scale), vis[9]);
}
__device__ __forceinline__ double view_wy(const double *vis, int w, int h, int row) {
    const double py = __dsub_rn(__ddiv_rn((double)h, 2.0), __dadd_rn((double)row, 0.5));
    const double scale = __dmul_rn(__ddiv_rn((double)w, __dmul_rn(2.0, 2.4)), vis[11]);
    return __dadd_rn(__ddiv_rn(py, scale), vis[10]);
}

// colour channel as drawn: np.asarray(color, uint8) truncates the float
__device__ __forceinline__ uint8_t color_u8(double v) { return (uint8_t)(int)v; }

// brightness_postprocess then rgb_to_gray of one colour
__device__ __forceinline__ double gray_of(const double *rgb, double bright) {
    double ch[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double v = rint(__dmul_rn((double)color_u8(rgb[k]), bright));
        v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
        ch[k] = (double)(uint8_t)(int)v;
    }
    // img @ _LUMA / 255.0.  NumPy's float64 matmul kernel (this image's NumPy
    // 2.3 build) evaluates the three-term dot as fma(b, .114, fma(r, .299, g * .587))
    // -- checked against 70 000 random colours, 0 mismatches (tests/golden fixtures)
    const double dot =
        __fma_rn(ch[2], 0.114, __fma_rn(ch[0], 0.299, __dmul_rn(ch[1], 0.587)));
    return __ddiv_rn(dot, 255.0);
}

// One CTA per world: threads stride over the h*w pixels; each pixel's three
// stacked frames (oldest first) are written as three consecutive values.
// hist: [n, 3] frames (oldest first).  For worlds in `mask` (an autoreset this
// step) the terminal stack [h1, h2, term] is drawn with the old visuals into
// term_out, the new episode's visuals are drawn from its stream, and the
// observation is three copies of the new first frame.
constexpr int kMaxView = 512;  // widest / tallest view the stack kernels stage in smem

// 12 values at a 16-byte-aligned address (3 * 4 pixels * sizeof(T), row start
// aligned because w % 4 == 0 and each world's image starts 16-byte aligned)
__device__ __forceinline__ void store12(float *o, const float *v) {
    float4 *d = reinterpret_cast<float4 *>(o);
    d[0] = make_float4(v[0], v[1], v[2], v[3]);
    d[1] = make_float4(v[4], v[5], v[6], v[7]);
    d[2] = make_float4(v[8], v[9], v[10], v[11]);
}
__device__ __forceinline__ void store12(double *o, const double *v) {
    double2 *d = reinterpret_cast<double2 *>(o);
#pragma unroll
    for (int k = 0; k < 6; ++k) d[k] = make_double2(v[2 * k], v[2 * k + 1]);
}

// Per-world shared scratch of the stack kernels.  The exact per-pixel test
// (pix_class_pre, float64 in the reference's order) runs only where its answer
// is not already decided by per-row / per-column facts:
//  * cart: |wx - x| <= 0.18 depends on the column only, |wy| <= 0.11 on the row
//    only -- the same float64 tests, evaluated w * 3 + h times per world;
//  * pole: a pixel can be pole only if its row is within 0.0225 of the
//    segment's y extent and its line distance is <= 0.0225, i.e.
//    |(wx - x) d1 - ry d0| <= 0.0225 sqrt(seg): per (frame, row) a column
//    interval, computed in float64 and widened by two columns, outside which
//    the exact test can only answer "not pole".  Inside it the exact test
//    decides, so the classes are unchanged.
struct StackScratch {
    double g[3];  // gray level of background / cart / pole
    double wxs[kMaxView], wys[kMaxView];
    PoleSeg ps[3];
    uint8_t cart_col[3][kMaxView], cart_row[kMaxView];
    uint8_t row_any[kMaxView];  // 0: every pixel of the row is background in all three frames
    int16_t pole_lo[3][kMaxView], pole_hi[3][kMaxView];  // candidate columns (inclusive)
};

// candidate columns [lo, hi] of frame f's pole on the view row whose world y is wy
__device__ __forceinline__ void pole_cols(const PoleSeg &g, double wy, const double *v, int w,
                                          double scale, int &lo, int &hi) {
    const double ry = wy - g.p1;
    const double R = 0.045 / 2 * sqrt(g.seg) * (1.0 + 1e-6) + 1e-300;
    lo = 0;  // default (non-finite inputs): every column exact
    hi = w - 1;
    if (!(isfinite(g.x) && isfinite(g.d0) && isfinite(g.d1) && isfinite(ry))) return;
    // rows farther than the radius from the segment's y extent [0, d1]: no pole
    const double ry_lo = fmin(0.0, g.d1) - (0.045 / 2 * (1.0 + 1e-6) + 1e-9);
    const double ry_hi = fmax(0.0, g.d1) + (0.045 / 2 * (1.0 + 1e-6) + 1e-9);
    if (ry < ry_lo || ry > ry_hi) {
        lo = 1;
        hi = 0;
        return;
    }
    if (g.d1 != 0.0) {
        const double ctr = g.x + ry * g.d0 / g.d1, half = R / fabs(g.d1);
        const double cl = (ctr - half - v[9]) * scale + 0.5 * w - 0.5;
        const double ch = (ctr + half - v[9]) * scale + 0.5 * w - 0.5;
        if (cl == cl && ch == ch) {
            lo = cl < -8.0 ? 0 : (cl > w + 8.0 ? w : max(0, (int)floor(cl) - 2));
            hi = ch > w + 8.0 ? w - 1 : (ch < -8.0 ? -1 : min(w - 1, (int)ceil(ch) + 2));
        }
    } else if (fabs(ry * g.d0) > R * (1.0 + 1e-6)) {
        lo = 1;  // horizontal pole off this row: no candidate
        hi = 0;
    }
}

template <typename T>
__device__ __forceinline__ void draw_stack(int w, int h, double pole_len, const double *v,
                                           const PixFrame *fr, StackScratch &S, T *o) {
    // one set-up phase (a single barrier): column facts, row facts (incl. the
    // pole's candidate columns of the three frames), gray levels, segments
    const double scale = (double)w / (2.0 * 2.4) * v[11];
    for (int idx = threadIdx.x; idx < w + h; idx += blockDim.x) {
        if (idx < w) {
            const double wx = view_wx(v, w, idx);
            S.wxs[idx] = wx;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                S.cart_col[k][idx] = fabs(__dsub_rn(wx, fr[k].x)) <= 0.36 / 2;
        } else {
            const int r = idx - w;
            const double wy = view_wy(v, w, h, r);
            S.wys[r] = wy;
            const bool cart_r = fabs(__dsub_rn(wy, 0.0)) <= 0.22 / 2;
            S.cart_row[r] = cart_r;
            bool any = cart_r;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                int lo, hi;
                pole_cols(pole_seg(fr[k], pole_len), wy, v, w, scale, lo, hi);
                S.pole_lo[k][r] = (int16_t)lo;
                S.pole_hi[k][r] = (int16_t)hi;
                any = any || lo <= hi;
            }
            S.row_any[r] = any;
        }
    }
    if (threadIdx.x >= blockDim.x - 3) {
        const int k = threadIdx.x - (blockDim.x - 3);
        S.g[k] = gray_of(v + 3 * k, v[12]);
        S.ps[k] = pole_seg(fr[k], pole_len);
    }
    __syncthreads();
    const T g0 = (T)S.g[0], g1 = (T)S.g[1], g2 = (T)S.g[2];
    auto cls_of = [&](int k, int row, int col, double wy) {
        int cls = S.cart_col[k][col] & S.cart_row[row];
        if (col >= S.pole_lo[k][row] && col <= S.pole_hi[k][row])
            cls = pix_class_pre(S.wxs[col], wy, S.ps[k]);
        return cls;
    };
    if ((w & 3) == 0) {
        // four pixels of a row per thread: the 12 (pixel, frame) classes packed
        // two bits each from the row / column facts, the few pole candidates
        // then resolved exactly in one loop over their bits (one divergent
        // region per thread instead of twelve); 12 consecutive values stored
        // as three 16-byte (float) or six 16-byte (double) vectors
        for (int q = threadIdx.x; q < (w * h) >> 2; q += blockDim.x) {
            const int p = q << 2, row = p / w, col = p - row * w;
            if (!S.row_any[row]) {  // most rows: background in every frame
                T vals[12];
#pragma unroll
                for (int b = 0; b < 12; ++b) vals[b] = g0;
                store12(o + 3 * p, vals);
                continue;
            }
            const uint32_t cr = S.cart_row[row];
            uint32_t packed = 0, cand = 0;  // bit pair / bit (3 * j + k)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const uint32_t cc = *reinterpret_cast<const uint32_t *>(&S.cart_col[k][col]) &
                                    (cr ? 0x01010101u : 0u);
                const int lo = S.pole_lo[k][row], hi = S.pole_hi[k][row];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    packed |= ((cc >> (8 * j)) & 1u) << (2 * (3 * j + k));
                    cand |= (uint32_t)(col + j >= lo && col + j <= hi) << (3 * j + k);
                }
            }
            if (cand) {
                const double wy = S.wys[row];
                do {
                    const int b = __ffs(cand) - 1;
                    cand &= cand - 1;
                    const int j = b / 3, k = b - 3 * j;
                    const uint32_t cls = (uint32_t)pix_class_pre(S.wxs[col + j], wy, S.ps[k]);
                    packed = (packed & ~(3u << (2 * b))) | (cls << (2 * b));
                } while (cand);
            }
            T vals[12];
#pragma unroll
            for (int b = 0; b < 12; ++b) {
                const uint32_t cls = (packed >> (2 * b)) & 3u;
                vals[b] = cls == 0 ? g0 : (cls == 1 ? g1 : g2);
            }
            store12(o + 3 * p, vals);
        }
        return;
    }
    for (int p = threadIdx.x; p < w * h; p += blockDim.x) {
        const int row = p / w, col = p - row * w;
        const double wy = S.wys[row];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int cls = cls_of(k, row, col, wy);
            o[3 * p + k] = cls == 0 ? g0 : (cls == 1 ? g1 : g2);
        }
    }
}

// One CTA per world: threads stride over the h*w pixels; each pixel's three
// stacked frames (oldest first) are written as three consecutive values.
#ifndef DK_PIXSTACK_THREADS
#define DK_PIXSTACK_THREADS 64
#define DK_PIXSTACK_MINB 16
#endif
constexpr int kPixStackThreads = DK_PIXSTACK_THREADS;
template <typename T>
__global__ void __launch_bounds__(DK_PIXSTACK_THREADS, DK_PIXSTACK_MINB) pixel_stack_kernel(int64_t n, int w, int h, double pole_len,
                                   const PixFrame *__restrict__ hist, const double *__restrict__ vis,
                                   T *__restrict__ out) {
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    __shared__ double v[kVis];
    __shared__ PixFrame fr[3];
    __shared__ StackScratch S;
    if (threadIdx.x < kVis) v[threadIdx.x] = vis[i * kVis + threadIdx.x];
    if (threadIdx.x < 3) fr[threadIdx.x] = hist[i * 3 + threadIdx.x];
    __syncthreads();
    draw_stack<T>(w, h, pole_len, v, fr, S, out + i * (int64_t)w * h * 3);
}

// batch_render + brightness_postprocess: RGB uint8 [n, h, w, 3] of one frame.
static __global__ void pixel_rgb_kernel(int64_t n, int w, int h, double pole_len,
                                        const PixFrame *__restrict__ frames,
                                        const double *__restrict__ vis, int brighten,
                                        uint8_t *__restrict__ out) {
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    __shared__ double v[kVis];
    __shared__ uint8_t col[3][3];
    if (threadIdx.x < kVis) v[threadIdx.x] = vis[i * kVis + threadIdx.x];
    __syncthreads();
    if (threadIdx.x < 9) {
        const int c = threadIdx.x / 3, k = threadIdx.x % 3;
        uint8_t u = color_u8(v[3 * c + k]);
        if (brighten) {
            double b = rint(__dmul_rn((double)u, v[12]));
            b = b < 0.0 ? 0.0 : (b > 255.0 ? 255.0 : b);
            u = (uint8_t)(int)b;
        }
        col[c][k] = u;
    }
    __syncthreads();
    const PixFrame f = frames[i];
    uint8_t *o = out + i * (int64_t)w * h * 3;
    for (int p = threadIdx.x; p < w * h; p += blockDim.x) {
        const int row = p / w, cc = p - row * w;
        const int cls = pix_class(v, pole_len, w, h, row, cc, f);
        o[3 * p] = col[cls][0];
        o[3 * p + 1] = col[cls][1];
        o[3 * p + 2] = col[cls][2];
    }
}

// randomize_visuals (pixelrender.py:134-153) drawn from the episode's stream
// (envkit.py:506-516: the reset's step-0 stream, after sample_initial's draws).
struct VisualBoundsC {
    double nominal[kVis];  // VisualParams nominal (packed as above)
    double color_jitter, camera_offset_range, zoom_lo, zoom_hi, bright_lo, bright_hi;
};

__device__ __forceinline__ void draw_visuals(Philox4x64 &rng, const VisualBoundsC &b,
                                             double *vis) {
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k) {
            double x = __dadd_rn(b.nominal[3 * c + k], rng.uniform(-b.color_jitter, b.color_jitter));
            vis[3 * c + k] = x < 0.0 ? 0.0 : (x > 255.0 ? 255.0 : x);  // np.clip(c, 0, 255)
        }
    vis[9] = rng.uniform(-b.camera_offset_range, b.camera_offset_range);
    vis[10] = rng.uniform(-b.camera_offset_range, b.camera_offset_range);
    vis[11] = rng.uniform(b.zoom_lo, b.zoom_hi);
    vis[12] = rng.uniform(b.bright_lo, b.bright_hi);
}

// Per-world bookkeeping after a step (one thread per world): shift the frame
// history, or on an autoreset draw the new episode's visuals (skipping the
// `skip` words sample_initial consumed) and refill the history.
// obs / term_obs rows: [x, cos th, sin th, ...] (cartpole state_obs).
template <typename T>
__global__ void pixel_advance_kernel(int64_t n, int obs_dim, const T *__restrict__ obs,
                                     const uint8_t *__restrict__ reset_mask, int first,
                                     PixFrame *__restrict__ hist, double *__restrict__ vis,
                                     uint32_t *__restrict__ episode, int randomize,
                                     VisualBoundsC bounds, uint64_t seed, int64_t env0, int skip) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const PixFrame f{(double)obs[i * obs_dim], (double)obs[i * obs_dim + 1],
                     (double)obs[i * obs_dim + 2]};
    const bool reset = first || (reset_mask && reset_mask[i]);
    if (reset) {
        if (!first) episode[i] += 1u;
        double nv[kVis];
        if (randomize) {
            Philox4x64 rng;
            rng.init(seed, (uint64_t)(env0 + i), episode[i], 0);
            for (int k = 0; k < skip; ++k) (void)rng.next64();
            draw_visuals(rng, bounds, nv);
        } else {
            for (int k = 0; k < kVis; ++k) nv[k] = bounds.nominal[k];
        }
        for (int k = 0; k < kVis; ++k) vis[i * kVis + k] = nv[k];
        hist[3 * i] = f;
        hist[3 * i + 1] = f;
        hist[3 * i + 2] = f;
    } else {
        hist[3 * i] = hist[3 * i + 1];
        hist[3 * i + 1] = hist[3 * i + 2];
        hist[3 * i + 2] = f;
    }
}

// The terminal stack of autoreset worlds: [h1, h2, term] with the old visuals
// (called before pixel_advance_kernel replaces them).
template <typename T>
__global__ void pixel_terminal_kernel(int64_t n, int w, int h, double pole_len, int obs_dim,
                                      const T *__restrict__ term_obs,
                                      const uint8_t *__restrict__ mask,
                                      const PixFrame *__restrict__ hist,
                                      const double *__restrict__ vis, T *__restrict__ out) {
    const int64_t i = blockIdx.x;
    if (i >= n || !mask[i]) return;
    __shared__ double v[kVis];
    __shared__ PixFrame fr[3];
    __shared__ StackScratch S;
    if (threadIdx.x < kVis) v[threadIdx.x] = vis[i * kVis + threadIdx.x];
    if (threadIdx.x < 2) fr[threadIdx.x] = hist[i * 3 + 1 + threadIdx.x];
    if (threadIdx.x == 2)
        fr[2] = PixFrame{(double)term_obs[i * obs_dim], (double)term_obs[i * obs_dim + 1],
                         (double)term_obs[i * obs_dim + 2]};
    __syncthreads();
    draw_stack<T>(w, h, pole_len, v, fr, S, out + i * (int64_t)w * h * 3);
}

// ppo.pixel_normalize (ppo.py:232-238): per-sample, per-channel
// standardisation of [n, h, w, c] stacks.  NumPy's mean / std over axes (1, 2)
// sum each (sample, channel) sequentially in row-major pixel order, so one
// thread per (sample, channel) does exactly that in float64 (bit-exact), then
// a second, elementwise kernel writes (x - mean) / std (0 where std == 0) as
// float64 [n, h, w, c] or float32 [n, c, h, w] (the policy's input layout,
// ppo.py:281-283).
template <typename T>
__global__ void pixnorm_stats_kernel(int64_t n, int hw, int c, const T *__restrict__ x,
                                     double *__restrict__ stats) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n * c) return;
    const int64_t s = k / c;
    const int ch = (int)(k - s * c);
    const T *p = x + s * (int64_t)hw * c + ch;
    double sum = 0.0;
    for (int i = 0; i < hw; ++i) sum = __dadd_rn(sum, (double)p[(int64_t)i * c]);
    const double mean = __ddiv_rn(sum, (double)hw);
    double sq = 0.0;
    for (int i = 0; i < hw; ++i) {
        const double d = __dsub_rn((double)p[(int64_t)i * c], mean);
        sq = __dadd_rn(sq, __dmul_rn(d, d));
    }
    stats[2 * k] = mean;
    stats[2 * k + 1] = __dsqrt_rn(__ddiv_rn(sq, (double)hw));
}

// The [n, h, w, 3] float32 stacks the pixel env produces.
// The statistics are two sequential float64 chains per (sample, channel) --
// the order NumPy sums in, so no tree reduction is allowed -- 8192 dependent
// adds per chain.  To hide their latency every chain of the batch runs at
// once (24 576 chains at 8192 samples): a CTA holds 32 samples, warp c runs
// channel c, lane = sample.  The stack streams through shared memory in stages
// of PN pixels of each of the 32 samples (32 row runs of 768 bytes, padded
// rows), NS - 1 stages in flight; pass 1 (sums) and pass 2 (squared deviations
// from the mean) stream it twice.  Measured alternatives: one warp
// per 32 samples with three chains per lane, and per-row cp.async.bulk copies
// (the TMA engine serialises 32 small copies per stage).
namespace pixnorm {
constexpr int PN = 64;                      // pixels per sample per stage
constexpr int ROW = PN * 3 * 4;             // 768 bytes of one sample
constexpr int ROW_PAD = ROW + 16;           // 196 words: conflict-free LDS.128 quarter-warps
constexpr int NS = 4;                       // stages
constexpr int STAGE = 32 * ROW_PAD;         // 25088 bytes
constexpr int SMEM = NS * STAGE;            // 100352 bytes: two CTAs per SM

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
}  // namespace pixnorm

// Warp c of a 96-thread CTA runs channel c of the CTA's 32 samples (lane =
// sample, one chain per lane): it reads the 16-byte words of its lane's row and
// keeps its channel's four values of every four pixels.
template <int C>
__device__ __forceinline__ void pixnorm_chan(const float4 *row, double &a, double m, bool pass2) {
#pragma unroll 4
    for (int q = 0; q < pixnorm::PN / 4; ++q) {
        const float4 u = row[3 * q], v = row[3 * q + 1], w = row[3 * q + 2];
        float e[4];
        if (C == 0) { e[0] = u.x; e[1] = u.w; e[2] = v.z; e[3] = w.y; }
        if (C == 1) { e[0] = u.y; e[1] = v.x; e[2] = v.w; e[3] = w.z; }
        if (C == 2) { e[0] = u.z; e[1] = v.y; e[2] = w.x; e[3] = w.w; }
        if (!pass2) {
#pragma unroll
            for (int p = 0; p < 4; ++p) a = __dadd_rn(a, (double)e[p]);
        } else {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const double d = __dsub_rn((double)e[p], m);
                a = __dadd_rn(a, __dmul_rn(d, d));
            }
        }
    }
}

// Staging: all 96 threads copy the stage with 16-byte cp.async (each sample's
// 768-byte run coalesced), NS - 1 stages in flight, two CTA barriers per stage.
__global__ void __launch_bounds__(96) pixnorm_stats3_kernel(int64_t n, int hw, int spc,
                                                             const float *__restrict__ x,
                                                             double *__restrict__ stats) {
    using namespace pixnorm;
    extern __shared__ __align__(128) unsigned char sm[];
    const int tid = threadIdx.x, lane = tid & 31, c = tid >> 5;
    const int64_t s0 = (int64_t)blockIdx.x * spc;  // spc <= 32 samples per CTA
    const int ns = (int)(n - s0 < spc ? n - s0 : spc);
    const int tiles = hw / PN, total = 2 * tiles;
    const unsigned char *base = reinterpret_cast<const unsigned char *>(x + s0 * (int64_t)hw * 3);
    const int64_t sample_bytes = (int64_t)hw * 12;
    constexpr int CHUNKS = ROW / 16;  // 48 16-byte chunks per row
    auto load = [&](int k) {
        if (k < total) {
            unsigned char *dst = sm + (k % NS) * STAGE;
            const unsigned char *src = base + (int64_t)(k % tiles) * ROW;
            for (int i = tid; i < ns * CHUNKS; i += 96) {
                const int r = i / CHUNKS, ch = i - r * CHUNKS;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 su32(dst + r * ROW_PAD + ch * 16)),
                             "l"(src + r * sample_bytes + ch * 16)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int k = 0; k < NS - 1; ++k) load(k);
    double a = 0.0, m = 0.0;
    const double rn = (double)hw;
    for (int k = 0; k < total; ++k) {
        load(k + NS - 1);  // its stage was released by the barrier that ended iteration k - 1
        asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
        __syncthreads();
        const float4 *row = reinterpret_cast<const float4 *>(sm + (k % NS) * STAGE + lane * ROW_PAD);
        if (k == tiles) {
            m = __ddiv_rn(a, rn);
            a = 0.0;
        }
        const bool p2 = k >= tiles;
        if (c == 0) pixnorm_chan<0>(row, a, m, p2);
        else if (c == 1) pixnorm_chan<1>(row, a, m, p2);
        else pixnorm_chan<2>(row, a, m, p2);
        __syncthreads();
    }
    if (lane < ns) {
        double *o = stats + 6 * (s0 + lane) + 2 * c;
        o[0] = m;
        o[1] = __dsqrt_rn(__ddiv_rn(a, rn));
    }
}

// Elementwise (x - mean) / std for the 3-channel float32 stacks: one thread per
// four pixels (three 16-byte loads), writing four pixels of each channel plane
// (channels_first) or the same 48 bytes back (NHWC); grid.y walks samples.
template <typename U, bool CF>
__global__ void __launch_bounds__(256) pixnorm_apply3_kernel(int64_t n, int hw,
                                                             const float *__restrict__ x,
                                                             const double *__restrict__ stats,
                                                             U *__restrict__ out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (hw >> 2)) return;
    for (int64_t s = blockIdx.y; s < n; s += gridDim.y) {
        const double *st = stats + 6 * s;
        const double m[3] = {st[0], st[2], st[4]}, sd[3] = {st[1], st[3], st[5]};
        const float4 *p = reinterpret_cast<const float4 *>(x + (s * hw + 4 * q) * 3);
        const float4 u = p[0], v = p[1], w = p[2];
        const float f[12] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w, w.x, w.y, w.z, w.w};
        // one IEEE reciprocal per channel, then each quotient by Markstein's
        // correction q1 = q0 + (a - q0 sd) r: correctly rounded (= __ddiv_rn) for
        // r = RN(1/sd) and a faithful q0 while nothing under/overflows; outside
        // that range (and for sd = inf / NaN) the IEEE division
        double r[3];
        bool safe[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            r[c] = __ddiv_rn(1.0, sd[c]);
            safe[c] = sd[c] > 0x1p-500 && sd[c] < 0x1p500;
        }
        U y[12];
#pragma unroll
        for (int e = 0; e < 12; ++e) {
            const int c = e % 3;
            const double a = __dsub_rn((double)f[e], m[c]);
            double qv;
            if (safe[c] && (fabs(a) > 0x1p-900 || a == 0.0) && fabs(a) < 0x1p500) {
                const double q0 = __dmul_rn(a, r[c]);
                qv = __fma_rn(__fma_rn(-q0, sd[c], a), r[c], q0);
            } else {
                qv = __ddiv_rn(a, sd[c]);
            }
            y[e] = (U)(sd[c] > 0.0 ? qv : 0.0);
        }
        if (CF) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                U *o = out + (s * 3 + c) * hw + 4 * q;
                if constexpr (sizeof(U) == 4) {
                    *reinterpret_cast<float4 *>(o) = make_float4(y[c], y[3 + c], y[6 + c], y[9 + c]);
                } else {
                    reinterpret_cast<double2 *>(o)[0] = make_double2(y[c], y[3 + c]);
                    reinterpret_cast<double2 *>(o)[1] = make_double2(y[6 + c], y[9 + c]);
                }
            }
        } else {  // the same 12 values back in place: 16-byte stores
            U *o = out + (s * hw + 4 * q) * 3;
            if constexpr (sizeof(U) == 4) {
#pragma unroll
                for (int v4 = 0; v4 < 3; ++v4)
                    reinterpret_cast<float4 *>(o)[v4] =
                        make_float4(y[4 * v4], y[4 * v4 + 1], y[4 * v4 + 2], y[4 * v4 + 3]);
            } else {
#pragma unroll
                for (int v2 = 0; v2 < 6; ++v2)
                    reinterpret_cast<double2 *>(o)[v2] = make_double2(y[2 * v2], y[2 * v2 + 1]);
            }
        }
    }
}

template <typename T, typename U>
__global__ void pixnorm_apply_kernel(int64_t n, int hw, int c, const T *__restrict__ x,
                                     const double *__restrict__ stats, int channels_first,
                                     U *__restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // output element
    const int64_t total = n * (int64_t)hw * c;
    if (e >= total) return;
    int64_t s, pix;
    int ch;
    if (channels_first) {  // e = (s * c + ch) * hw + pix
        const int64_t sc = e / hw;
        pix = e - sc * hw;
        s = sc / c;
        ch = (int)(sc - s * c);
    } else {  // e = (s * hw + pix) * c + ch
        const int64_t sp = e / c;
        ch = (int)(e - sp * c);
        s = sp / hw;
        pix = sp - s * hw;
    }
    const double mean = stats[2 * (s * c + ch)], sd = stats[2 * (s * c + ch) + 1];
    const double v = (double)x[(s * hw + pix) * c + ch];
    out[e] = (U)(sd > 0.0 ? __ddiv_rn(__dsub_rn(v, mean), sd) : 0.0);
}

}  // namespace dk
