// kernels.cuh -- sm_100a device code of the MBP decoder.
//
// Layout ("frame-interleaved", lane = frame): frames are processed in groups
// of 32; group g's per-edge message for edge e lives in one 128-byte line
// c2v[(g*E + e)*32 + lane] (256 B in fp64 mode), its posterior for variable i
// in post[(g*n + i)*32 + lane].  A warp therefore updates one check (or one
// variable) for 32 frames at once: the graph indices it reads are
// warp-uniform, every message access is one fully used, coalesced line, and
// rows of different degree never diverge a warp.  Bits (noisy key, hard
// decision, syndrome) are 32-frame words: word[g*n + i] bit f = frame 32g+f.
//
// This header holds the device primitives (cache-control loads, the grid
// barrier, the check-node rule, bit transposes, the Alice-side syndrome and
// the single-phase kernels); the persistent decode kernel is in decode.cuh.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mbp {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxU = 16;

// ---------------------------------------------------------------------------
// cache-control loads.  Messages and bit words are rewritten by other SMs
// between phases of the same launch, so they are read L2-coherent (.cg,
// never from a possibly stale L1 line); graph indices are immutable (.nc).
// ---------------------------------------------------------------------------
template <class T> __device__ __forceinline__ T ld_cg(const T* p) { return __ldcg(p); }
template <class T> __device__ __forceinline__ T ld_ro(const T* p) { return __ldg(p); }

// relaxed (no L1 invalidation per poll, unlike ld.acquire which emits CCTL.IVALL)
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// predicated loads/stores without branches (uniform or per-lane predicate).
// ld_cg_pred leaves the destination undefined when the predicate is off
// (callers mask those values); ld_cg_if zero-fills.
__device__ __forceinline__ float ld_cg_pred(const float* p, bool pred)
{
    float v;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cg.f32 %0, [%1];\n\t}"
                 : "=f"(v) : "l"(p), "r"((int)pred));
    return v;
}
__device__ __forceinline__ double ld_cg_pred(const double* p, bool pred)
{
    double v;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cg.f64 %0, [%1];\n\t}"
                 : "=d"(v) : "l"(p), "r"((int)pred));
    return v;
}
__device__ __forceinline__ float ld_cg_if(const float* p, bool pred)
{
    float v = 0.0f;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cg.f32 %0, [%1];\n\t}"
                 : "+f"(v) : "l"(p), "r"((int)pred));
    return v;
}
__device__ __forceinline__ double ld_cg_if(const double* p, bool pred)
{
    double v = 0.0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cg.f64 %0, [%1];\n\t}"
                 : "+d"(v) : "l"(p), "r"((int)pred));
    return v;
}
__device__ __forceinline__ void st_if(float* p, float v, bool pred)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f32 [%0], %1;\n\t}"
                 :: "l"(p), "f"(v), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void st_if(double* p, double v, bool pred)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}"
                 :: "l"(p), "d"(v), "r"((int)pred) : "memory");
}

// Grid-wide barrier for a cooperatively launched (co-resident) grid.
// bar[0] = arrival count, bar[1] = generation.
__device__ __forceinline__ void grid_barrier(unsigned* bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_relaxed(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (ld_relaxed(bar + 1) == gen) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Eq. 6 in fp32, complement-product form.  The reference rule
//   c2v_a = (-1)^z_j * 2 atanh( prod_{b != a} tanh(x_b / 2) )      (clamped)
// is evaluated with |tanh(x/2)| = 1 - c, c = 2u/(1+u), u = e^-|x|, and the
// magnitude of the product carried as its complement Q = 1 - prod t_b,
// combined by the exact identity 1 - (1-Q)(1-c) = Q + c(1 - Q).  Q keeps
// full relative precision where the plain fp32 product of tanh values
// rounds to 1 (|x| >~ 17, the failure of naive fp32 tanh);
// the output is 2 atanh(1 - Q) = ln((2 - Q) / Q).  Exclusive products come
// from prefix and suffix complements (no division), padding slots have c = 0
// (t = 1, neutral), and |x| >= sat also gives c = 0: that is where the
// reference's float64 tanh(x/2) rounds to exactly 1.0, and all-others-
// saturated then yields Q = 0 -> +-clamp as in its `prod >= 1.0` branch
// (_kernels.py:249-252).  4 MUFU + ~15 FMA-pipe ops per edge; max error
// |d| <= 4e-7 * max(|ref|, 1) against the exact rule (tools/ notes,
// DESIGN.md §3).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2_approx(float x)
{
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int D>
__device__ __forceinline__ void c2v_rule(const float (&x)[D], int d, unsigned flip, float clamp,
                                         float sat, float (&out)[D])
{
    // x[k] for k >= d may be garbage (predicated-off loads): masked here
    float c[D];
    unsigned sb[D];
    unsigned tot = flip << 31;  // syndrome sign (-1)^z_j folded into the parity
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const bool in = k < d;
        const float a = fabsf(x[k]);
        const float u = ex2_approx(-1.44269504088896341f * a);
        const float ck = 2.0f * u * rcp_approx(1.0f + u);
        c[k] = (in && a < sat) ? ck : 0.0f;
        sb[k] = in ? (__float_as_uint(x[k]) & 0x80000000u) : 0u;
        tot ^= sb[k];
    }
    float qs[D];
    float q = 0.0f;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
        qs[k] = q;
        q = fmaf(c[k], 1.0f - q, q);
    }
    float qp = 0.0f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float r = 1.0f - qp;
        const float qx = fmaf(qs[k], r, qp);
        qp = fmaf(c[k], r, qp);
        const float mag = fminf((lg2_approx(2.0f - qx) - lg2_approx(qx)) * 0.69314718055994531f, clamp);
        out[k] = __uint_as_float(__float_as_uint(mag) | (tot ^ sb[k]));
    }
}

// Eq. 6 literally (fp64 parity mode): t_b = tanh(x_b/2), product over the
// other edges in ascending order with no division (prefix, then the rest in
// order -- the exact multiplication sequence of c2v_pass), saturation,
// 2*atanh, syndrome sign, clamp.
template <int D>
__device__ __forceinline__ void c2v_rule(const double (&x)[D], int d, unsigned flip, double clamp,
                                         float /*sat*/, double (&out)[D])
{
    double t[D];
#pragma unroll
    for (int k = 0; k < D; ++k) t[k] = k < d ? tanh(0.5 * x[k]) : 1.0;
    double pre = 1.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        if (a < d) {
            double prod = pre;
#pragma unroll 4
            for (int b = a + 1; b < D; ++b)
                if (b < d) prod *= t[b];
            pre *= t[a];
            double r = prod >= 1.0 ? clamp : (prod <= -1.0 ? -clamp : 2.0 * atanh(prod));
            if (flip) r = -r;
            out[a] = r > clamp ? clamp : (r < -clamp ? -clamp : r);
        }
    }
}

template <class Real> __device__ __forceinline__ Real clampr(Real v, Real c)
{
    return v > c ? c : (v < -c ? -c : v);
}
template <> __device__ __forceinline__ float clampr<float>(float v, float c)
{
    return fminf(fmaxf(v, -c), c);
}

#ifndef MBP_DECODE_THREADS
#define MBP_DECODE_THREADS 256
#endif
constexpr int kDecodeThreads = MBP_DECODE_THREADS;  // decode kernel block size (decode.cuh, scatter.cuh)

// ---------------------------------------------------------------------------
// bit-matrix transposes between BitBlock rows and 32-frame words
// ---------------------------------------------------------------------------
// 32x32 bit transpose across a warp: in lane l holds row l; out lane l holds
// column l (bit f of out = bit l of lane f's input).  Recursive block swap:
// at stage j the lanes l and l^j exchange the j x j blocks off the diagonal
// (5 shuffles instead of 32 ballots).
__device__ __forceinline__ unsigned warp_transpose32(unsigned x, int lane)
{
    constexpr unsigned kM[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int j = 16 >> q;
        const unsigned m = kM[q];
        const unsigned y = __shfl_xor_sync(kFull, x, j);
        x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
    }
    return x;
}

// Tiled transposes between BitBlock rows and 32-frame words.  A block owns
// one tile: 32 rows (frames 32g..32g+31) x 128 bytes (1024 bits) of segment
// s.  Rows are staged in shared memory with coalesced byte accesses (row
// stride 132 B: the per-lane column reads below are bank-conflict free); each
// warp converts 4 of the tile's 32 bit-chunks with ballot transposes and
// writes whole 128-byte lines of words.
constexpr int kTileBytes = 128;
constexpr int kTileStride = kTileBytes + 4;

// rows [B][row_bytes]: segment s = bytes [s*seg_bytes, +seg_bytes) holding
// seg_bits bits -> words[g][s*seg_bits + bit] (and words2 if given)
static __global__ void __launch_bounds__(256) rows_to_words_kernel(
    const uint8_t* __restrict__ rows, long long row_bytes, int B, int G, int nseg, int seg_bits,
    long long seg_bytes, unsigned* __restrict__ words, unsigned* __restrict__ words2, long long words_per_group)
{
    __shared__ __align__(16) uint8_t tile[32 * kTileStride];
    const int tiles = (int)((seg_bytes + kTileBytes - 1) / kTileBytes);
    const long long total = (long long)G * nseg * tiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // 16-byte row accesses when every row segment is 16-byte aligned
    const bool vec = row_bytes % 16 == 0 && seg_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(rows) & 15) == 0;
    for (long long it = blockIdx.x; it < total; it += gridDim.x) {
        const int xt = (int)(it % tiles);
        const int s = (int)((it / tiles) % nseg);
        const int g = (int)(it / ((long long)tiles * nseg));
        const long long b0 = (long long)xt * kTileBytes;
        if (vec) {
            // one 16-byte load per thread: row r = tid / 8, bytes 16 (tid % 8)
            const int r = threadIdx.x >> 3, b = (threadIdx.x & 7) * 16;
            const int f = g * 32 + r;
            uint4 x = make_uint4(0u, 0u, 0u, 0u);
            if (f < B && b0 + b < seg_bytes)
                x = __ldg(reinterpret_cast<const uint4*>(rows + (long long)f * row_bytes + (long long)s * seg_bytes + b0 + b));
            unsigned* t = reinterpret_cast<unsigned*>(tile + r * kTileStride + b);
            t[0] = x.x;
            t[1] = x.y;
            t[2] = x.z;
            t[3] = x.w;
        } else {
            uint8_t v[32 * kTileBytes / 256];   // all loads in flight before the stores
#pragma unroll
            for (int q = 0; q < 32 * kTileBytes / 256; ++q) {
                const int idx = threadIdx.x + 256 * q;
                const int r = idx / kTileBytes, b = idx % kTileBytes;
                const int f = g * 32 + r;
                v[q] = (f < B && b0 + b < seg_bytes) ? rows[(long long)f * row_bytes + (long long)s * seg_bytes + b0 + b] : 0;
            }
#pragma unroll
            for (int q = 0; q < 32 * kTileBytes / 256; ++q) {
                const int idx = threadIdx.x + 256 * q;
                tile[(idx / kTileBytes) * kTileStride + idx % kTileBytes] = v[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = warp + 8 * q;   // 32-bit chunk of the tile
            const unsigned x = *reinterpret_cast<const unsigned*>(tile + lane * kTileStride + 4 * c);
            const unsigned w = warp_transpose32(x, lane);
            const long long bit = b0 * 8 + 32LL * c + lane;
            if (bit < seg_bits) {
                const long long o = (long long)g * words_per_group + (long long)s * seg_bits + bit;
                words[o] = w;
                if (words2) words2[o] = w;
            }
        }
        __syncthreads();
    }
}

// words[g][s*seg_bits + bit] -> rows (inverse of rows_to_words_kernel); row
// padding bits come out zero because words past seg_bits read as 0
static __global__ void __launch_bounds__(256) words_to_rows_kernel(
    const unsigned* __restrict__ words, long long words_per_group, int B, int G, int nseg, int seg_bits,
    long long seg_bytes, uint8_t* __restrict__ rows, long long row_bytes)
{
    __shared__ __align__(16) uint8_t tile[32 * kTileStride];
    const int tiles = (int)((seg_bytes + kTileBytes - 1) / kTileBytes);
    const long long total = (long long)G * nseg * tiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // 16-byte row accesses when every row segment is 16-byte aligned
    const bool vec = row_bytes % 16 == 0 && seg_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(rows) & 15) == 0;
    for (long long it = blockIdx.x; it < total; it += gridDim.x) {
        const int xt = (int)(it % tiles);
        const int s = (int)((it / tiles) % nseg);
        const int g = (int)(it / ((long long)tiles * nseg));
        const long long b0 = (long long)xt * kTileBytes;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = warp + 8 * q;
            const long long bit = b0 * 8 + 32LL * c + lane;
            const unsigned w = bit < seg_bits ? words[(long long)g * words_per_group + (long long)s * seg_bits + bit] : 0u;
            *reinterpret_cast<unsigned*>(tile + lane * kTileStride + 4 * c) = warp_transpose32(w, lane);
        }
        __syncthreads();
        if (vec) {
            const int r = threadIdx.x >> 3, b = (threadIdx.x & 7) * 16;
            const int f = g * 32 + r;
            if (f < B && b0 + b < seg_bytes) {
                const unsigned* t = reinterpret_cast<const unsigned*>(tile + r * kTileStride + b);
                *reinterpret_cast<uint4*>(rows + (long long)f * row_bytes + (long long)s * seg_bytes + b0 + b) =
                    make_uint4(t[0], t[1], t[2], t[3]);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 32 * kTileBytes / 256; ++q) {
                const int idx = threadIdx.x + 256 * q;
                const int r = idx / kTileBytes, b = idx % kTileBytes;
                const int f = g * 32 + r;
                if (f < B && b0 + b < seg_bytes)
                    rows[(long long)f * row_bytes + (long long)s * seg_bytes + b0 + b] = tile[r * kTileStride + b];
            }
        }
        __syncthreads();
    }
}

// Alice side, Eq. 1: syndrome words of 32 frames per check, z = XOR of key
// words over the row (syndrome_pass, _kernels.py:220-227, 32 frames wide).
static __global__ void syndrome_words_kernel(const uint8_t* __restrict__ deg, const int* __restrict__ chk_ell, int D,
                                      int n, int C, int G, const unsigned* __restrict__ key_w,
                                      unsigned* __restrict__ syn_w)
{
    const long long total = (long long)G * C;
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < total; it += nth) {
        const int g = (int)(it / C), j = (int)(it % C);
        const unsigned* kw = key_w + (long long)g * n;
        const int* row = chk_ell + (long long)j * D;
        unsigned p = 0;
        const int d = __ldg(deg + j);
        for (int k0 = 0; k0 < d; k0 += 8) {   // 8 row loads, then 8 word loads, in flight
            int id[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) id[k] = k0 + k < d ? __ldg(row + k0 + k) : -1;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (id[k] >= 0) p ^= __ldg(kw + id[k]);
        }
        syn_w[it] = p;
    }
}

// prior magnitude ln((1-e)/e) per frame (init_priors, decoder.py:147-152),
// computed in double and stored in the message type; padding frames get 0.
template <class Real>
__global__ void prior_kernel(const double* __restrict__ e, int e_stride, int B, int F, Real* __restrict__ L)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < F) {
        double v = 0.0;
        if (f < B) {
            const double ef = e[(long long)f * e_stride];
            v = log((1.0 - ef) / ef);
        }
        L[f] = (Real)v;
    }
}

// ---------------------------------------------------------------------------
// single-frame phases on explicit messages (c2v_update / v2c_update /
// soft_decision, decoder.py:155-200) -- thread per check / variable.
// ---------------------------------------------------------------------------
template <class Real, int D>
__global__ void c2v_phase_kernel(const int* __restrict__ chk_ptr, int lo, int hi,
                                 const uint8_t* __restrict__ syn_bits, Real clamp, float sat,
                                 const Real* __restrict__ v2c, Real* __restrict__ c2v)
{
    const int j = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= hi) return;
    const int e0 = chk_ptr[j], d = chk_ptr[j + 1] - e0;
    Real x[D], out[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = k < d ? v2c[e0 + k] : Real(0);
    c2v_rule<D>(x, d, syn_bits[j - lo] ? 1u : 0u, clamp, sat, out);
#pragma unroll
    for (int k = 0; k < D; ++k)
        if (k < d) c2v[e0 + k] = out[k];
}

template <class Real>
__global__ void v2c_phase_kernel(const int* __restrict__ var_ptr, const int* __restrict__ var_edge,
                                 int n, int lo_edge, int hi_edge, int joint, Real damping, Real clamp,
                                 const Real* __restrict__ c2v, const Real* __restrict__ priors,
                                 Real* __restrict__ v2c)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Real total = priors[i];
    for (int t = var_ptr[i]; t < var_ptr[i + 1]; ++t) {
        const int e = var_edge[t];
        if (joint || (e >= lo_edge && e < hi_edge)) total += c2v[e];
    }
    for (int t = var_ptr[i]; t < var_ptr[i + 1]; ++t) {
        const int e = var_edge[t];
        if (e < lo_edge || e >= hi_edge) continue;
        Real val = total - c2v[e];
        if (damping != Real(0)) val = (Real(1) - damping) * val + damping * v2c[e];
        v2c[e] = clampr(val, clamp);
    }
}

template <class Real>
__global__ void posterior_phase_kernel(const int* __restrict__ var_ptr, const int* __restrict__ var_edge,
                                       int n, const Real* __restrict__ c2v,
                                       const Real* __restrict__ priors, Real* __restrict__ post)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Real total = priors[i];
    for (int t = var_ptr[i]; t < var_ptr[i + 1]; ++t) total += c2v[var_edge[t]];
    post[i] = total;
}

// state readback: one frame's lane of an interleaved [..][32] array -> double,
// optionally through an index map (reference edge id -> internal slot)
template <class Real>
__global__ void gather_lane_kernel(const Real* __restrict__ src, long long count, int lane,
                                   const int* __restrict__ map, double* __restrict__ dst)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < count) dst[k] = (double)src[(map ? (long long)map[k] : k) * 32 + lane];
}

}  // namespace mbp
