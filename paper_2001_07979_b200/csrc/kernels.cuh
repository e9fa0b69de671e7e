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
// One persistent cooperative kernel runs the whole flooding decode
// (decode_loop, _kernels.py:323-379): per sweep a check phase (Eq. 6,
// c2v_pass _kernels.py:230-261, with the variable-to-check message formed on
// the fly in APP form v2c = clamp(post - c2v), exact because the reference's
// joint `total` IS the posterior sum, _kernels.py:276-279 vs 296-300), a
// variable phase (posterior Eq. 2 + hard decision, _kernels.py:293-307), and
// a syndrome phase (mismatch_count, _kernels.py:310-320) whose per-frame
// counts drive early termination; phases are separated by a grid barrier.
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

// ---------------------------------------------------------------------------
// decode kernel arguments
//
// Internal edge numbering (padded ELL): edge k of stacked check j is slot
// j*D + k, D = the kernel's degree bound.  A check's var ids chk_ell[j*D..]
// and its message lines are contiguous and need no chk_ptr lookup (one
// dependent load less per item); slot order is monotone in the reference's
// edge order, so ascending var_edge lists and matrix boundaries
// (edge_off[l] = l*m*D) keep the reference's summation order.
// ---------------------------------------------------------------------------
template <class Real>
struct DecodeArgs {
    // graph
    int n, m, u, C;
    int Ds;                            // ELL row stride (= max check degree)
    long long slots;                   // C * Ds
    const uint8_t* __restrict__ deg;   // [C] row degree
    const int* __restrict__ chk_ell;   // [C*Ds] var ids (pad 0)
    const int* __restrict__ var_ptr;   // [n+1] into var_edge (CSR; unused when dv > 0)
    const int* __restrict__ var_edge;  // [E] slot ids, ascending per variable
    int dv;                            // regular column degree, 0 if irregular
    long long edge_off[kMaxU + 1];     // slot offsets of the matrices
    // batch
    int G;                       // groups of 32 frames
    // state
    Real* __restrict__ c2v;      // [G][slots][32]
    Real* __restrict__ post;     // [G][P][n][32], P = ISO ? u+1 : 1
    Real* __restrict__ v2c;      // [G][slots][32] (damping only)
    const Real* __restrict__ Lmag;         // [G*32] prior magnitude per frame
    const unsigned* __restrict__ noisy_w;  // [G][n]
    const unsigned* __restrict__ syn_w;    // [G][C]
    unsigned* __restrict__ hard_w;         // [G][n]
    unsigned* __restrict__ hist_w;         // [(T+1)][G][n] or null
    int* __restrict__ cnt;       // [2][G*32] mismatch counts by sweep parity
    int* __restrict__ any_bad;   // [2]
    int* __restrict__ iters;     // [G*32] first converged sweep, -1 unset
    unsigned* __restrict__ barrier;  // [2]
    unsigned* __restrict__ work;     // [3*(T+1)+1] dynamic work counters, zeroed per launch
    int* __restrict__ sweeps_run;    // [1]
    unsigned long long* __restrict__ ts;  // phase timestamps (globaltimer ns) or null
    int ts_cap;
    // outputs (per frame, batch B)
    int B;
    uint8_t* __restrict__ out_conv;
    int* __restrict__ out_iters;
    int* __restrict__ out_mism;
    // config
    int max_it;
    Real clamp;
    Real damping;
    float sat;
};

// Check phase item: check j of group g at sweep t; `act` = lanes (frames)
// still decoding.  Reads post_{t-1}, c2v_{t-1}, writes c2v_t.  The row's
// variable ids, degree and syndrome word come from the warp's shared-memory
// stage of its work chunk (one coalesced load per chunk, not per item), so
// an item costs one memory round trip.  Branch-free over the D slots
// (D = the launch's degree bound): slots k >= d are predicated off.
template <class Real, int D, bool DAMP, bool ISO>
__device__ __forceinline__ void check_item(const DecodeArgs<Real>& A, int g, int j, int t,
                                           unsigned act, int lane, const int* srow, int d,
                                           unsigned synword, Real L)
{
    const bool live = (act >> lane) & 1u;
    const unsigned flip = (synword >> lane) & 1u;
    const int mat = ISO ? j / A.m : 0;
    Real* c2v_row = A.c2v + ((size_t)g * A.slots + (size_t)j * A.Ds) * 32 + lane;
    Real* v2c_row = DAMP ? A.v2c + ((size_t)g * A.slots + (size_t)j * A.Ds) * 32 + lane : nullptr;
    const Real* postg = A.post + ((size_t)g * (ISO ? A.u + 1 : 1) + mat) * A.n * 32 + lane;

    Real x[D];
    if (t == 1) {
        // sweep 1 reads the UNCLAMPED prior (decode_loop init, _kernels.py:353-355)
        const unsigned* nw = A.noisy_w + (size_t)g * A.n;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const unsigned w = k < d ? ld_ro(nw + srow[k]) : 0u;
            x[k] = k < d ? (((w >> lane) & 1u) ? -L : L) : Real(0);
        }
        if (DAMP) {
#pragma unroll
            for (int k = 0; k < D; ++k) st_if(v2c_row + k * 32, x[k], live && k < d);
        }
    } else {
        Real p[D], q[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const bool pk = live && k < d;
            p[k] = ld_cg_if(postg + (unsigned)srow[k] * 32u, pk);
            q[k] = ld_cg_if(c2v_row + k * 32, pk);
        }
        if (DAMP) {
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const Real old = ld_cg_if(v2c_row + k * 32, live && k < d);
                x[k] = clampr((Real(1) - A.damping) * (p[k] - q[k]) + A.damping * old, A.clamp);
                st_if(v2c_row + k * 32, x[k], live && k < d);
            }
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) x[k] = clampr(p[k] - q[k], A.clamp);
        }
    }
    Real out[D];
    c2v_rule<D>(x, d, flip, A.clamp, A.sat, out);
#pragma unroll
    for (int k = 0; k < D; ++k) st_if(c2v_row + k * 32, out[k], live && k < d);
}

// Variable phase, regular column degree DV, NV variables per warp pass
// (independent load streams in flight): joint posterior prior + sum of every
// matrix's c2v in ascending edge order (posterior_pass, _kernels.py:293-301),
// hard decision post < 0 (ties -> 0) as a ballot (hard_pass).  Edge slots,
// noisy words and previous hard words come from the chunk's shared stage.
template <class Real, int DV, int NV>
__device__ __forceinline__ void var_items_regular(const DecodeArgs<Real>& A, int g, int i0, int nv, int t,
                                                  unsigned act, int lane, const int* sedge, int sstride,
                                                  const unsigned* snoisy, const unsigned* sold, Real L)
{
    const bool live = (act >> lane) & 1u;
    const Real* c2vg = A.c2v + (size_t)g * A.slots * 32 + lane;
    Real c[NV][DV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int k = 0; k < DV; ++k) {
            const int e = v < nv ? sedge[v * sstride + k] : 0;
            c[v][k] = ld_cg_if(c2vg + (unsigned)e * 32u, live && v < nv);
        }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        if (v >= nv) break;
        const int i = i0 + v;
        Real acc = ((snoisy[v] >> lane) & 1u) ? -L : L;
#pragma unroll
        for (int k = 0; k < DV; ++k) acc += c[v][k];
        const size_t w = (size_t)g * A.n + i;
        st_if(A.post + w * 32 + lane, acc, live);
        const unsigned neg = __ballot_sync(kFull, acc < Real(0));
        if (lane == 0) {
            const unsigned hw = (neg & act) | (sold[v] & ~act);
            A.hard_w[w] = hw;
            if (A.hist_w) A.hist_w[((size_t)t * A.G) * A.n + w] = hw;
        }
    }
}

// Variable phase, general degrees (CSR) and isolated-per-matrix mode: also
// the per-matrix totals v2c_pass uses (_kernels.py:276-279).
template <class Real, bool ISO>
__device__ __forceinline__ void var_item(const DecodeArgs<Real>& A, int g, int i, int t,
                                         unsigned act, int lane)
{
    const int p0 = A.dv ? i * A.dv : ld_ro(A.var_ptr + i);
    const int dv = A.dv ? A.dv : ld_ro(A.var_ptr + i + 1) - p0;
    const bool live = (act >> lane) & 1u;
    const size_t w = (size_t)g * A.n + i;
    const unsigned nwd = ld_ro(A.noisy_w + w);
    const unsigned old = lane == 0 ? ld_cg(A.hard_w + w) : 0u;
    const Real L = ld_ro(A.Lmag + g * 32 + lane);
    const Real prior = ((nwd >> lane) & 1u) ? -L : L;
    const Real* c2vg = A.c2v + (size_t)g * A.slots * 32 + lane;
    Real acc = prior;
    if (!ISO) {
        for (int base = 0; base < dv; base += 32) {
            const int eid = base + lane < dv ? ld_ro(A.var_edge + p0 + base + lane) : 0;
            const int cnt = min(32, dv - base);
#pragma unroll 4
            for (int k = 0; k < cnt; ++k) {
                const int e = __shfl_sync(kFull, eid, k);
                acc += ld_cg_if(c2vg + (size_t)e * 32, live);
            }
        }
        st_if(A.post + w * 32 + lane, acc, live);
    } else {
        const size_t P = (size_t)(A.u + 1);
        Real part = prior;
        int l = 0;
        for (int base = 0; base < dv; base += 32) {
            const int eid = base + lane < dv ? ld_ro(A.var_edge + p0 + base + lane) : 0;
            const int cnt = min(32, dv - base);
            for (int k = 0; k < cnt; ++k) {
                const int e = __shfl_sync(kFull, eid, k);
                while (e >= A.edge_off[l + 1]) {  // close the totals of matrices before e's
                    st_if(A.post + (((size_t)g * P + l) * A.n + i) * 32 + lane, part, live);
                    part = prior;
                    ++l;
                }
                const Real cv = ld_cg_if(c2vg + (size_t)e * 32, live);
                acc += cv;
                part += cv;
            }
        }
        for (; l < A.u; ++l) {
            st_if(A.post + (((size_t)g * P + l) * A.n + i) * 32 + lane, part, live);
            part = prior;
        }
        st_if(A.post + (((size_t)g * P + A.u) * A.n + i) * 32 + lane, acc, live);
    }
    const unsigned neg = __ballot_sync(kFull, acc < Real(0));
    if (lane == 0) {
        const unsigned hw = (neg & act) | (old & ~act);
        A.hard_w[w] = hw;
        if (A.hist_w) A.hist_w[((size_t)t * A.G) * A.n + w] = hw;
    }
}

// Syndrome phase item: 32 consecutive checks (lane = check) of group g.
// Mismatch words (bit f = frame f) are turned into per-frame counts with 32
// ballots and added to cnt[t&1].
template <class Real>
__device__ __forceinline__ void syncheck_item(const DecodeArgs<Real>& A, int g, int blk, int t,
                                              unsigned act, int lane)
{
    const int j = blk * 32 + lane;
    unsigned mism = 0;
    if (j < A.C) {
        const unsigned* hw = A.hard_w + (size_t)g * A.n;
        const int d = ld_ro(A.deg + j);
        const int* row = A.chk_ell + j * A.Ds;
        unsigned par = 0;
        for (int k = 0; k < d; ++k) par ^= ld_cg(hw + ld_ro(row + k));
        mism = (par ^ ld_ro(A.syn_w + (size_t)g * A.C + j)) & act;
    }
    int c = 0;
#pragma unroll
    for (int f = 0; f < 32; ++f) {
        const int pc = __popc(__ballot_sync(kFull, (mism >> f) & 1u));
        if (lane == f) c = pc;
    }
    if (c) atomicAdd(A.cnt + (t & 1) * A.G * 32 + g * 32 + lane, c);
    if (__any_sync(kFull, c != 0) && lane == 0) atomicOr(A.any_bad + (t & 1), 1);
}

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <class Real>
__device__ __forceinline__ void stamp(const DecodeArgs<Real>& A, int& k)
{
    if (A.ts && blockIdx.x == 0 && threadIdx.x == 0 && k < A.ts_cap) A.ts[k] = globaltimer();
    ++k;
}

// Dynamic work distribution: warps claim chunks of consecutive items from a
// per-phase counter (balanced tails); a chunk's graph rows and per-item words
// are staged in the warp's shared-memory slice with one coalesced load.
template <int D> struct Chunk {
    static constexpr int CH = D <= 16 ? 32 : 8;   // items per claim (check / variable phases)
    static constexpr int SD = D | 1;               // odd smem row stride: conflict-free staging
};
constexpr int kSynChunk = 16;                      // syndrome-phase items (32 checks each)

// items per claim: CH for large phases, fewer when a phase has less than
// ~4 chunks per warp (small batches), so all warps get work
__device__ __forceinline__ int chunk_size(int total, int nwarps, int CH)
{
    return max(1, min(CH, total / (4 * nwarps)));
}

__device__ __forceinline__ int claim(unsigned* counter, int lane, int n)
{
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(counter, (unsigned)n);
    return (int)__shfl_sync(kFull, base, 0);
}

__device__ __forceinline__ unsigned group_mask(const int* cprev, int g, int lane)
{
    return __ballot_sync(kFull, ld_cg(cprev + g * 32 + lane) != 0);
}

// one claimed chunk of the check phase: items [base, end) of the G*C space
template <class Real, int D, bool DAMP, bool ISO>
__device__ __forceinline__ void check_chunk(const DecodeArgs<Real>& A, int base, int end, int t,
                                            const int* cprev, int lane, int* s_idx, unsigned* s_w,
                                            int* s_d)
{
    constexpr int SD = Chunk<D>::SD;
    const int rows = end - base;
    if (lane < rows) {
        const int item = base + lane;
        const int j = item % A.C;
        const int d = ld_ro(A.deg + j);
        s_d[lane] = d;
        s_w[lane] = ld_ro(A.syn_w + item);  // syn_w index == item (g*C + j)
        const int* row = A.chk_ell + j * A.Ds;
#pragma unroll
        for (int k = 0; k < D; ++k)
            if (k < d) s_idx[lane * SD + k] = ld_ro(row + k);
    }
    __syncwarp();
    int g = base / A.C;
    int j = base - g * A.C;
    unsigned act = group_mask(cprev, g, lane);
    Real L = ld_ro(A.Lmag + g * 32 + lane);
    for (int r = 0; r < rows; ++r) {
        if (act) check_item<Real, D, DAMP, ISO>(A, g, j, t, act, lane, s_idx + r * SD, s_d[r], s_w[r], L);
        if (++j == A.C && r + 1 < rows) {
            j = 0;
            ++g;
            act = group_mask(cprev, g, lane);
            L = ld_ro(A.Lmag + g * 32 + lane);
        }
    }
    __syncwarp();
}

// one claimed chunk of the variable phase (regular column degree DV)
template <class Real, int DV>
__device__ __forceinline__ void var_chunk_regular(const DecodeArgs<Real>& A, int base, int end, int t,
                                                  const int* cprev, int lane, int* s_idx, unsigned* s_w,
                                                  unsigned* s_old)
{
    constexpr int SV = DV | 1;
    const int rows = end - base;
    if (lane < rows) {
        const int item = base + lane;            // == g*n + i
        const int i = item % A.n;
        s_w[lane] = ld_ro(A.noisy_w + item);
        s_old[lane] = ld_cg(A.hard_w + item);
        const int* row = A.var_edge + i * DV;
#pragma unroll
        for (int k = 0; k < DV; ++k) s_idx[lane * SV + k] = ld_ro(row + k);
    }
    __syncwarp();
    int r = 0;
    while (r < rows) {
        const int item = base + r;
        const int g = item / A.n;
        const int i = item - g * A.n;
        const int span = min(rows - r, A.n - i);
        const unsigned act = group_mask(cprev, g, lane);
        const Real L = ld_ro(A.Lmag + g * 32 + lane);
        if (act) {
            for (int k = 0; k < span; k += 2)
                var_items_regular<Real, DV, 2>(A, g, i + k, min(2, span - k), t, act, lane,
                                               s_idx + (r + k) * SV, SV, s_w + r + k, s_old + r + k, L);
        }
        r += span;
    }
    __syncwarp();
}

#ifndef MBP_FP32_MIN_BLOCKS
#define MBP_FP32_MIN_BLOCKS 4
#endif
template <class Real, int D>
constexpr int decode_min_blocks() { return (sizeof(Real) == 4 && D <= 16) ? MBP_FP32_MIN_BLOCKS : 2; }

constexpr int kDecodeThreads = 256;

template <class Real, int D, bool DAMP, bool ISO>
__global__ void __launch_bounds__(kDecodeThreads, decode_min_blocks<Real, D>())
decode_kernel(const DecodeArgs<Real> A)
{
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthreads = gridDim.x * blockDim.x;
    const int nwarps = nthreads >> 5;
    const int F = A.G * 32;
    const int cblk = (A.C + 31) / 32;
    constexpr int CH = Chunk<D>::CH;
    constexpr int SLICE = CH * (Chunk<D>::SD > 9 ? Chunk<D>::SD : 9);   // ints per warp (check or var rows)
    __shared__ int s_idx_all[kDecodeThreads / 32][SLICE];
    __shared__ unsigned s_w_all[kDecodeThreads / 32][CH];
    __shared__ unsigned s_x_all[kDecodeThreads / 32][CH];
    int* s_idx = s_idx_all[warp];
    unsigned* s_w = s_w_all[warp];
    unsigned* s_x = s_x_all[warp];
    int ts_k = 0;
    int wc = 0;  // next work counter
    stamp(A, ts_k);

    // iteration 0: the uncorrected key against all u*m syndromes (_kernels.py:358-365)
    {
        const int total = A.G * cblk;
        for (int base = claim(A.work + wc, lane, kSynChunk); base < total;
             base = claim(A.work + wc, lane, kSynChunk))
            for (int item = base; item < min(base + kSynChunk, total); ++item)
                syncheck_item<Real>(A, item / cblk, item % cblk, 0, kFull, lane);
        ++wc;
    }

    int t = 1;
    int final_t = 0;
    for (;; ++t) {
        grid_barrier(A.barrier);
        stamp(A, ts_k);
        const int* cprev = A.cnt + ((t - 1) & 1) * F;
        // frames whose sweep t-1 decision satisfied every syndrome stop here
        for (int f = gtid; f < F; f += nthreads) {
            if (ld_cg(cprev + f) == 0 && A.iters[f] < 0) A.iters[f] = t - 1;
            A.cnt[(t & 1) * F + f] = 0;
        }
        if (ld_cg(A.any_bad + ((t - 1) & 1)) == 0 || t > A.max_it) {
            final_t = t - 1;
            break;
        }
        if (gtid == 0) A.any_bad[t & 1] = 0;

        {   // check phase
            const int total = A.G * A.C;
            const int ch = chunk_size(total, nwarps, CH);
            for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch))
                check_chunk<Real, D, DAMP, ISO>(A, base, min(base + ch, total), t, cprev, lane,
                                                s_idx, s_w, reinterpret_cast<int*>(s_x));
            ++wc;
        }
        grid_barrier(A.barrier);
        stamp(A, ts_k);
        {   // variable phase
            const int total = A.G * A.n;
            const int ch = chunk_size(total, nwarps, CH);
            for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch)) {
                const int end = min(base + ch, total);
                if (!ISO && A.dv == 6) {
                    var_chunk_regular<Real, 6>(A, base, end, t, cprev, lane, s_idx, s_w, s_x);
                } else if (!ISO && A.dv == 9) {
                    var_chunk_regular<Real, 9>(A, base, end, t, cprev, lane, s_idx, s_w, s_x);
                } else {
                    int item = base;
                    while (item < end) {
                        const int g = item / A.n;
                        const int i = item - g * A.n;
                        const unsigned act = group_mask(cprev, g, lane);
                        const int span = min(end - item, A.n - i);
                        if (act)
                            for (int k = 0; k < span; ++k) var_item<Real, ISO>(A, g, i + k, t, act, lane);
                        item += span;
                    }
                }
            }
            ++wc;
        }
        grid_barrier(A.barrier);
        stamp(A, ts_k);
        {   // syndrome phase
            const int total = A.G * cblk;
            for (int base = claim(A.work + wc, lane, kSynChunk); base < total;
                 base = claim(A.work + wc, lane, kSynChunk)) {
                const int end = min(base + kSynChunk, total);
                int g = base / cblk;
                unsigned act = group_mask(cprev, g, lane);
                for (int item = base; item < end; ++item) {
                    const int gi = item / cblk;
                    if (gi != g) { g = gi; act = group_mask(cprev, g, lane); }
                    if (act) syncheck_item<Real>(A, g, item - g * cblk, t, act, lane);
                }
            }
            ++wc;
        }
    }

    // per-frame results (DecodeResult fields, decoder.py:246-274)
    const int* cfin = A.cnt + (final_t & 1) * F;
    for (int f = gtid; f < A.B; f += nthreads) {
        const int c = ld_cg(cfin + f);
        const int it = A.iters[f];
        const bool conv = it >= 0;
        A.out_conv[f] = conv ? 1 : 0;
        A.out_iters[f] = conv ? it : A.max_it;
        A.out_mism[f] = conv ? 0 : c;
    }
    if (gtid == 0) *A.sweeps_run = final_t;
    stamp(A, ts_k);
}

// ---------------------------------------------------------------------------
// bit-matrix transposes between BitBlock rows and 32-frame words
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned load_row_u32(const uint8_t* row, long long byte0, long long nbytes)
{
    unsigned x = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
        if (byte0 + b < nbytes) x |= (unsigned)row[byte0 + b] << (8 * b);
    return x;
}

// 32x32 bit transpose across a warp: in lane l holds row l; out lane l holds
// column l (bit f of out = bit l of lane f's input).
__device__ __forceinline__ unsigned warp_transpose32(unsigned x, int lane)
{
    unsigned r = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const unsigned w = __ballot_sync(kFull, (x >> b) & 1u);
        if (lane == b) r = w;
    }
    return r;
}

// rows [B][row_bytes], bits [seg_off*8 + 32c, +32) of segment s of each row ->
// words[g][word_off + 32c + lane].  grid-stride over (g, segment, chunk).
__global__ void rows_to_words_kernel(const uint8_t* __restrict__ rows, long long row_bytes, int B,
                                     int G, int nseg, int seg_bits, long long seg_bytes,
                                     unsigned* __restrict__ words, unsigned* __restrict__ words2,
                                     long long words_per_group)
{
    const int lane = threadIdx.x & 31;
    const int chunks = (seg_bits + 31) / 32;
    const long long total = (long long)G * nseg * chunks;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long it = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < total; it += nw) {
        const int c = (int)(it % chunks);
        const int s = (int)((it / chunks) % nseg);
        const int g = (int)(it / ((long long)chunks * nseg));
        const int f = g * 32 + lane;
        unsigned x = 0;
        if (f < B) x = load_row_u32(rows + (long long)f * row_bytes + (long long)s * seg_bytes, 4LL * c, seg_bytes);
        const unsigned w = warp_transpose32(x, lane);
        const int bit = 32 * c + lane;
        if (bit < seg_bits) {
            const long long o = (long long)g * words_per_group + (long long)s * seg_bits + bit;
            words[o] = w;
            if (words2) words2[o] = w;
        }
    }
}

// words[g][word_off + 32c + lane] -> rows (inverse of rows_to_words_kernel)
__global__ void words_to_rows_kernel(const unsigned* __restrict__ words, long long words_per_group,
                                     int B, int G, int nseg, int seg_bits, long long seg_bytes,
                                     uint8_t* __restrict__ rows, long long row_bytes)
{
    const int lane = threadIdx.x & 31;
    const int chunks = (seg_bits + 31) / 32;
    const long long total = (long long)G * nseg * chunks;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long it = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < total; it += nw) {
        const int c = (int)(it % chunks);
        const int s = (int)((it / chunks) % nseg);
        const int g = (int)(it / ((long long)chunks * nseg));
        const int bit = 32 * c + lane;
        const unsigned w = bit < seg_bits ? words[(long long)g * words_per_group + (long long)s * seg_bits + bit] : 0u;
        const unsigned x = warp_transpose32(w, lane);
        const int f = g * 32 + lane;
        if (f < B) {
            uint8_t* r = rows + (long long)f * row_bytes + (long long)s * seg_bytes;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (4LL * c + b < seg_bytes) r[4LL * c + b] = (uint8_t)(x >> (8 * b));
        }
    }
}

// Alice side, Eq. 1: syndrome words of 32 frames per check, z = XOR of key
// words over the row (syndrome_pass, _kernels.py:220-227, 32 frames wide).
__global__ void syndrome_words_kernel(const uint8_t* __restrict__ deg, const int* __restrict__ chk_ell, int D,
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
        for (int k = 0, d = __ldg(deg + j); k < d; ++k) p ^= __ldg(kw + __ldg(row + k));
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
