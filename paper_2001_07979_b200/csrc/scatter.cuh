// scatter.cuh -- the production decode kernel: fp32, joint graph, no damping.
//
// Same flooding schedule, stopping rule and outputs as decode_kernel
// (decode.cuh; decode_loop, _kernels.py:323-379), restructured so that the
// edge messages of the common 2-3 sweep decode never touch HBM:
//
//  * sweep 1 needs no check phase.  Its inputs are the unclamped priors +-L
//    (_kernels.py:353-355), so every message of check j is
//        c2v_1(j -> b) = (-1)^(s_j xor y_b) * M_{d_j}(L),
//    s_j = the iteration-0 mismatch bit of check j (z_j xor parity of the
//    noisy key over the row), M_d(L) = 2 atanh(tanh(L/2)^(d-1)) clamped --
//    the reference's product of d-1 equal factors (c2v_pass,
//    _kernels.py:240-258), evaluated once per frame and degree in fp64.
//    The sweep-1 posterior is a gather of bits and table entries.
//  * posteriors are accumulated from the check side: a check phase adds its
//    new messages into acc[var] with red.global.add.s32 on fixed-point
//    values round(c2v * 2^S) (S chosen per launch so |acc| < 2^30).  Integer
//    addition is associative, so the posterior is deterministic and
//    independent of the order the checks run in; its error (<= dv * 2^-S-1)
//    is of the order of the fp32 summation it replaces.  The variable phase
//    only converts acc -> post (fp32), takes the hard decision (acc < 0,
//    ties -> 0 as in hard_pass, _kernels.py:304-307) and re-arms acc with the
//    prior.
//  * c2v_{t-1}, needed as the extrinsic correction v2c = post - c2v
//    (_kernels.py:276-281), is recomputed rather than stored for t <= 3:
//    sweep 2 rebuilds c2v_1 from bits, sweep 3 rebuilds c2v_1 and c2v_2 from
//    the stored sweep-1 posterior.  From sweep kStoreFrom on, c2v_t is also
//    stored (the few frames that need 4+ sweeps read it back).
//  * everything runs in the noisy-relative domain: for variable b the kernel
//    keeps post'_b = (-1)^y_b post_b and c2v'(j -> b) = (-1)^y_b c2v(j -> b)
//    (y = noisy key bit).  Negation is exact and commutes with clamp and
//    round-to-nearest, so this is the reference's arithmetic bit for bit, up
//    to the sign.  In this domain the prior is +L for every bit, Eq. 6's
//    syndrome sign (-1)^z_j becomes (-1)^s_j (z_j xor the row's noisy
//    parity), and every sweep-1 message of check j is the same value
//    (-1)^s_j M_{d_j}: the check phase needs no per-edge key bits.  The hard
//    decision is post_b < 0  <=>  (y_b ? post'_b > 0 : post'_b < 0).
//  * LLRs are carried in log2 units (x log2 e: u = 2^-|x| and the message
//    log2(S/D) need no scaling); posteriors are converted back on readback.
//  * Eq. 6 in (S, Delta) form: with u = e^-|x|, tanh(|x|/2) = (1-u)/(1+u);
//    for a set of edges A = prod(1+u), B = prod(1-u), S = A + B, D = A - B
//    combine as (S, D) x (1, u) = (S + uD, D + uS) -- only additions of
//    non-negative terms, so no cancellation where the product of tanh values
//    approaches 1 (the naive fp32 failure) -- and the
//    message is 2 atanh(B/A) = ln(S/D).  Exclusive products come from prefix
//    and suffix pairs; 3 MUFU per edge (ex2, 2 x lg2).
//
// Layout as in kernels.cuh (lane = frame, groups of 32 frames), plus
//   vb[Gc][n][3][32]   one 384-byte block per variable and group: line 0/1 =
//                      post' of even/odd sweeps (f32), line 2 = acc (s32), so
//                      one address per edge serves the posterior gathers and
//                      the accumulation (immediate offsets +128 / +256)
//   mis_w[Gc][C]       u32    iteration-0 mismatch words
//   Mtab[Dm+1][Fc]     f32    sweep-1 message magnitude per degree and frame
// (Gc = groups of the layout's allocation, Fc = 32 Gc).
#pragma once

#include "decode.cuh"

namespace mbp {

constexpr int kStoreFrom = 3;   // c2v_t is stored for t >= kStoreFrom
constexpr int kHotSweeps = 3;   // the hot instance runs sweeps 1..kHotSweeps

#ifndef MBP_SPAN_UNROLL
#define MBP_SPAN_UNROLL 2
#endif
constexpr int kSpanUnroll = MBP_SPAN_UNROLL;   // check-phase row loop unroll
constexpr int kVB = 96;         // 32-bit words per variable block (3 lines)

#ifndef MBP_SCATTER_MIN_BLOCKS
#define MBP_SCATTER_MIN_BLOCKS 4
#endif
// resident blocks per SM: 64 registers up to degree 8; wider rows keep two
// rows' gathers in flight and get 128.  Both budgets spill (ptxas -v: D = 7
// 3.4 KB, D = 14 2.0 KB of spill stores, mostly cold paths: the explicit-base
// and saturation variants); measured trade-off in DESIGN.md §10
template <int D>
#ifndef MBP_WIDE_MIN_BLOCKS
#define MBP_WIDE_MIN_BLOCKS 2
#endif
constexpr int scatter_min_blocks() { return D <= 8 ? MBP_SCATTER_MIN_BLOCKS : MBP_WIDE_MIN_BLOCKS; }

struct ScatterArgs {
    // graph
    int n, m, u, C, Ds;
    long long slots;                  // C * Ds
    const uint8_t* __restrict__ deg;  // [C]
    const int* __restrict__ chk_ell;  // [C*Ds]
    const int* __restrict__ var_ptr;  // [n+1] CSR into var_chk
    const int* __restrict__ var_chk;  // stacked check id of each edge, ascending edge order per variable
    int dv_max;
    int var_ptr_regular;              // every variable has degree dv_max (var_chk is [n][dv_max])
    int Dm;                           // Mtab degree bound (= Ds)
    // primary layout
    int G, B;
    float* vb;                        // [G][n][3][32]
    float* c2v;                       // [G][slots][32]
    const float* Lmag;                // [F]
    const float* Mtab;                // [Dm+1][F]
    int* Lfix;                        // [F]   round(L * 2^S), written by the kernel
    int* Mfix;                        // [Dm+1][F]
    const unsigned* noisy_w;
    const unsigned* syn_w;
    unsigned* mis_w;
    unsigned* hard_w;
    unsigned* hist_w;
    int* cnt;
    // compacted layout (capacity Gb groups)
    int Gb;
    float* vb_b;
    float* c2v_b;
    float* Mtab_b;
    int* Lfix_b;
    unsigned* noisy_b;
    unsigned* syn_b;
    unsigned* mis_b;
    unsigned* hard_b;
    int* cnt_b;
    int* fid_b;
    int* src_b;
    int* newslot;
    int* grp_cnt;
    int* ctrl;
    // hot/tail split: the hot instance (sweeps <= kHotSweeps, no saturating
    // inputs) stores its loop state here when frames remain; the tail
    // instance launched after it resumes from that state or exits at once.
    // nullptr: one full-instance launch runs the whole decode.
    int* resume;                      // [8]: flag, t, cpt, G, tc, may_compact, wc, ts_k
    // control
    int* any_bad;
    int* iters;
    unsigned* barrier;
    unsigned* work;
    int* sweeps_run;
    unsigned long long* ts;
    int ts_cap;
    const float* Lmax;                // [1] max prior magnitude of the batch
    // outputs
    uint8_t* out_conv;
    int* out_iters;
    int* out_mism;
    // config
    int max_it;
    float clamp;
    float sat;
};

template <bool CPT>
struct SL {
    const ScatterArgs& A;
    int G;                            // groups of the current layout
    __device__ __forceinline__ int Gc() const { return CPT ? A.Gb : A.G; }
    // lane's word of variable i's block in group g
    __device__ __forceinline__ float* vrow(size_t w, int lane) const { return (CPT ? A.vb_b : A.vb) + w * kVB + lane; }
    __device__ __forceinline__ float* c2v() const { return CPT ? A.c2v_b : A.c2v; }
    __device__ __forceinline__ unsigned* hard_w() const { return CPT ? A.hard_b : A.hard_w; }
    __device__ __forceinline__ unsigned* mis() const { return CPT ? A.mis_b : A.mis_w; }
    __device__ __forceinline__ int* cnt() const { return CPT ? A.cnt_b : A.cnt; }
    __device__ __forceinline__ unsigned noisy(size_t w) const { return CPT ? ld_cg(A.noisy_b + w) : ld_ro(A.noisy_w + w); }
    __device__ __forceinline__ unsigned syn(size_t w) const { return CPT ? ld_cg(A.syn_b + w) : ld_ro(A.syn_w + w); }
    __device__ __forceinline__ float M1(int d, int s) const
    {
        return CPT ? ld_cg(A.Mtab_b + (size_t)d * Gc() * 32 + s) : ld_ro(A.Mtab + (size_t)d * Gc() * 32 + s);
    }
    __device__ __forceinline__ int Lfix(int s) const { return ld_cg((CPT ? A.Lfix_b : A.Lfix) + s); }
};

// round(c * scale) for a message |c| <= clamp.  With MBP_FIX_MAGIC the
// conversion runs on the FMA pipe (c * 2^S + 1.5 * 2^23 rounds to the nearest
// integer, ties to even, when |c * 2^S| < 2^22 -- the kernel caps S for
// that) instead of F2I, which issues on the XU pipe next to the rule's MUFUs.
#ifndef MBP_FIX_MAGIC
#define MBP_FIX_MAGIC 0   // off: the 2^-16 resolution it forces changes failing frames' final states (measured)
#endif
__device__ __forceinline__ int fixq(float c, float scale)
{
#if MBP_FIX_MAGIC
    return __float_as_int(fmaf(c, scale, 12582912.0f)) - 0x4B400000;
#else
    return __float2int_rn(c * scale);
#endif
}

__device__ __forceinline__ const float* byte_off(const float* p, unsigned off)
{
    return reinterpret_cast<const float*>(reinterpret_cast<const char*>(p) + off);
}

// ptxas branches around a lane-predicated REDG (BSSY/BRA/BSYNC per edge), so
// dead lanes add 0 instead: the warp's line request is issued either way.
__device__ __forceinline__ void red_add(const float* p, int v)
{
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// Eq. 6, (S, Delta) form (header comment), in log2 units: inputs are the raw
// differences x = post' - c2v' (the clamp is applied here as min(|x|, clamp),
// the sign taken from x), u = 2^-|x|, output log2(S/D).  Slots k >= d (PAD)
// and, when SAT, inputs with |x| >= sat (where the reference's float64
// tanh(x/2) is exactly 1.0) get u = 0, the neutral factor (1, 0); a message
// whose other factors are all neutral has D = 0 -> log2(S/0) = inf -> +-clamp,
// the reference's `prod >= 1.0` branch (_kernels.py:249-252).  With
// clamp < sat no clamped input can reach sat, so SAT = false is exact.
// ---------------------------------------------------------------------------
template <int DD, bool PAD, bool SAT>
__device__ __forceinline__ void rule_sd(const float (&x)[DD], int d, unsigned flip, float clamp, float sat,
                                        float (&out)[DD])
{
    float uu[DD];
    unsigned sb[DD];
    unsigned tot = flip << 31;
#pragma unroll
    for (int k = 0; k < DD; ++k) {
        const bool in = !PAD || k < d;
        const float a = fminf(fabsf(x[k]), clamp);
        const float u = ex2_approx(-a);
        uu[k] = (in && (!SAT || a < sat)) ? u : 0.0f;
        sb[k] = in ? (__float_as_uint(x[k]) & 0x80000000u) : 0u;
        tot ^= sb[k];
    }
    // The first factor of each pass is (1, 0) x (1, u) = (1, u) exactly (u is
    // finite, in [0, 1]): written out so that the compiler folds the
    // multiplications by 1 and 0 it cannot prove away (0 * u for a NaN u).
    float sS[DD], sD[DD];
    float S = 1.0f, Dl = 0.0f;
#pragma unroll
    for (int k = DD - 1; k >= 0; --k) {
        sS[k] = S;
        sD[k] = Dl;
        if (k == DD - 1) {
            S = 1.0f;
            Dl = uu[k];
        } else {
            const float S2 = fmaf(Dl, uu[k], S);
            Dl = fmaf(S, uu[k], Dl);
            S = S2;
        }
    }
    float pS = 1.0f, pD = 0.0f;
#pragma unroll
    for (int k = 0; k < DD; ++k) {
        const float eS = k == 0 ? sS[k] : fmaf(pS, sS[k], pD * sD[k]);
        const float eD = k == 0 ? sD[k] : fmaf(pS, sD[k], pD * sS[k]);
        const float mag = fminf(lg2_approx(eS) - lg2_approx(eD), clamp);
        out[k] = __uint_as_float(__float_as_uint(mag) | (tot ^ sb[k]));
        if (k == 0) {
            pS = 1.0f;
            pD = uu[k];
        } else {
            const float S2 = fmaf(pD, uu[k], pS);
            pD = fmaf(pS, uu[k], pD);
            pS = S2;
        }
    }
}

// ---------------------------------------------------------------------------
// check phase (t >= 2).  A warp owns a claimed chunk of rows (checks) of one
// or two groups; lane = frame.  Row variable offsets are staged in shared
// memory as byte offsets of variable blocks (pad slots -> 0: they read
// variable 0 and add 0 to it, so no load needs a per-slot predicate).
// The base message c2v'_{s0-1} is rebuilt from the mismatch bit while
// t <= kStoreFrom (s0 = 2), read from the stored row otherwise (s0 = t); the
// chain c2v'_s = rule(clamp(post'_{s-1} - c2v'_{s-1})), s = s0..t, ends in
// c2v'_t, which is added into acc (and stored when t >= kStoreFrom).  The
// first gather (post'_{s0-1}) of the next row is issued before the current
// row's rule (software pipeline).  Dead lanes (converged frames, empty
// slots) run the same unpredicated gathers and rules (every word they read
// is allocated, every rule output finite: min(|x|, clamp) drops NaN) and
// are masked by their zero `scale`: their acc deltas round to 0.
// ---------------------------------------------------------------------------
template <int D, int DD, bool PAD, bool SAT, bool T2, bool CPT, bool C3 = false>
__device__ __forceinline__ void sc_row(const ScatterArgs& A, const SL<CPT>& S, const float (&p)[D], int d,
                                       unsigned sj, float M1, const unsigned* soff, bool live, int t_,
                                       const float* gb, const float* qrow, float* crow, float scale, bool absolute,
                                       const float (&p2)[D])
{
    // C3: sweep 3 with the rebuilt chain, post'_2 values prefetched by the caller
    // T2: sweep 2, the hot case (no chain, no store) compiled on its own
    const int t = T2 ? 2 : t_;
    const bool explicit_base = !T2 && t > kStoreFrom;
    float c[DD];
    if (!explicit_base) {
        const float c1 = sj ? -M1 : M1;          // c2v'_1, the same on every edge of the row
#pragma unroll
        for (int k = 0; k < DD; ++k) c[k] = c1;
    } else {
#pragma unroll
        for (int k = 0; k < DD; ++k) c[k] = ld_cg_if(qrow + k * 32, live && (!PAD || k < d));   // 0 when dead
    }
    float x[DD];
#pragma unroll
    for (int k = 0; k < DD; ++k) x[k] = p[k] - c[k];
    // acc holds prior + sum of c2v'_{t-1} (fixed point); adding the rounded
    // differences c2v'_t - c2v'_{t-1} leaves prior + sum of c2v'_t exactly
    int vold[DD];
    if (t == 2) {
        const int v1 = fixq(c[0], scale);   // row constant
#pragma unroll
        for (int k = 0; k < DD; ++k) vold[k] = v1;
    } else if (explicit_base) {
#pragma unroll
        for (int k = 0; k < DD; ++k) vold[k] = fixq(c[k], scale);
    }
    rule_sd<DD, PAD, SAT>(x, d, sj, A.clamp, A.sat, c);
    if (t > 2 && !explicit_base) {
        // chain: c2v'_s from post'_{s-1}, s = 3 .. t (vold = c2v'_{t-1})
        for (int s = 3; s <= t; ++s) {
            const float* gs = gb + ((s - 1) & 1) * 32;   // post'_{s-1} line
#pragma unroll
            for (int k = 0; k < DD; ++k) {
                float pv;
                if constexpr (C3) {
                    pv = p2[k];
                } else {
                    const float* q = byte_off(gs, soff[k]);
                    pv = ld_cg(q);
                }
                x[k] = pv - c[k];
                if (s == t) vold[k] = fixq(c[k], scale);
            }
            rule_sd<DD, PAD, SAT>(x, d, sj, A.clamp, A.sat, c);
        }
    }
    if (t >= kStoreFrom) {
        // only the row's own slots: the instance's degree bound D may exceed
        // the ELL stride Ds (rounded-up instances, rows of degree < 3)
#pragma unroll
        for (int k = 0; k < DD; ++k) st_if(crow + k * 32, c[k], !PAD || k < d);
    }
#pragma unroll
    for (int k = 0; k < DD; ++k) {
        const int v = fixq(c[k], scale) - (CPT && absolute ? 0 : vold[k]);
        red_add(byte_off(gb, soff[k]) + 64, (!PAD || k < d) ? v : 0);   // acc line
    }
}

// c2v'_{t-1} row base for lane `lane` of group g (explicit base only); the
// first sweep after a compaction reads it in place from the frame's
// original lane of the primary layout.
template <bool CPT>
__device__ __forceinline__ const float* sc_c2v_in_base(const ScatterArgs& A, const SL<CPT>& S, int g, int lane,
                                                       bool first_after_compaction)
{
    if (CPT && first_after_compaction) {
        const int s = ld_cg(A.src_b + g * 32 + lane);
        if (s >= 0) return A.c2v + (size_t)(s >> 5) * A.slots * 32 + (s & 31);
    }
    return S.c2v() + (size_t)g * A.slots * 32 + lane;
}

// rows [r0, r1) of the staged chunk, all in group g (first row j0)
template <int D, bool SAT, bool T2, bool CPT, bool C3 = false>
__device__ __forceinline__ void sc_span(const ScatterArgs& A, const SL<CPT>& S, int g, int j0, int r0, int r1, int t,
                                        unsigned act, int lane, const unsigned* s_off, const unsigned* s_m,
                                        const int* s_d, const float* s_m1, bool first, float scale)
{
    constexpr int SD = Chunk<D>::SD;
    if (T2) t = 2;
    if (C3) t = 3;
    const bool live = (act >> lane) & 1u;
    scale = live ? scale : 0.0f;
    const bool explicit_base = !T2 && t > kStoreFrom;
    const float* gb = S.vrow((size_t)g * A.n, lane);
    const float* qb = explicit_base ? sc_c2v_in_base<CPT>(A, S, g, lane, first) : nullptr;
    // first gather: post'_{s0-1}
    const float* gf = gb + (((explicit_base ? t : 2) - 1) & 1) * 32;
    const float* g2 = gb;    // post'_2 line (C3)
    float pn[D], pn2[C3 ? D : 1];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float* q = byte_off(gf, s_off[r0 * SD + k]);
        pn[k] = ld_cg(q);
        if constexpr (C3) {
            const float* q2 = byte_off(g2, s_off[r0 * SD + k]);
            pn2[k] = ld_cg(q2);
        }
    }
    int dn = s_d[r0];
    // two rows per loop pass for the narrow (64-register) instances: the
    // prefetch buffers alternate instead of being copied; wide rows keep one
    // (their 128-register budget is taken by the two-row chain prefetch)
#ifndef MBP_C3_UR
#define MBP_C3_UR 1   // the two-rule sweep-3 rows: one row per pass (registers for the chain)
#endif
    constexpr int UR = D <= 8 ? (C3 ? MBP_C3_UR : kSpanUnroll) : 1;
#pragma unroll (UR)
    for (int r = r0; r < r1; ++r) {
        float p[D], p2[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            p[k] = pn[k];
            if constexpr (C3) p2[k] = pn2[k];
        }
        const int d = dn;
        if (r + 1 < r1) {
            dn = s_d[r + 1];
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float* q = byte_off(gf, s_off[(r + 1) * SD + k]);
                pn[k] = ld_cg(q);
                if constexpr (C3) {
                    const float* q2 = byte_off(g2, s_off[(r + 1) * SD + k]);
                    pn2[k] = ld_cg(q2);
                }
            }
        }
        const unsigned sj = (s_m[r] >> lane) & 1u;
        float M1 = 0.0f;
        if (!explicit_base) {
            if constexpr (D <= 16) M1 = s_m1[d * 32 + lane];
            else M1 = S.M1(d, g * 32 + lane);
        }
        const unsigned* soff = s_off + r * SD;
        const int j = j0 + (r - r0);
        const float* qrow = explicit_base ? qb + (size_t)j * A.Ds * 32 : nullptr;
        float* crow = t >= kStoreFrom ? S.c2v() + ((size_t)g * A.slots + (size_t)j * A.Ds) * 32 + lane : nullptr;
        if (d == D)
            sc_row<D, D, false, SAT, T2, CPT, C3>(A, S, p, d, sj, M1, soff, live, t, gb, qrow, crow, scale,
                                                        first, p2);
        else if (D > 1 && d == D - 1)
            sc_row<D, (D > 1 ? D - 1 : 1), false, SAT, T2, CPT, C3>(A, S, p, d, sj, M1, soff, live, t, gb,
                                                                          qrow, crow, scale, first, p2);
        else
            sc_row<D, D, true, SAT, T2, CPT, C3>(A, S, p, d, sj, M1, soff, live, t, gb, qrow, crow, scale,
                                                       first, p2);
    }
}

template <int D, bool CPT, bool HOT>
__device__ __forceinline__ void sc_check_chunk(const ScatterArgs& A, const SL<CPT>& S, int base, int end, int t,
                                               const int* cprev, int lane, unsigned* s_off, unsigned* s_m,
                                               int* s_d, float* s_m1, bool first, float scale)
{
#ifndef MBP_C3
#define MBP_C3 1
#endif
    static_assert(!HOT || (MBP_C3 && kStoreFrom == 3 && kHotSweeps == 3),
                  "the hot instance runs sweeps 2 and 3 on the T2 / C3 variants only");
    constexpr int SD = Chunk<D>::SD;
    const int rows = end - base;
    if (lane < rows) {
        const int item = base + lane;
        const int j = item % A.C;
        const int d = ld_ro(A.deg + j);
        s_d[lane] = d;
        s_m[lane] = ld_cg(S.mis() + item);     // mis index == item (g*C + j)
        const int* row = A.chk_ell + (size_t)j * A.Ds;
#pragma unroll
        for (int k = 0; k < D; ++k) s_off[lane * SD + k] = k < d ? (unsigned)ld_ro(row + k) * (kVB * 4u) : 0u;
    }
    __syncwarp();
    int r = 0;
    while (r < rows) {
        const int item = base + r;
        const int g = item / A.C;
        const int j0 = item - g * A.C;
        const int span = min(rows - r, A.C - j0);
        const unsigned act = group_mask(cprev, g, lane);
        if (act) {
            if constexpr (D <= 16) {
                if (t <= kStoreFrom) {
#pragma unroll
                    for (int dd = 0; dd <= D; ++dd) s_m1[dd * 32 + lane] = S.M1(dd, g * 32 + lane);
                    __syncwarp();
                }
            }
            // fast variants: no input can saturate; sweeps 2 and 3 (the hot
            // cases) compiled on their own.  The hot instance has only these
            // two (the host launches it only when clamp < sat; it stops
            // before sweep kHotSweeps + 1), which keeps the cold
            // explicit-base and saturation code out of its register
            // allocation
            if (HOT || A.clamp < A.sat) {
                if (t == 2)
                    sc_span<D, false, true, CPT>(A, S, g, j0, r, r + span, t, act, lane, s_off, s_m, s_d, s_m1, first,
                                                 scale);
                else if (MBP_C3 && t == 3 && kStoreFrom == 3)
                    sc_span<D, false, false, CPT, true>(A, S, g, j0, r, r + span, t, act, lane, s_off, s_m, s_d, s_m1,
                                                        first, scale);
                else if constexpr (!HOT)
                    sc_span<D, false, false, CPT>(A, S, g, j0, r, r + span, t, act, lane, s_off, s_m, s_d, s_m1, first,
                                                  scale);
            } else if constexpr (!HOT) {
                sc_span<D, true, false, CPT>(A, S, g, j0, r, r + span, t, act, lane, s_off, s_m, s_d, s_m1, first,
                                             scale);
            }
            __syncwarp();
        }
        r += span;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// variable phases
// ---------------------------------------------------------------------------

// Sweep 1: post'_1 = L + sum of the sweep-1 messages (-1)^s_j M_{d_j}, in
// fixed point (what the check-side accumulation of later sweeps computes);
// arms acc with the prior for sweep 2.  General column degrees: lanes load
// the variable's check ids, mismatch words and degrees, the warp walks them
// with shuffles.
// RECOMP (compaction at t = kStoreFrom, MBP_CMP_RECOMP): rebuild post'_1 of a
// compacted frame from its moved mismatch words instead of gathering it from
// the frame's old lane; writes the post'_1 line only (the move re-armed acc,
// hard words are not touched).  Mfix rows have stride A.G * 32.
template <bool CPT, bool RECOMP = false>
__device__ __forceinline__ void sc_var1_item(const ScatterArgs& A, const SL<CPT>& S, int g, int i, unsigned act,
                                             int lane, const int* Mfix, int Lf, float iscale)
{
    const bool live = (act >> lane) & 1u;
    const size_t w = (size_t)g * A.n + i;
    const unsigned yw = S.noisy(w);
    const unsigned y = (yw >> lane) & 1u;
    int a = Lf;
    const int p0 = ld_ro(A.var_ptr + i), dv = ld_ro(A.var_ptr + i + 1) - p0;
    for (int base = 0; base < dv; base += 32) {
        unsigned mk = 0;
        int dk = 0;
        if (base + lane < dv) {
            const int j = ld_ro(A.var_chk + p0 + base + lane);
            mk = ld_cg(S.mis() + (size_t)g * A.C + j);
            dk = ld_ro(A.deg + j);
        }
        const int cntk = min(32, dv - base);
        for (int k = 0; k < cntk; ++k) {
            const unsigned mw = __shfl_sync(kFull, mk, k);
            const int d = __shfl_sync(kFull, dk, k);
            const int mf = ld_cg(Mfix + (size_t)d * A.G * 32);
            a += ((mw >> lane) & 1u) ? -mf : mf;
        }
    }
    float* vr = S.vrow(w, lane);
    st_if(vr + 32, (float)a * iscale, live);
    if constexpr (RECOMP) return;
    if (live) reinterpret_cast<int*>(vr)[64] = a;   // acc = post'_1 in fixed point
    const unsigned neg = __ballot_sync(kFull, y ? a > 0 : a < 0);
    if (lane == 0) {
        // the iteration-0 decision of every frame is its noisy key
        const unsigned hw = (neg & act) | (yw & ~act);
        S.hard_w()[w] = hw;
        if (A.hist_w) A.hist_w[((size_t)1 * A.G) * A.n + w] = hw;
    }
}

// Sweep 1 for a regular column degree DV (6 or 9), check degree D <= 16: one
// chunk of <= 32 variables.  The chunk's mismatch words and check degrees
// are staged in shared memory with independent loads (two dependent round
// trips per chunk), the lane's Mfix row per degree sits in a shared table.
template <int D, int DV, bool CPT, bool RECOMP = false>
__device__ __forceinline__ void sc_var1_chunk(const ScatterArgs& A, const SL<CPT>& S, int base, int end,
                                              const int* cprev, int lane, unsigned* s_mis, uint8_t* s_deg,
                                              unsigned* s_y, int* s_mf, float iscale)
{
    const int rows = end - base;
    const int tot = rows * DV;
    // lane v: group / variable of chunk row v (one division per lane)
    const int gl_ = (base + lane) / A.n;
    const int il_ = base + lane - gl_ * A.n;
    if (lane < rows) s_y[lane] = S.noisy(base + lane);
    for (int b0 = 0; b0 < tot; b0 += 32) {
        const int idx = b0 + lane;
        const int v = idx < tot ? idx / DV : 0;
        const int k = idx - v * DV;
        const int gv = __shfl_sync(kFull, gl_, v);
        const int iv = __shfl_sync(kFull, il_, v);
        if (idx < tot) {
            const int j = ld_ro(A.var_chk + (size_t)iv * DV + k);
            s_mis[idx] = ld_cg(S.mis() + (size_t)gv * A.C + j);
            s_deg[idx] = ld_ro(A.deg + j);
        }
    }
    __syncwarp();
#ifndef MBP_V1_UNI
#define MBP_V1_UNI 0   // off: no gain measured (the phase is latency-bound, not issue-bound)
#endif
    // variables whose checks all have one degree d (95 % of cfg 2's): the
    // sum of +-M_d is M_d * (DV - 2 * #mismatches) -- one table read instead
    // of a dependent (degree, table) pair per edge; the same integer
    int8_t* s_uni = reinterpret_cast<int8_t*>(s_deg + 32 * 9);
    if (MBP_V1_UNI && lane < rows) {
        const int d0 = s_deg[lane * DV];
        bool same = true;
#pragma unroll
        for (int k = 1; k < DV; ++k) same &= s_deg[lane * DV + k] == d0;
        s_uni[lane] = same ? (int8_t)d0 : (int8_t)-1;
    }
    __syncwarp();
    int r = 0;
    while (r < rows) {
        const int item = base + r;
        const int g = __shfl_sync(kFull, gl_, r);
        const int i = item - g * A.n;
        const int span = min(rows - r, A.n - i);
        const unsigned act = group_mask(cprev, g, lane);
        if (act) {
            {
                // the lane's frame slot in the primary layout (Mfix is indexed by it)
                int src = g * 32 + lane;
                if constexpr (RECOMP) src = max(ld_cg(A.src_b + g * 32 + lane), 0);
#pragma unroll
                for (int d = 0; d <= D; ++d) s_mf[d * 32 + lane] = ld_cg(A.Mfix + (size_t)d * A.G * 32 + src);
            }
            __syncwarp();
            const bool live = (act >> lane) & 1u;
            const int Lf = S.Lfix(g * 32 + lane);
            const unsigned lbit = 1u << lane;
            if (act == kFull && !A.hist_w) {
                // every lane live, no history: UV variables per pass, no predicates
#ifndef MBP_V1_UV
#define MBP_V1_UV 8   // 8 variables per pass: cfg 3 3.033 -> 3.009 ms (the D = 14 sweep-3 check, register allocation), cfg 2 unchanged
#endif
                constexpr int UV = MBP_V1_UV;
                int v = r;
                for (; v + UV - 1 < r + span; v += UV) {
                    int a[UV];
#pragma unroll
                    for (int q = 0; q < UV; ++q) {
                        const int du = MBP_V1_UNI ? (int)s_uni[v + q] : -1;
                        if (du >= 0) {
                            int cnt = 0;
#pragma unroll
                            for (int k = 0; k < DV; ++k) cnt += (s_mis[(v + q) * DV + k] >> lane) & 1u;
                            a[q] = Lf + s_mf[du * 32 + lane] * (DV - 2 * cnt);
                        } else {
                            a[q] = Lf;
#pragma unroll
                            for (int k = 0; k < DV; ++k) {
                                const int mq = s_mf[s_deg[(v + q) * DV + k] * 32 + lane];
                                a[q] += (s_mis[(v + q) * DV + k] & lbit) ? -mq : mq;
                            }
                        }
                    }
                    const size_t w = (size_t)base + v;
                    float* vr = S.vrow(w, lane);
                    if constexpr (RECOMP) {
#pragma unroll
                        for (int q = 0; q < UV; ++q) vr[q * kVB + 32] = (float)a[q] * iscale;
                        continue;
                    }
                    unsigned nq[UV];
#pragma unroll
                    for (int q = 0; q < UV; ++q) {
                        vr[q * kVB + 32] = (float)a[q] * iscale;
                        reinterpret_cast<int*>(vr)[q * kVB + 64] = a[q];   // acc = post'_1 in fixed point
                        const unsigned yq = s_y[v + q] & lbit;
                        nq[q] = __ballot_sync(kFull, yq ? a[q] > 0 : a[q] < 0);
                    }
                    if (lane < UV) {
                        unsigned hw = nq[0];
#pragma unroll
                        for (int q = 1; q < UV; ++q) hw = lane == q ? nq[q] : hw;
                        S.hard_w()[w + lane] = hw;
                    }
                }
                for (; v < r + span; ++v) {
                    int a0 = Lf;
#pragma unroll
                    for (int k = 0; k < DV; ++k) {
                        const int m0 = s_mf[s_deg[v * DV + k] * 32 + lane];
                        a0 += (s_mis[v * DV + k] & lbit) ? -m0 : m0;
                    }
                    const size_t w = (size_t)base + v;
                    float* vr = S.vrow(w, lane);
                    vr[32] = (float)a0 * iscale;
                    if constexpr (RECOMP) continue;
                    reinterpret_cast<int*>(vr)[64] = a0;
                    const unsigned n0 = __ballot_sync(kFull, (s_y[v] & lbit) ? a0 > 0 : a0 < 0);
                    if (lane == 0) S.hard_w()[w] = n0;
                }
            } else {
                for (int v = r; v < r + span; ++v) {
                    const size_t w = (size_t)base + v;
                    const unsigned yw = s_y[v];
                    const unsigned y = (yw >> lane) & 1u;
                    int a = Lf;
#pragma unroll
                    for (int k = 0; k < DV; ++k) {
                        const unsigned mw = s_mis[v * DV + k];
                        const int mf = s_mf[s_deg[v * DV + k] * 32 + lane];
                        a += ((mw >> lane) & 1u) ? -mf : mf;
                    }
                    float* vr = S.vrow(w, lane);
                    st_if(vr + 32, (float)a * iscale, live);
                    if constexpr (RECOMP) continue;
                    if (live) reinterpret_cast<int*>(vr)[64] = a;   // acc = post'_1 in fixed point
                    const unsigned neg = __ballot_sync(kFull, y ? a > 0 : a < 0);
                    if (lane == 0) {
                        const unsigned hw = (neg & act) | (yw & ~act);
                        S.hard_w()[w] = hw;
                        if (A.hist_w) A.hist_w[((size_t)1 * A.G) * A.n + w] = hw;
                    }
                }
            }
            __syncwarp();
        }
        r += span;
    }
    __syncwarp();
}

// sweep t >= 2: acc -> post'_t and the hard decision (acc is not re-armed:
// the check phase adds message differences).
template <bool CPT, int U>
__device__ __forceinline__ void sc_var_chunk(const ScatterArgs& A, const SL<CPT>& S, int base, int end, int t,
                                             const int* cprev, int lane, unsigned* s_w, unsigned* s_old,
                                             float iscale)
{
    const int rows = end - base;
    if (lane < rows) {
        s_w[lane] = S.noisy(base + lane);
        s_old[lane] = ld_cg(S.hard_w() + base + lane);
    }
    __syncwarp();
    const int slot = (t & 1) * 32;
    int r = 0;
    while (r < rows) {
        const int item = base + r;
        const int g = item / A.n;
        const int i = item - g * A.n;
        const int span = min(rows - r, A.n - i);
        const unsigned act = group_mask(cprev, g, lane);
        if (act) {
            const bool live = (act >> lane) & 1u;
            for (int k0 = 0; k0 < span; k0 += U) {
                int a[U];
#pragma unroll
                for (int v = 0; v < U; ++v) {
                    const size_t w = (size_t)item + k0 + v;
                    a[v] = (k0 + v < span && live) ? ld_cg(reinterpret_cast<const int*>(S.vrow(w, lane)) + 64) : 0;
                }
#pragma unroll
                for (int v = 0; v < U; ++v) {
                    if (k0 + v >= span) break;
                    const size_t w = (size_t)item + k0 + v;
                    const unsigned y = (s_w[r + k0 + v] >> lane) & 1u;
                    float* vr = S.vrow(w, lane);
                    st_if(vr + slot, (float)a[v] * iscale, live);
                    const unsigned neg = __ballot_sync(kFull, y ? a[v] > 0 : a[v] < 0);
                    if (lane == 0) {
                        const unsigned hw = (neg & act) | (s_old[r + k0 + v] & ~act);
                        S.hard_w()[w] = hw;
                        if (A.hist_w) A.hist_w[((size_t)t * A.G) * A.n + w] = hw;
                    }
                }
            }
        }
        r += span;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// syndrome phase (mismatch_count, _kernels.py:310-320): 32 consecutive checks
// of group g per warp item (lane = check); the mismatch word (bit f = frame
// f) becomes per-frame counts via a bit transpose + popc, returned in lane f.  At t = 0
// the full mismatch words are stored (the sweep-1 message signs).  Callers
// accumulate counts over their chunk and flush once per group: per-item
// atomics on the 32 counters of a group all land on one L2 line and
// serialise.
// ---------------------------------------------------------------------------
template <int D, bool CPT>
__device__ __forceinline__ int sc_syncheck_item(const ScatterArgs& A, const SL<CPT>& S, int g, int blk, int t,
                                                unsigned act, int lane)
{
    constexpr int DU = D < 16 ? D : 16;      // row ids loaded in parallel
    const int j = blk * 32 + lane;
    unsigned mism = 0;
    if (j < A.C) {
        const unsigned* hw = S.hard_w() + (size_t)g * A.n;
        const int d = ld_ro(A.deg + j);
        const int* row = A.chk_ell + (size_t)j * A.Ds;
        unsigned par = 0;
        for (int k0 = 0; k0 < d; k0 += DU) {
            int id[DU];
#pragma unroll
            for (int k = 0; k < DU; ++k) id[k] = k0 + k < d ? ld_ro(row + k0 + k) : -1;
#pragma unroll
            for (int k = 0; k < DU; ++k)
                if (id[k] >= 0) par ^= ld_cg(hw + id[k]);
        }
        const unsigned full = par ^ S.syn((size_t)g * A.C + j);
        if (t == 0) S.mis()[(size_t)g * A.C + j] = full;
        mism = full & act;
    }
    // lane f: popcount of bit f over the 32 checks = transpose, then popc
    return __any_sync(kFull, mism != 0) ? __popc(warp_transpose32(mism, lane)) : 0;
}

// Two items of one group at once (MBP_SYN_PAIR): the rows' id and
// hard-word loads are issued together, so each lane has twice the loads in
// flight through the two dependent rounds (ids, then words).
template <int D, bool CPT>
__device__ __forceinline__ int sc_syncheck_pair(const ScatterArgs& A, const SL<CPT>& S, int g, int blk, int t,
                                                unsigned act, int lane)
{
    constexpr int DU = D < 16 ? D : 16;
    const int j0 = blk * 32 + lane, j1 = j0 + 32;
    const bool v0 = j0 < A.C, v1 = j1 < A.C;
    const unsigned* hw = S.hard_w() + (size_t)g * A.n;
    const int d0 = v0 ? ld_ro(A.deg + j0) : 0, d1 = v1 ? ld_ro(A.deg + j1) : 0;
    const int* r0 = A.chk_ell + (size_t)j0 * A.Ds;
    const int* r1 = A.chk_ell + (size_t)j1 * A.Ds;
    unsigned p0 = 0, p1 = 0;
    const int dm = max(d0, d1);
    for (int k0 = 0; k0 < dm; k0 += DU) {
        int a[DU], b[DU];
#pragma unroll
        for (int k = 0; k < DU; ++k) {
            a[k] = k0 + k < d0 ? ld_ro(r0 + k0 + k) : -1;
            b[k] = k0 + k < d1 ? ld_ro(r1 + k0 + k) : -1;
        }
#pragma unroll
        for (int k = 0; k < DU; ++k) {
            if (a[k] >= 0) p0 ^= ld_cg(hw + a[k]);
            if (b[k] >= 0) p1 ^= ld_cg(hw + b[k]);
        }
    }
    unsigned m0 = 0, m1 = 0;
    if (v0) {
        const unsigned full = p0 ^ S.syn((size_t)g * A.C + j0);
        if (t == 0) S.mis()[(size_t)g * A.C + j0] = full;
        m0 = full & act;
    }
    if (v1) {
        const unsigned full = p1 ^ S.syn((size_t)g * A.C + j1);
        if (t == 0) S.mis()[(size_t)g * A.C + j1] = full;
        m1 = full & act;
    }
    int c = 0;
    if (__any_sync(kFull, m0 != 0)) c += __popc(warp_transpose32(m0, lane));
    if (__any_sync(kFull, m1 != 0)) c += __popc(warp_transpose32(m1, lane));
    return c;
}

// items per claim: about one claim per warp (few flushes per group line),
// at least 8 so small batches do not spread thin
__device__ __forceinline__ int syn_chunk(int total, int nwarps)
{
    return min(64, max(8, (total + nwarps - 1) / nwarps));
}

// one claimed chunk [base, end) of the syndrome phase (items g*cblk + blk)
template <int D, bool CPT>
__device__ __forceinline__ void sc_syncheck_chunk(const ScatterArgs& A, const SL<CPT>& S, int base, int end, int t,
                                                  const int* cprev, int cblk, int lane)
{
    int g = base / cblk;
    unsigned act = cprev ? group_mask(cprev, g, lane) : kFull;
    int c = 0;
    bool bad = false;
#ifndef MBP_SYN_PAIR
#define MBP_SYN_PAIR 1
#endif
    for (int item = base; item < end;) {
        const int gi = item / cblk;
        if (gi != g) {
            if (c) atomicAdd(S.cnt() + (t & 1) * S.G * 32 + g * 32 + lane, c);
            bad |= c != 0;
            c = 0;
            g = gi;
            act = cprev ? group_mask(cprev, g, lane) : kFull;
        }
        const bool pair = MBP_SYN_PAIR && item + 1 < end && (item + 1) / cblk == g;
        if (act) {
            if (pair) c += sc_syncheck_pair<D, CPT>(A, S, g, item - g * cblk, t, act, lane);
            else c += sc_syncheck_item<D, CPT>(A, S, g, item - g * cblk, t, act, lane);
        }
        item += pair ? 2 : 1;
    }
    if (c) atomicAdd(S.cnt() + (t & 1) * S.G * 32 + g * 32 + lane, c);
    bad |= c != 0;
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(A.any_bad + (t & 1), 1);
}

// MBP_CMP_RECOMP: a compaction at t <= kStoreFrom moves post'_2 and re-arms
// acc, and post'_1 (= L + sum of +-M_d over the iteration-0 mismatch bits,
// integer arithmetic: the same value) is rebuilt in the compacted layout from
// the moved mismatch words instead of being gathered sector by sector from
// the frames' old lanes.
#ifndef MBP_CMP_RECOMP
#define MBP_CMP_RECOMP 1   // cfg 2: move 0.117 -> 0.080 ms, + 0.033 ms rebuild phase: kernel 1.342 -> 1.332 ms
#endif
// short keys: the rebuild phase's fixed cost (a claimed phase + a grid
// barrier) exceeds the sectors it saves (cfg 1, n = 4096: +0.01 ms)
__device__ __forceinline__ bool cmp_recomp(const ScatterArgs& A, int t)
{
    return MBP_CMP_RECOMP && t <= kStoreFrom && A.n >= 16384;
}

// ---------------------------------------------------------------------------
// compaction (cf. decode.cuh compact()): repack the undecided frames into
// dense groups of the secondary layout at the start of sweep t >= 2
// ---------------------------------------------------------------------------
__device__ __forceinline__ int sc_compact(const ScatterArgs& A, int t, int gw, int nw, int gtid, int nthreads,
                                          int lane)
{
    const int F = A.G * 32;
    const int* cprev = A.cnt + ((t - 1) & 1) * F;
    stamp_compact(A, 0);
    if (blockIdx.x == 0) {
        __shared__ int s_part[kDecodeThreads];
        const int per = (A.G + blockDim.x - 1) / blockDim.x;
        const int g0 = threadIdx.x * per, g1 = min(A.G, g0 + per);
        int sum = 0;
        for (int g = g0; g < g1; ++g) sum += ld_cg(A.grp_cnt + g);
        s_part[threadIdx.x] = sum;
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
            for (int k = 0; k < (int)blockDim.x; ++k) { const int v = s_part[k]; s_part[k] = run; run += v; }
        }
        __syncthreads();
        int run = s_part[threadIdx.x];
        for (int g = g0; g < g1; ++g) { const int v = ld_cg(A.grp_cnt + g); A.grp_cnt[g] = run; run += v; }
    }
    grid_barrier(A.barrier);
    for (int g = gw; g < A.G; g += nw) {
        const bool und = ld_cg(cprev + g * 32 + lane) != 0;
        const unsigned msk = __ballot_sync(kFull, und);
        if (und) {
            const int s2 = ld_cg(A.grp_cnt + g) + __popc(msk & ((1u << lane) - 1u));
            A.newslot[g * 32 + lane] = s2;
            A.src_b[s2] = g * 32 + lane;
            A.fid_b[s2] = g * 32 + lane;
        }
    }
    grid_barrier(A.barrier);
    stamp_compact(A, 1);
    const int nund = ld_cg(A.ctrl + 2 * t);
    const int Gn = (nund + 31) / 32;
    const int Fb = Gn * 32;
    // variable blocks: the posteriors the next check phase reads (post'_1 and
    // post'_2 while the base is rebuilt from bits, t <= kStoreFrom, else
    // post'_{t-1}); acc is re-armed with the prior (+L in the relative
    // domain) and the first compacted check phase adds absolute messages
    {
        const bool both = t <= kStoreFrom;
        const bool recomp = cmp_recomp(A, t);   // post'_1 rebuilt after the move (sc_recomp_post1)
        const int keep = ((t - 1) & 1) * 32;
#ifndef MBP_MOVE_XU
#define MBP_MOVE_XU 4
#endif
        constexpr int XU = MBP_MOVE_XU;   // variables per lane and pass (gathers in flight)
        const long long xchunks = (A.n + XU - 1) / XU;
        for (long long it = gw; it < (long long)Gn * xchunks; it += nw) {
            const int g2 = (int)(it / xchunks);
            const int i0 = (int)(it - (long long)g2 * xchunks) * XU;
            const int s = ld_cg(A.src_b + g2 * 32 + lane);
            const float* src = A.vb + (s >= 0 ? ((size_t)(s >> 5) * A.n * kVB + (s & 31)) : 0);
            float* dst = A.vb_b + (size_t)g2 * A.n * kVB + lane;
            const int Lf = s >= 0 ? ld_cg(A.Lfix + s) : 0;
            float v0[XU], v1[XU];
#pragma unroll
            for (int k = 0; k < XU; ++k) {
                const bool ok = s >= 0 && i0 + k < A.n;
                const size_t o = (size_t)(i0 + k) * kVB;
                v0[k] = ok && (both || keep == 0) ? __ldca(src + o) : 0.0f;
                v1[k] = ok && ((both && !recomp) || keep == 32) ? __ldca(src + o + 32) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < XU; ++k) {
                if (i0 + k >= A.n) break;
                float* d = dst + (size_t)(i0 + k) * kVB;
                d[0] = v0[k];
                if (!recomp) d[32] = v1[k];
                reinterpret_cast<int*>(d)[64] = Lf;
            }
        }
    }
    // (hard words are not moved: every moved frame is live in sweep t, whose
    // variable phase writes its compacted hard word before any reader)
    move_bits(A.noisy_w, A.noisy_b, A.n, Gn, A.src_b, gw, nw, lane);
    move_bits(A.syn_w, A.syn_b, A.C, Gn, A.src_b, gw, nw, lane);
    move_bits(A.mis_w, A.mis_b, A.C, Gn, A.src_b, gw, nw, lane);
    for (int s2 = gtid; s2 < Fb; s2 += nthreads) {
        const int s = ld_cg(A.src_b + s2);
        A.Lfix_b[s2] = s >= 0 ? ld_cg(A.Lfix + s) : 0;
        for (int d = 0; d <= A.Dm; ++d)
            A.Mtab_b[(size_t)d * A.Gb * 32 + s2] = s >= 0 ? A.Mtab[(size_t)d * A.G * 32 + s] : 0.0f;
        A.cnt_b[((t - 1) & 1) * Fb + s2] = s >= 0 ? ld_cg(cprev + s) : 0;
        A.cnt_b[(t & 1) * Fb + s2] = 0;
    }
    stamp_compact(A, 2);
    grid_barrier(A.barrier);
    stamp_compact(A, 3);
    if (gtid == 0) A.sweeps_run[1] = t;
    return Gn;
}

// post'_1 of the compacted frames (MBP_CMP_RECOMP), right after a compaction
// at sweep t <= kStoreFrom: the sweep-1 variable phase in RECOMP mode
template <int D>
__device__ __forceinline__ void sc_recomp_post1(const ScatterArgs& A, int G, int t, int& wc, int lane, int nwarps,
                                                unsigned* s_w, unsigned* s_v1m, uint8_t* s_v1d, int* s_mf,
                                                float iscale)
{
    const SL<true> S{A, G};
    const int* cp = A.cnt_b + ((t - 1) & 1) * G * 32;   // compacted frames' counts: live lanes
    const int total = G * A.n;
    const bool v1_staged = D <= 16 && (A.dv_max == 6 || A.dv_max == 9) && A.var_ptr_regular;
    if (v1_staged) {
        if constexpr (D <= 16) {
            const int ch = chunk_size(total, nwarps, 32);
            for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch)) {
                if (A.dv_max == 6)
                    sc_var1_chunk<D, 6, true, true>(A, S, base, min(base + ch, total), cp, lane, s_v1m, s_v1d, s_w,
                                                    s_mf, iscale);
                else
                    sc_var1_chunk<D, 9, true, true>(A, S, base, min(base + ch, total), cp, lane, s_v1m, s_v1d, s_w,
                                                    s_mf, iscale);
            }
        }
    } else {
        for (int base = claim(A.work + wc, lane, 8); base < total; base = claim(A.work + wc, lane, 8)) {
            const int end = min(base + 8, total);
            for (int item = base; item < end; ++item) {
                const int g = item / A.n;
                const unsigned act = group_mask(cp, g, lane);
                if (act) {
                    const int src = max(ld_cg(A.src_b + g * 32 + lane), 0);
                    sc_var1_item<true, true>(A, S, g, item - g * A.n, act, lane, A.Mfix + src,
                                             S.Lfix(g * 32 + lane), iscale);
                }
            }
        }
    }
    ++wc;
}

// ---------------------------------------------------------------------------
// one sweep t in a given layout
// ---------------------------------------------------------------------------
template <int D, bool CPT, bool HOT>
__device__ __forceinline__ void sc_sweep(const ScatterArgs& A, int G, int t, int& wc, int& ts_k, int lane, int nwarps,
                                         int* s_idx, unsigned* s_w, unsigned* s_x, unsigned* s_m, unsigned* s_v1m,
                                         uint8_t* s_v1d, int* s_mf, bool first, float scale, float iscale)
{
    const SL<CPT> S{A, G};
    constexpr int CH = Chunk<D>::CH;
    const int cblk = (A.C + 31) / 32;
    const int* cp = S.cnt() + ((t - 1) & 1) * G * 32;
    if (t >= 2) {   // check phase
        const int total = G * A.C;
        const int ch = chunk_size(total, nwarps, CH);
        for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch)) {
            sc_check_chunk<D, CPT, HOT>(A, S, base, min(base + ch, total), t, cp, lane,
                                   reinterpret_cast<unsigned*>(s_idx), s_m, reinterpret_cast<int*>(s_x),
                                   reinterpret_cast<float*>(s_v1m), first, scale);
        }
        ++wc;
        grid_barrier(A.barrier);
        stamp(A, ts_k);
    } else {
        stamp(A, ts_k);   // keep three stamps per sweep
    }
    {   // variable phase
        const int total = G * A.n;
        const bool v1_staged = D <= 16 && (A.dv_max == 6 || A.dv_max == 9) && A.var_ptr_regular;
        if (t == 1 && v1_staged) {
            if constexpr (D <= 16) {
                const int ch = chunk_size(total, nwarps, 32);
                for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch)) {
                    if (A.dv_max == 6)
                        sc_var1_chunk<D, 6, CPT>(A, S, base, min(base + ch, total), cp, lane, s_v1m, s_v1d, s_w,
                                                 s_mf, iscale);
                    else
                        sc_var1_chunk<D, 9, CPT>(A, S, base, min(base + ch, total), cp, lane, s_v1m, s_v1d, s_w,
                                                 s_mf, iscale);
                }
            }
        } else if (t == 1) {
            // general column degrees: one variable per warp pass
            for (int base = claim(A.work + wc, lane, 8); base < total; base = claim(A.work + wc, lane, 8)) {
                const int end = min(base + 8, total);
                int g = base / A.n;
                unsigned act = group_mask(cp, g, lane);
                for (int item = base; item < end; ++item) {
                    const int gi = item / A.n;
                    if (gi != g) { g = gi; act = group_mask(cp, g, lane); }
                    if (act)
                        sc_var1_item<CPT>(A, S, g, item - g * A.n, act, lane, A.Mfix + g * 32 + lane,
                                          S.Lfix(g * 32 + lane), iscale);
                }
            }
        } else {
            const int ch = chunk_size(total, nwarps, 32);
            for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch))
                sc_var_chunk<CPT, (D <= 8 ? 16 : 32)>(A, S, base, min(base + ch, total), t, cp, lane, s_w, s_x,
                                                      iscale);   // acc loads in flight: register budget
        }
        ++wc;
    }
    grid_barrier(A.barrier);
    stamp(A, ts_k);
    {   // syndrome phase
        const int total = G * cblk;
        const int sc = syn_chunk(total, nwarps);
        for (int base = claim(A.work + wc, lane, sc); base < total; base = claim(A.work + wc, lane, sc))
            sc_syncheck_chunk<D, CPT>(A, S, base, min(base + sc, total), t, cp, cblk, lane);
        ++wc;
    }
}

// Per-warp shared-memory carve-out of decode_scatter_kernel, in 32-bit words
// (one contiguous slice per warp, dynamic shared memory; measured against the
// per-array static layout it replaced: sweep-1 variable phase 0.219 ->
// 0.201 ms, cfg 2 kernel 1.375 -> 1.342 ms):
//   idx  check phases: row variable offsets [CH][SD]; sweep 1: Mfix table
//   w, x, m  [CH] staging words
//   raw  sweep-1 staging (regular column degree 6 or 9, check degree <= 16:
//        mismatch words + degrees + per-variable uniform degree) or, in
//        check phases, the lane's sweep-1 magnitude per degree
template <int D> struct ScatterSmem {
    static constexpr int CH = Chunk<D>::CH;
    static constexpr int MF = D <= 16 ? (D + 1) * 32 : 1;
    static constexpr int kSlice = CH * Chunk<D>::SD > MF ? CH * Chunk<D>::SD : MF;
    static constexpr int kCH = CH > 32 ? CH : 32;
    static constexpr int kV1 = D <= 16 ? 32 * 9 : 0;
    static constexpr int M1T = D <= 16 ? (D + 1) * 32 : 0;
    static constexpr int kRaw = (kV1 + kV1 / 4 + 8) > M1T ? (kV1 + kV1 / 4 + 8) + 1 : M1T + 1;
    static constexpr int kWarp = (kSlice + 3 * kCH + kRaw + 1) & ~1;
    static constexpr size_t bytes = (size_t)(kDecodeThreads / 32) * kWarp * 4;
};

// HOT = true: the hot instance (sweeps 1..kHotSweeps, clamp < sat).  When
// frames remain undecided after sweep kHotSweeps it stores its loop state in
// A.resume and exits; the full instance launched behind it (HOT = false,
// A.resume set) resumes there, or returns at once when the flag is clear.
// With A.resume == nullptr the full instance runs the whole decode.
template <int D, bool HOT>
__global__ void __launch_bounds__(kDecodeThreads, scatter_min_blocks<D>()) decode_scatter_kernel(const ScatterArgs A)
{
    const bool resumed = !HOT && A.resume;
    if (resumed && ld_cg(A.resume) == 0) return;   // the hot instance finished the decode
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthreads = gridDim.x * blockDim.x;
    const int nwarps = nthreads >> 5;
    const int gw = gtid >> 5;
    const int cblk = (A.C + 31) / 32;
    using SM = ScatterSmem<D>;
    extern __shared__ __align__(16) unsigned s_dyn[];   // SM::bytes, set by launch_scatter
    unsigned* s_warp = s_dyn + warp * SM::kWarp;
    int* s_idx = reinterpret_cast<int*>(s_warp);
    unsigned* s_w = s_warp + SM::kSlice;
    unsigned* s_x = s_w + SM::kCH;
    unsigned* s_m = s_x + SM::kCH;
    unsigned* s_v1m = s_m + SM::kCH;
    uint8_t* s_v1d = reinterpret_cast<uint8_t*>(s_v1m + SM::kV1);
    int* s_mf = s_idx;   // only used in the sweep-1 variable phase

    // fixed-point scale: |acc| <= Lmax + dv_max * clamp (+ rounding) < 2^30
    int ex;
    frexpf(ld_cg(A.Lmax) + (float)A.dv_max * A.clamp + 2.0f, &ex);
    int S = min(30 - ex, 40);
#if MBP_FIX_MAGIC
    {   // fixq's range: |message| * 2^S < 2^22
        int ec;
        frexpf(A.clamp, &ec);
        S = min(S, 22 - ec);
    }
#endif
    const float scale = ldexpf(1.0f, S), iscale = ldexpf(1.0f, -S);

    bool cpt = false;
    int tc = 0;
    int G = A.G;
    bool may_compact = A.Gb > 0;
    int ts_k = 0;
    int wc = 0;
    int t = 1;
    if (resumed) {
        t = ld_cg(A.resume + 1);
        cpt = ld_cg(A.resume + 2) != 0;
        G = ld_cg(A.resume + 3);
        tc = ld_cg(A.resume + 4);
        may_compact = ld_cg(A.resume + 5) != 0;
        wc = ld_cg(A.resume + 6);
        ts_k = ld_cg(A.resume + 7);
    } else {
        stamp(A, ts_k);

        // fixed-point prior and sweep-1 magnitudes per frame
        for (int f = gtid; f < A.G * 32; f += nthreads) {
            A.Lfix[f] = __float2int_rn(A.Lmag[f] * scale);
            for (int d = 0; d <= A.Dm; ++d)
                A.Mfix[(size_t)d * A.G * 32 + f] = __float2int_rn(A.Mtab[(size_t)d * A.G * 32 + f] * scale);
        }
        // iteration 0: the uncorrected key against all u*m syndromes
        // (_kernels.py:358-365); keeps the mismatch words for sweeps 1-3
        {
            const SL<false> S0{A, A.G};
            const int total = A.G * cblk;
            const int sc = syn_chunk(total, nwarps);
            for (int base = claim(A.work + wc, lane, sc); base < total; base = claim(A.work + wc, lane, sc))
                sc_syncheck_chunk<D, false>(A, S0, base, min(base + sc, total), 0, nullptr, cblk, lane);
            ++wc;
        }
    }

    int final_t = 0;
    bool top = !resumed;   // the resumed sweep's loop-top bookkeeping ran in the hot instance
    for (;; ++t) {
        if (top) {
            grid_barrier(A.barrier);
            stamp(A, ts_k);
            const int F = G * 32;
            int* cnt = cpt ? A.cnt_b : A.cnt;
            const int* cprev = cnt + ((t - 1) & 1) * F;
            for (int f = gtid; f < F; f += nthreads) {
                const int c = ld_cg(cprev + f);
                const int fr = cpt ? ld_cg(A.fid_b + f) : f;
                if (fr >= 0 && c == 0 && ld_cg(A.iters + fr) < 0) A.iters[fr] = t - 1;
                cnt[(t & 1) * F + f] = 0;
                if (may_compact) {
                    const unsigned msk = __ballot_sync(kFull, c != 0);
                    if (lane == 0) {
                        A.grp_cnt[f >> 5] = __popc(msk);
                        if (msk) {
                            atomicAdd(A.ctrl + 2 * t, __popc(msk));
                            atomicAdd(A.ctrl + 2 * t + 1, 1);
                        }
                    }
                }
            }
            if (ld_cg(A.any_bad + ((t - 1) & 1)) == 0 || t > A.max_it) {
                final_t = t - 1;
                break;
            }
            if (gtid == 0) A.any_bad[t & 1] = 0;
            if (HOT && t > kHotSweeps) {
                if (gtid == 0) {
                    A.resume[1] = t;
                    A.resume[2] = cpt;
                    A.resume[3] = G;
                    A.resume[4] = tc;
                    A.resume[5] = may_compact;
                    A.resume[6] = wc;
                    A.resume[7] = ts_k;
                    A.resume[0] = 1;
                }
                return;
            }
        }
        top = true;
        if (may_compact && t >= 2) {
            grid_barrier(A.barrier);
            const int nund = ld_cg(A.ctrl + 2 * t);
            const int gact = ld_cg(A.ctrl + 2 * t + 1);
            const int gn = (nund + 31) / 32;
            if (nund * 2 <= gact * 32 && gn < gact && gn <= A.Gb) {
                G = sc_compact(A, t, gw, nwarps, gtid, nthreads, lane);
                if (cmp_recomp(A, t)) {
                    sc_recomp_post1<D>(A, G, t, wc, lane, nwarps, s_w, s_v1m, s_v1d, s_mf, iscale);
                    grid_barrier(A.barrier);
                }
                cpt = true;
                tc = t;
                may_compact = false;
            }
        }
        if (cpt)
            sc_sweep<D, true, HOT>(A, G, t, wc, ts_k, lane, nwarps, s_idx, s_w, s_x, s_m, s_v1m, s_v1d, s_mf, t == tc,
                                   scale, iscale);
        else
            sc_sweep<D, false, HOT>(A, G, t, wc, ts_k, lane, nwarps, s_idx, s_w, s_x, s_m, s_v1m, s_v1d, s_mf, false,
                                    scale, iscale);
    }

    if (cpt) grid_barrier(A.barrier);
    const int* cfin = (cpt ? A.cnt_b : A.cnt) + (final_t & 1) * G * 32;
    for (int f = gtid; f < A.B; f += nthreads) {
        const int s = cpt ? ld_cg(A.newslot + f) : f;
        const int c = s >= 0 ? ld_cg(cfin + s) : 0;
        const int it = ld_cg(A.iters + f);
        const bool conv = it >= 0;
        A.out_conv[f] = conv ? 1 : 0;
        A.out_iters[f] = conv ? it : A.max_it;
        A.out_mism[f] = conv ? 0 : c;
    }
    if (cpt) scatter_back(A, gw, nwarps, lane);
    if (gtid == 0) A.sweeps_run[0] = final_t;
    stamp(A, ts_k);
}

// Per-frame setup: prior magnitude L = ln((1-e)/e) (init_priors,
// decoder.py:147-152), the sweep-1 message magnitude for every degree
// d <= Dm (the reference's sequential product of d-1 factors tanh(L/2),
// saturation and clamp, in fp64), and the batch maximum of L -- all stored
// in the kernel's log2 units (x log2 e).
static __global__ void scatter_setup_kernel(const double* __restrict__ e, int e_stride, int B, int F, int Dm,
                                     double clamp, float* __restrict__ Lmag, float* __restrict__ Mtab,
                                     float* __restrict__ Lmax)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    double L = 0.0;
    if (f < B) {
        const double ef = e[(long long)f * e_stride];
        L = log((1.0 - ef) / ef);
    }
    constexpr double kLog2e = 1.4426950408889634074;
    Lmag[f] = (float)(L * kLog2e);
    const double th = tanh(0.5 * L);
    double prod = 1.0;
    Mtab[f] = 0.0f;
    for (int d = 1; d <= Dm; ++d) {
        double r = prod >= 1.0 ? clamp : (prod <= -1.0 ? -clamp : 2.0 * atanh(prod));
        r = r > clamp ? clamp : r;
        Mtab[(size_t)d * F + f] = f < B ? (float)(r * kLog2e) : 0.0f;
        prod *= th;
    }
    if (f < B) atomicMax(reinterpret_cast<int*>(Lmax), __float_as_int((float)(L * kLog2e)));
}

}  // namespace mbp
