// decode.cuh -- the persistent cooperative MBP decode kernel (sm_100a).
//
// One launch runs the whole flooding decode of a batch (decode_loop,
// _kernels.py:323-379).  Per sweep:
//   check phase     Eq. 6 for every check of every active group (c2v_pass,
//                   _kernels.py:230-261); the variable-to-check message is
//                   formed on the fly in APP form v2c = clamp(post - c2v),
//                   exact because the reference's joint `total` IS the
//                   posterior sum (_kernels.py:276-279 vs 293-301);
//   variable phase  posterior (Eq. 2) + hard decision as 32-frame words
//                   (posterior_pass / hard_pass, _kernels.py:293-307);
//   syndrome phase  per-frame mismatch counts (mismatch_count,
//                   _kernels.py:310-320) that drive early termination;
// separated by grid barriers.  Layout: see kernels.cuh (lane = frame,
// groups of 32 frames, padded-ELL edge slots).
//
// Frame compaction: a group runs the sweeps of its slowest frame.  Once at
// most half of the lanes of the still-active groups carry an undecided
// frame, the active frames are repacked into dense groups in a second set of
// buffers (layout switch); a slot -> frame map routes the outputs.  Messages and
// decisions are moved bit for bit, so compaction never changes a result.
#pragma once

#include "kernels.cuh"

namespace mbp {

// ---------------------------------------------------------------------------
// arguments
//
// Internal edge numbering (padded ELL): edge k of stacked check j is slot
// j*Ds + k (Ds = max row degree).  A check's var ids chk_ell[j*Ds..] and its
// message lines are contiguous; slot order is monotone in the reference's
// edge order, so ascending var_edge lists and matrix boundaries
// (edge_off[l] = l*m*Ds) keep the reference's summation order.
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
    // batch, primary (original) layout
    int G;                             // groups of 32 frames
    int B;                             // frames
    Real* c2v;                         // [G][slots][32]
    Real* post;                        // [G][P][n][32], P = ISO ? u+1 : 1
    Real* v2c;                         // [G][slots][32] (damping only)
    const Real* Lmag;                  // [G*32] prior magnitude per frame
    const unsigned* noisy_w;           // [G][n]
    const unsigned* syn_w;             // [G][C]
    unsigned* hard_w;                  // [G][n]
    unsigned* hist_w;                  // [(T+1)][G][n] or null
    int* cnt;                          // [2][G*32] mismatch counts by sweep parity
    // compaction: secondary layout of capacity Gb groups (Gb == 0: disabled)
    int Gb;
    Real* c2v_b;
    Real* post_b;
    Real* v2c_b;
    Real* Lmag_b;
    unsigned* noisy_b;
    unsigned* syn_b;
    unsigned* hard_b;
    int* cnt_b;                        // [2][Gb*32]
    int* fid_b;                        // [Gb*32] compacted slot -> frame, -1 empty (preset -1)
    int* src_b;                        // [Gb*32] compacted slot -> original slot, -1 empty (preset -1)
    int* newslot;                      // [G*32] original slot -> compacted slot, -1 (preset -1)
    int* grp_cnt;                      // [G] undecided frames per group at the decision
    int* ctrl;                         // [2*(T+2)] per-sweep (undecided frames, active groups), zeroed
    // control
    int* any_bad;                      // [2]
    int* iters;                        // [G*32] per frame: first converged sweep, -1 unset
    unsigned* barrier;                 // [2]
    unsigned* work;                    // [3*(T+1)+2] dynamic work counters, zeroed per launch
    int* sweeps_run;                   // [2]: sweeps, compaction sweep (0 = none)
    unsigned long long* ts;            // phase timestamps (globaltimer ns) or null
    int ts_cap;
    // outputs (per frame)
    uint8_t* out_conv;
    int* out_iters;
    int* out_mism;
    // config
    int max_it;
    Real clamp;
    Real damping;
    float sat;
};

// The buffers of a layout, selected at compile time: CPT = false is the
// primary (original) layout, CPT = true the compacted one.  Pointers stay in
// the kernel's parameter (constant) bank; only the compacted group count is
// a register.  Primary-layout inputs are never written by the kernel, so they
// are read through the non-coherent path; compacted ones are written by the
// compaction step of the same launch and are read L2-coherent.
template <class Real, bool CPT>
struct L {
    const DecodeArgs<Real>& A;
    int G;
    __device__ __forceinline__ Real* c2v() const { return CPT ? A.c2v_b : A.c2v; }
    __device__ __forceinline__ Real* post() const { return CPT ? A.post_b : A.post; }
    __device__ __forceinline__ Real* v2c() const { return CPT ? A.v2c_b : A.v2c; }
    __device__ __forceinline__ unsigned* hard_w() const { return CPT ? A.hard_b : A.hard_w; }
    __device__ __forceinline__ int* cnt() const { return CPT ? A.cnt_b : A.cnt; }
    __device__ __forceinline__ Real Lmag(int s) const { return CPT ? ld_cg(A.Lmag_b + s) : ld_ro(A.Lmag + s); }
    __device__ __forceinline__ unsigned noisy(size_t w) const { return CPT ? ld_cg(A.noisy_b + w) : ld_ro(A.noisy_w + w); }
    __device__ __forceinline__ unsigned syn(size_t w) const { return CPT ? ld_cg(A.syn_b + w) : ld_ro(A.syn_w + w); }
    __device__ __forceinline__ int fid(int s) const { return CPT ? ld_cg(A.fid_b + s) : s; }
};

// ---------------------------------------------------------------------------
// check phase
// ---------------------------------------------------------------------------

// Check j of group g at sweep t; `act` = lanes (frames) still decoding.
// Reads post_{t-1}, c2v_{t-1}, writes c2v_t.  The row's variable ids, degree
// and syndrome word come from the warp's shared-memory stage of its chunk,
// so an item costs one memory round trip.  Branch-free over the D slots
// (D = the launch's degree bound): slots k >= d are predicated off.
template <class Real, int D, bool DAMP, bool ISO, bool CPT>
__device__ __forceinline__ void check_item(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int g, int j,
                                           int t, unsigned act, int lane, const int* srow, int d,
                                           unsigned synword, Real L, const Real* qbase)
{
    const bool live = (act >> lane) & 1u;
    const unsigned flip = (synword >> lane) & 1u;
    const int mat = ISO ? j / A.m : 0;
    Real* c2v_row = S.c2v() + ((size_t)g * A.slots + (size_t)j * A.Ds) * 32 + lane;
    // c2v_{t-1} comes from this lane's own row, except in the first sweep after
    // a compaction, when it is read in place from the frame's original lane
    const Real* q_row = qbase + (size_t)j * A.Ds * 32;
    Real* v2c_row = DAMP ? S.v2c() + ((size_t)g * A.slots + (size_t)j * A.Ds) * 32 + lane : nullptr;
    const Real* postg = S.post() + ((size_t)g * (ISO ? A.u + 1 : 1) + mat) * A.n * 32 + lane;

    Real x[D];
    if (t == 1) {
        // sweep 1 reads the UNCLAMPED prior (decode_loop init, _kernels.py:353-355)
        const size_t nw = (size_t)g * A.n;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const unsigned w = k < d ? S.noisy(nw + srow[k]) : 0u;
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
            q[k] = ld_cg_if(q_row + k * 32, pk);
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

// ---------------------------------------------------------------------------
// variable phase
// ---------------------------------------------------------------------------

// Regular column degree DV, NV variables per warp pass (independent load
// streams in flight): joint posterior prior + sum of every matrix's c2v in
// ascending edge order (posterior_pass, _kernels.py:293-301), hard decision
// post < 0 (ties -> 0) as a ballot (hard_pass).  Edge slots, noisy words and
// previous hard words come from the chunk's shared stage.
template <class Real, int DV, int NV, bool CPT>
__device__ __forceinline__ void var_items_regular(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int g,
                                                  int i0, int nv, int t, unsigned act, int lane,
                                                  const int* sedge, int sstride, const unsigned* snoisy,
                                                  const unsigned* sold, Real L)
{
    const bool live = (act >> lane) & 1u;
    const Real* c2vg = S.c2v() + (size_t)g * A.slots * 32 + lane;
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
        st_if(S.post() + w * 32 + lane, acc, live);
        const unsigned neg = __ballot_sync(kFull, acc < Real(0));
        if (lane == 0) {
            const unsigned hw = (neg & act) | (sold[v] & ~act);
            S.hard_w()[w] = hw;
            if (A.hist_w) A.hist_w[((size_t)t * A.G) * A.n + w] = hw;
        }
    }
}

// General degrees (CSR) and isolated-per-matrix mode: also the per-matrix
// totals v2c_pass uses in isolated mode (_kernels.py:276-279).
template <class Real, bool ISO, bool CPT>
__device__ __forceinline__ void var_item(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int g, int i, int t,
                                         unsigned act, int lane)
{
    const int p0 = A.dv ? i * A.dv : ld_ro(A.var_ptr + i);
    const int dv = A.dv ? A.dv : ld_ro(A.var_ptr + i + 1) - p0;
    const bool live = (act >> lane) & 1u;
    const size_t w = (size_t)g * A.n + i;
    const unsigned nwd = S.noisy(w);
    const unsigned old = lane == 0 ? ld_cg(S.hard_w() + w) : 0u;
    const Real L = S.Lmag(g * 32 + lane);
    const Real prior = ((nwd >> lane) & 1u) ? -L : L;
    const Real* c2vg = S.c2v() + (size_t)g * A.slots * 32 + lane;
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
        st_if(S.post() + w * 32 + lane, acc, live);
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
                    st_if(S.post() + (((size_t)g * P + l) * A.n + i) * 32 + lane, part, live);
                    part = prior;
                    ++l;
                }
                const Real cv = ld_cg_if(c2vg + (size_t)e * 32, live);
                acc += cv;
                part += cv;
            }
        }
        for (; l < A.u; ++l) {
            st_if(S.post() + (((size_t)g * P + l) * A.n + i) * 32 + lane, part, live);
            part = prior;
        }
        st_if(S.post() + (((size_t)g * P + A.u) * A.n + i) * 32 + lane, acc, live);
    }
    const unsigned neg = __ballot_sync(kFull, acc < Real(0));
    if (lane == 0) {
        const unsigned hw = (neg & act) | (old & ~act);
        S.hard_w()[w] = hw;
        if (A.hist_w) A.hist_w[((size_t)t * A.G) * A.n + w] = hw;
    }
}

__device__ __forceinline__ unsigned group_mask(const int* cprev, int g, int lane)
{
    return __ballot_sync(kFull, ld_cg(cprev + g * 32 + lane) != 0);
}

// ---------------------------------------------------------------------------
// syndrome phase: 32 consecutive checks (lane = check) of group g.  Mismatch
// words (bit f = frame f) become per-frame counts via 32 ballots, added to
// cnt[t&1].
// ---------------------------------------------------------------------------
template <class Real, bool CPT>
__device__ __forceinline__ int syncheck_item(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int g, int blk,
                                             int t, unsigned act, int lane)
{
    const int j = blk * 32 + lane;
    unsigned mism = 0;
    if (j < A.C) {
        const unsigned* hw = S.hard_w() + (size_t)g * A.n;
        const int d = ld_ro(A.deg + j);
        const int* row = A.chk_ell + j * A.Ds;
        unsigned par = 0;
        for (int k = 0; k < d; ++k) par ^= ld_cg(hw + ld_ro(row + k));
        mism = (par ^ S.syn((size_t)g * A.C + j)) & act;
    }
    // lane f: popcount of bit f over the 32 checks (bit transpose + popc)
    return __any_sync(kFull, mism != 0) ? __popc(warp_transpose32(mism, lane)) : 0;
}

// A claimed run of syndrome items; per-frame counts accumulate in registers
// and are flushed once per group (per-item atomics on a group's 32 counters
// all hit one L2 line and serialise).
template <class Real, bool CPT>
__device__ __forceinline__ void syncheck_run(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int base, int end,
                                             int t, const int* cprev, int cblk, int lane)
{
    int g = base / cblk;
    unsigned act = cprev ? group_mask(cprev, g, lane) : kFull;
    int c = 0;
    bool bad = false;
    for (int item = base; item < end; ++item) {
        const int gi = item / cblk;
        if (gi != g) {
            if (c) atomicAdd(S.cnt() + (t & 1) * S.G * 32 + g * 32 + lane, c);
            bad |= c != 0;
            c = 0;
            g = gi;
            act = cprev ? group_mask(cprev, g, lane) : kFull;
        }
        if (act) c += syncheck_item<Real, CPT>(A, S, g, item - g * cblk, t, act, lane);
    }
    if (c) atomicAdd(S.cnt() + (t & 1) * S.G * 32 + g * 32 + lane, c);
    bad |= c != 0;
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(A.any_bad + (t & 1), 1);
}

// ---------------------------------------------------------------------------
// scheduling helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// compaction stamps live in the last 4 timestamp slots
template <class Args>
__device__ __forceinline__ void stamp_compact(const Args& A, int k)
{
    if (A.ts && blockIdx.x == 0 && threadIdx.x == 0 && A.ts_cap >= 8) A.ts[A.ts_cap - 4 + k] = globaltimer();
}

template <class Args>
__device__ __forceinline__ void stamp(const Args& A, int& k)
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



// one claimed chunk of the check phase: items [base, end) of the G*C space
// input row base of c2v_{t-1} for lane `lane` of group g (see check_item)
template <class Real, bool CPT>
__device__ __forceinline__ const Real* c2v_in_base(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int g, int lane,
                                                   bool first_after_compaction)
{
    if (CPT && first_after_compaction) {
        const int s = ld_cg(A.src_b + g * 32 + lane);
        if (s >= 0) return A.c2v + (size_t)(s >> 5) * A.slots * 32 + (s & 31);
    }
    return S.c2v() + (size_t)g * A.slots * 32 + lane;
}

template <class Real, int D, bool DAMP, bool ISO, bool CPT>
__device__ __forceinline__ void check_chunk(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int base, int end,
                                            int t, const int* cprev, int lane, int* s_idx, unsigned* s_w,
                                            int* s_d, bool first)
{
    constexpr int SD = Chunk<D>::SD;
    const int rows = end - base;
    if (lane < rows) {
        const int item = base + lane;
        const int j = item % A.C;
        const int d = ld_ro(A.deg + j);
        s_d[lane] = d;
        s_w[lane] = S.syn(item);  // syn_w index == item (g*C + j)
        const int* row = A.chk_ell + j * A.Ds;
#pragma unroll
        for (int k = 0; k < D; ++k)
            if (k < d) s_idx[lane * SD + k] = ld_ro(row + k);
    }
    __syncwarp();
    int g = base / A.C;
    int j = base - g * A.C;
    unsigned act = group_mask(cprev, g, lane);
    Real L = S.Lmag(g * 32 + lane);
    const Real* qb = c2v_in_base<Real, CPT>(A, S, g, lane, first);
    for (int r = 0; r < rows; ++r) {
        if (act)
            check_item<Real, D, DAMP, ISO, CPT>(A, S, g, j, t, act, lane, s_idx + r * SD, s_d[r], s_w[r], L, qb);
        if (++j == A.C && r + 1 < rows) {
            j = 0;
            ++g;
            act = group_mask(cprev, g, lane);
            L = S.Lmag(g * 32 + lane);
            qb = c2v_in_base<Real, CPT>(A, S, g, lane, first);
        }
    }
    __syncwarp();
}

// one claimed chunk of the variable phase (regular column degree DV)
template <class Real, int DV, bool CPT>
__device__ __forceinline__ void var_chunk_regular(const DecodeArgs<Real>& A, const L<Real, CPT>& S, int base,
                                                  int end, int t, const int* cprev, int lane, int* s_idx,
                                                  unsigned* s_w, unsigned* s_old)
{
    constexpr int SV = DV | 1;
    const int rows = end - base;
    if (lane < rows) {
        const int item = base + lane;            // == g*n + i
        const int i = item % A.n;
        s_w[lane] = S.noisy(item);
        s_old[lane] = ld_cg(S.hard_w() + item);
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
        const Real L = S.Lmag(g * 32 + lane);
        if (act) {
            for (int k = 0; k < span; k += 2)
                var_items_regular<Real, DV, 2, CPT>(A, S, g, i + k, min(2, span - k), t, act, lane,
                                               s_idx + (r + k) * SV, SV, s_w + r + k, s_old + r + k, L);
        }
        r += span;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// compaction (all threads of the grid; contains grid barriers)
// ---------------------------------------------------------------------------

// Move lane values of an interleaved [G][X][32] array into the compacted
// layout: dst[g'][x][l'] = src[s/32][x][s%32], s = src_b[g'*32 + l'].
// The source reads are scattered (one sector per lane), so each warp item
// keeps XU independent loads in flight.  They go through L1 (ld.ca): lanes
// of one source group share sectors, and no source array changes during
// the compaction (L1 is invalidated by the __threadfence of every grid
// barrier, so no stale line survives from an earlier phase).
template <class T>
__device__ __forceinline__ void move_lanes(const T* src, T* dst, long long X, int Gn, const int* src_b,
                                           int gw, int nw, int lane)
{
    constexpr int XU = 32;
    const long long xchunks = (X + XU - 1) / XU;
    for (long long it = gw; it < (long long)Gn * xchunks; it += nw) {
        const int g2 = (int)(it / xchunks);
        const long long x0 = (it - (long long)g2 * xchunks) * XU;
        const int s = ld_cg(src_b + g2 * 32 + lane);
        const T* sp = src + (s >= 0 ? ((size_t)(s >> 5) * X * 32 + (s & 31)) : 0) + x0 * 32;
        T* dp = dst + ((size_t)g2 * X + x0) * 32 + lane;
        T v[XU];
#pragma unroll
        for (int k = 0; k < XU; ++k) v[k] = (s >= 0 && x0 + k < X) ? __ldca(sp + k * 32) : T(0);
#pragma unroll
        for (int k = 0; k < XU; ++k)
            if (x0 + k < X) dp[k * 32] = v[k];
    }
}

// Same for 32-frame bit words [G][X]: dst[g'][x] bit l' = src[s/32][x] bit s%32.
__device__ __forceinline__ void move_bits(const unsigned* src, unsigned* dst, long long X, int Gn, const int* src_b,
                                          int gw, int nw, int lane)
{
    constexpr int XU = 16;
    const long long xchunks = (X + XU - 1) / XU;
    for (long long it = gw; it < (long long)Gn * xchunks; it += nw) {
        const int g2 = (int)(it / xchunks);
        const long long x0 = (it - (long long)g2 * xchunks) * XU;
        const int s = ld_cg(src_b + g2 * 32 + lane);
        const unsigned* sp = src + (s >= 0 ? (size_t)(s >> 5) * X : 0) + x0;
        unsigned w[XU];
#pragma unroll
        for (int k = 0; k < XU; ++k) w[k] = (s >= 0 && x0 + k < X) ? __ldca(sp + k) : 0u;
        unsigned mine = 0;
#pragma unroll
        for (int k = 0; k < XU; ++k) {
            const unsigned b = __ballot_sync(kFull, (w[k] >> (s & 31)) & 1u & (s >= 0));
            if (lane == k) mine = b;
        }
        if (lane < XU && x0 + lane < X) dst[(size_t)g2 * X + x0 + lane] = mine;
    }
}

// Repack the undecided frames of the primary layout (counts per group in
// grp_cnt, total in ctrl[2t]) into ceil(total/32) dense groups of the
// secondary buffers.  Returns the compacted group count.
template <class Real, bool DAMP, bool ISO>
__device__ __forceinline__ int compact(const DecodeArgs<Real>& A, int t, int gw, int nw, int gtid, int nthreads,
                                       int lane)
{
    const int F = A.G * 32;
    const int* cprev = A.cnt + ((t - 1) & 1) * F;
    stamp_compact(A, 0);
    // 1. exclusive scan of the per-group undecided counts (block 0), slot maps
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
    for (int g = gw; g < A.G; g += nw) {   // warp per original group
        const bool und = ld_cg(cprev + g * 32 + lane) != 0;
        const unsigned m = __ballot_sync(kFull, und);
        if (und) {
            const int s2 = ld_cg(A.grp_cnt + g) + __popc(m & ((1u << lane) - 1u));
            A.newslot[g * 32 + lane] = s2;
            A.src_b[s2] = g * 32 + lane;
            A.fid_b[s2] = g * 32 + lane;   // before compaction slot == frame
        }
    }
    grid_barrier(A.barrier);
    stamp_compact(A, 1);
    const int nund = ld_cg(A.ctrl + 2 * t);
    const int Gn = (nund + 31) / 32;
    const int Fb = Gn * 32;   // parity stride of the compacted counts
    // 2. move the per-frame arrays into the compacted layout (c2v excepted:
    //    the next check phase reads it in place, see check_item)
    move_lanes<Real>(A.post, A.post_b, (long long)(ISO ? A.u + 1 : 1) * A.n, Gn, A.src_b, gw, nw, lane);
    if (DAMP) move_lanes<Real>(A.v2c, A.v2c_b, A.slots, Gn, A.src_b, gw, nw, lane);
    move_bits(A.noisy_w, A.noisy_b, A.n, Gn, A.src_b, gw, nw, lane);
    move_bits(A.hard_w, A.hard_b, A.n, Gn, A.src_b, gw, nw, lane);
    move_bits(A.syn_w, A.syn_b, A.C, Gn, A.src_b, gw, nw, lane);
    for (int s2 = gtid; s2 < Fb; s2 += nthreads) {
        const int s = ld_cg(A.src_b + s2);
        A.Lmag_b[s2] = s >= 0 ? A.Lmag[s] : Real(0);
        A.cnt_b[((t - 1) & 1) * Fb + s2] = s >= 0 ? ld_cg(cprev + s) : 0;
        A.cnt_b[(t & 1) * Fb + s2] = 0;
    }
    stamp_compact(A, 2);
    grid_barrier(A.barrier);
    stamp_compact(A, 3);
    if (gtid == 0) A.sweeps_run[1] = t;
    return Gn;
}

// After a compacted decode: final hard words of the frames that moved go back
// into the primary hard_w (original layout) for the row transpose.  Warp item
// = 32 consecutive words of one original group (lane = word); the group's
// moved frames (a few) are walked one by one with coalesced word loads.
template <class Args>
__device__ __forceinline__ void scatter_back(const Args& A, int gw, int nw, int lane)
{
    const int xchunks = (A.n + 31) / 32;
    for (long long it = gw; it < (long long)A.G * xchunks; it += nw) {
        const int g = (int)(it / xchunks);
        const int x = (int)(it - (long long)g * xchunks) * 32 + lane;
        const int s2l = ld_cg(A.newslot + g * 32 + lane);
        unsigned moved = __ballot_sync(kFull, s2l >= 0);
        if (!moved) continue;
        const size_t o = (size_t)g * A.n + x;
        unsigned w = x < A.n ? ld_cg(A.hard_w + o) : 0u;
        while (moved) {
            const int l0 = __ffs(moved) - 1;
            moved &= moved - 1;
            const int s2 = __shfl_sync(kFull, s2l, l0);
            const unsigned src = x < A.n ? ld_cg(A.hard_b + (size_t)(s2 >> 5) * A.n + x) : 0u;
            w = (w & ~(1u << l0)) | (((src >> (s2 & 31)) & 1u) << l0);
        }
        if (x < A.n) A.hard_w[o] = w;
    }
}

// ---------------------------------------------------------------------------
// one sweep's three phases in a given layout (called between the sweep's
// leading barrier and the next sweep's)
// ---------------------------------------------------------------------------
template <class Real, int D, bool DAMP, bool ISO, bool CPT>
__device__ __forceinline__ void sweep_phases(const DecodeArgs<Real>& A, int G, int t, int& wc, int& ts_k, int lane,
                                             int nwarps, int* s_idx, unsigned* s_w, unsigned* s_x, bool first)
{
    const L<Real, CPT> S{A, G};
    constexpr int CH = Chunk<D>::CH;
    const int cblk = (A.C + 31) / 32;
    const int* cp = S.cnt() + ((t - 1) & 1) * G * 32;
    {   // check phase
        const int total = G * A.C;
        const int ch = chunk_size(total, nwarps, CH);
        for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch))
            check_chunk<Real, D, DAMP, ISO, CPT>(A, S, base, min(base + ch, total), t, cp, lane,
                                                 s_idx, s_w, reinterpret_cast<int*>(s_x), first);
        ++wc;
    }
    grid_barrier(A.barrier);
    stamp(A, ts_k);
    {   // variable phase
        const int total = G * A.n;
        const int ch = chunk_size(total, nwarps, CH);
        for (int base = claim(A.work + wc, lane, ch); base < total; base = claim(A.work + wc, lane, ch)) {
            const int end = min(base + ch, total);
            if (!ISO && A.dv == 6) {
                var_chunk_regular<Real, 6, CPT>(A, S, base, end, t, cp, lane, s_idx, s_w, s_x);
            } else if (!ISO && A.dv == 9) {
                var_chunk_regular<Real, 9, CPT>(A, S, base, end, t, cp, lane, s_idx, s_w, s_x);
            } else {
                int item = base;
                while (item < end) {
                    const int g = item / A.n;
                    const int i = item - g * A.n;
                    const unsigned act = group_mask(cp, g, lane);
                    const int span = min(end - item, A.n - i);
                    if (act)
                        for (int k = 0; k < span; ++k) var_item<Real, ISO, CPT>(A, S, g, i + k, t, act, lane);
                    item += span;
                }
            }
        }
        ++wc;
    }
    grid_barrier(A.barrier);
    stamp(A, ts_k);
    {   // syndrome phase
        const int total = G * cblk;
        const int sc = min(64, max(8, (total + nwarps - 1) / nwarps));   // ~one claim per warp
        for (int base = claim(A.work + wc, lane, sc); base < total; base = claim(A.work + wc, lane, sc))
            syncheck_run<Real, CPT>(A, S, base, min(base + sc, total), t, cp, cblk, lane);
        ++wc;
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
#ifndef MBP_FP32_MIN_BLOCKS
#define MBP_FP32_MIN_BLOCKS 4
#endif
template <class Real, int D>
constexpr int decode_min_blocks() { return (sizeof(Real) == 4 && D <= 16) ? MBP_FP32_MIN_BLOCKS : 2; }

template <class Real, int D, bool DAMP, bool ISO>
__global__ void __launch_bounds__(kDecodeThreads, decode_min_blocks<Real, D>())
decode_kernel(const DecodeArgs<Real> A)
{
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthreads = gridDim.x * blockDim.x;
    const int nwarps = nthreads >> 5;
    const int gw = gtid >> 5;
    const int cblk = (A.C + 31) / 32;
    constexpr int CH = Chunk<D>::CH;
    constexpr int SLICE = CH * (Chunk<D>::SD > 9 ? Chunk<D>::SD : 9);   // ints per warp (check or var rows)
    __shared__ int s_idx_all[kDecodeThreads / 32][SLICE];
    __shared__ unsigned s_w_all[kDecodeThreads / 32][CH];
    __shared__ unsigned s_x_all[kDecodeThreads / 32][CH];
    int* s_idx = s_idx_all[warp];
    unsigned* s_w = s_w_all[warp];
    unsigned* s_x = s_x_all[warp];

    bool cpt = false;          // compacted layout active
    int tc = 0;                // sweep at whose start the compaction happened
    int G = A.G;               // groups of the current layout
    bool may_compact = A.Gb > 0;

    int ts_k = 0;
    int wc = 0;  // next work counter
    stamp(A, ts_k);

    // iteration 0: the uncorrected key against all u*m syndromes (_kernels.py:358-365)
    {
        const L<Real, false> S0{A, A.G};
        const int total = A.G * cblk;
        const int sc = min(64, max(8, (total + nwarps - 1) / nwarps));
        for (int base = claim(A.work + wc, lane, sc); base < total; base = claim(A.work + wc, lane, sc))
            syncheck_run<Real, false>(A, S0, base, min(base + sc, total), 0, nullptr, cblk, lane);
        ++wc;
    }

    int t = 1;
    int final_t = 0;
    for (;; ++t) {
        grid_barrier(A.barrier);
        stamp(A, ts_k);
        const int F = G * 32;
        int* cnt = cpt ? A.cnt_b : A.cnt;
        const int* cprev = cnt + ((t - 1) & 1) * F;
        // frames whose sweep t-1 decision satisfied every syndrome stop here;
        // warps own whole groups, so undecided frames / active groups are
        // counted for the compaction decision on the way
        for (int f = gtid; f < F; f += nthreads) {
            const int c = ld_cg(cprev + f);
            const int fr = cpt ? ld_cg(A.fid_b + f) : f;
            if (fr >= 0 && c == 0 && ld_cg(A.iters + fr) < 0) A.iters[fr] = t - 1;
            cnt[(t & 1) * F + f] = 0;
            if (may_compact) {
                const unsigned m = __ballot_sync(kFull, c != 0);
                if (lane == 0) {
                    A.grp_cnt[f >> 5] = __popc(m);
                    if (m) {
                        atomicAdd(A.ctrl + 2 * t, __popc(m));
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
        if (may_compact) {
            grid_barrier(A.barrier);
            const int nund = ld_cg(A.ctrl + 2 * t);
            const int gact = ld_cg(A.ctrl + 2 * t + 1);
            const int gn = (nund + 31) / 32;
            // compact when at most half of the computed lanes are undecided and
            // at least one whole group of work disappears
            if (t >= 2 && nund * 2 <= gact * 32 && gn < gact && gn <= A.Gb) {
                G = compact<Real, DAMP, ISO>(A, t, gw, nwarps, gtid, nthreads, lane);
                cpt = true;
                tc = t;
                may_compact = false;
            }
        }
        if (cpt)
            sweep_phases<Real, D, DAMP, ISO, true>(A, G, t, wc, ts_k, lane, nwarps, s_idx, s_w, s_x, t == tc);
        else
            sweep_phases<Real, D, DAMP, ISO, false>(A, G, t, wc, ts_k, lane, nwarps, s_idx, s_w, s_x, false);
    }

    // per-frame results (DecodeResult fields, decoder.py:246-274).  After a
    // compaction the last bookkeeping wrote iters[] through the slot map, i.e.
    // from other threads than the ones reading it here: barrier first.
    if (cpt) grid_barrier(A.barrier);
    const int* cfin = (cpt ? A.cnt_b : A.cnt) + (final_t & 1) * G * 32;
    for (int f = gtid; f < A.B; f += nthreads) {
        // iters[f] / newslot[f] may have been written by another SM: read via L2
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

}  // namespace mbp
