// peg_gpu.cu -- exact progressive edge growth with the BFS on the GPU.
//
// Restates the reference's _kernels.peg_build (pkg/src/mmrecon/_kernels.py:
// 57-161) so that a seed gives the SAME matrix as peg.cpp (the sequential
// host restatement) and the reference: per new edge of variable v, a BFS
// over the current graph; the candidate scan runs over the unreached checks
// in ascending index when some are unreachable, else over the deepest BFS
// level in discovery order; the lowest degree wins and exact ties are broken
// by the xorshift64* reservoir stream.
//
// What is parallel and what is not:
//  * the BFS (O(E) per edge, ~10^13 steps over a 2^20 code) runs level-
//    synchronously on the whole GPU.  The reference's discovery order -- a
//    frontier walked in order, each node's adjacency in insertion order,
//    first sighting wins -- is the lexicographic minimum of (frontier
//    position, adjacency slot) over a node's discoverers: an atomicMin per
//    node, then an order-preserving compaction of the discoverers;
//  * the candidate scan is summarised on the GPU: dmin (lowest candidate
//    degree), p0 (its first position), T_pre (ties of the running minimum
//    before p0 -- draws whose outcome is overwritten at p0) and K* (degree-
//    dmin candidates after p0);
//  * the tie-break stream is inherently sequential (xorshift64* has no jump
//    ahead), so the host advances it: T_pre steps, then K* draws with
//    divisibility tests; the index of the last successful draw selects the
//    winner, which the next launch attaches before its own BFS.
// One cooperative launch per edge; the host waits for its 48-byte summary.
#include "../../include/mbp.h"
#include "kernels.cuh"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace mbp {
int set_error(int code, const char* msg);
}

namespace {

using mbp::grid_barrier;
using mbp::ld_cg;

constexpr int KV = 4;          // column-degree bound (slots per variable)
constexpr int KC = 16;         // check adjacency capacity (PEG keeps rows near the mean degree)
constexpr int PB = 512;        // threads per block
constexpr int INF = 1 << 30;
constexpr int ND = KC + 1;     // candidate degrees 0..KC
constexpr long long kSmallLevel = 8192;   // slots block 0 expands alone
constexpr int kMaxHalfLevels = (1 << 18) - 2;   // BFS depth bound of the key format

struct PegSummary {
    int mode;                  // 0: unreached checks in index order, 1: deepest level in BFS order
    int count;                 // length of the scanned sequence (m or the level size)
    int dmin;                  // lowest candidate degree (INF: no candidate)
    int p0;                    // first position of dmin
    unsigned long long t_pre;  // running-minimum ties before p0
    unsigned long long kstar;  // degree-dmin candidates after p0
    int winner;                // check attached by the last prologue (diagnostics)
    int overflow;              // a check exceeded KC
};

struct PegArgs {
    int n, m;
    int* vn_adj;               // [n][KV]
    int* vn_deg;               // [n]
    int* cn_adj;               // [m][KC]
    int* cn_deg;               // [m]
    int* vis_c;                // [m] token of the BFS that reached the check
    int* vis_v;                // [n]
    unsigned long long* key_c; // [m] (~token << 32 | discovery slot)
    unsigned long long* key_v; // [n]
    int* lvl;                  // current check level: block regions (see Level)
    int* fr;                   // current variable frontier: block regions
    int* lvl_cnt;              // [grid] discoverers per block region
    int* fr_cnt;               // [grid]
    long long* lvl_seg;        // region stride of lvl
    long long* fr_seg;         // region stride of fr
    int* blk_k;                // [grid] per-block dmin counts after p0 (kept for the next attach)
    int* blk_min;              // [grid] per-block candidate minimum (summary)
    int* st_cnt;               // [grid][ND] candidates per degree (summary)
    int* st_first;             // [grid][ND] first position per degree (summary)
    int* bfs;                  // [8] BFS state handed from block 0 to the grid
    unsigned* bar;             // grid barrier
    PegSummary* sum;
};

// Discovery key of slot `slot` in half-level `hl` of BFS `token`: the high
// word decreases with every (token, half-level), so a stale key from any
// earlier expansion loses the atomicMin, and a key can only match slots of
// the expansion that wrote it (slot numbers restart every half-level).
__device__ __forceinline__ unsigned long long mk(int token, int hl, long long slot)
{
    // [40 bits: ~(token << 18 | hl)] [24 bits: slot]; token < 2^22, hl < 2^18,
    // slot < 2^24 (an expansion has at most max(4n, 16m) slots)
    const unsigned long long hi = ~(((unsigned long long)token << 18) | (unsigned long long)hl) & ((1ull << 40) - 1);
    return (hi << 24) | (unsigned long long)slot;
}

// block-wide exclusive sum of one int per thread; returns the block total in *tot
__device__ __forceinline__ int block_excl_sum(int x, int* sh, int* tot)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int s = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
    }
    if (lane == 31) sh[w] = s;
    __syncthreads();
    if (w == 0) {
        int v = lane < PB / 32 ? sh[lane] : 0;
        int t = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        sh[32 + lane] = t - v;
        if (lane == 31) sh[64] = t;
    }
    __syncthreads();
    const int r = sh[32 + w] + s - x;
    *tot = sh[64];
    __syncthreads();
    return r;
}

// block-wide exclusive prefix minimum (identity INF); returns the block minimum in *bmin
__device__ __forceinline__ int block_excl_min(int x, int* sh, int* bmin)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int s = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s = min(s, y);
    }
    int ex = __shfl_up_sync(0xffffffffu, s, 1);
    if (lane == 0) ex = INF;
    if (lane == 31) sh[w] = s;
    __syncthreads();
    if (w == 0) {
        int v = lane < PB / 32 ? sh[lane] : INF;
        int t = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t = min(t, y);
        }
        int e2 = __shfl_up_sync(0xffffffffu, t, 1);
        if (lane == 0) e2 = INF;
        sh[32 + lane] = e2;
        if (lane == 31) sh[64] = t;
    }
    __syncthreads();
    const int r = min(sh[32 + w], ex);
    *bmin = sh[64];
    __syncthreads();
    return r;
}

// A BFS level as the grid leaves it: block b's discoverers, in order, at
// buf[b * seg ...], cnt[b] of them; the level's global order is block-major.
// pre[] (shared, grid+1 entries) holds the prefix counts.  Callers walk a
// level in tiles of consecutive positions: tile() finds the tile's first
// region once (binary search, one thread), at() steps forward from it.
struct Level {
    const int* buf;
    long long seg;
    const int* pre;   // shared
    int* hint;        // shared: region of the current tile's first position
    int total;
    __device__ __forceinline__ void tile(long long q0) const   // all threads; ends with __syncthreads
    {
        if (threadIdx.x == 0) {
            int lo = 0, hi = gridDim.x;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (pre[mid] <= q0) lo = mid; else hi = mid;
            }
            *hint = lo;
        }
        __syncthreads();
    }
    __device__ __forceinline__ int at(long long q) const
    {
        int r = *hint;
        while (r + 1 < (int)gridDim.x && pre[r + 1] <= q) ++r;
        return ld_cg(buf + (long long)r * seg + (q - pre[r]));
    }
};

// load a level descriptor's prefix table into shared memory (all threads)
__device__ __forceinline__ int load_prefix(const int* cnt, int* pre, int* sh)
{
    const int x = threadIdx.x < (int)gridDim.x ? ld_cg(cnt + threadIdx.x) : 0;
    int tot;
    const int e = block_excl_sum(x, sh, &tot);
    if (threadIdx.x < (int)gridDim.x) pre[threadIdx.x] = e;
    if (threadIdx.x == 0) pre[gridDim.x] = tot;
    __syncthreads();
    return tot;
}

// Attach check c to variable v (one thread).
__device__ __forceinline__ void attach(const PegArgs& A, int c, int v)
{
    const int d = A.cn_deg[c];
    if (d >= KC) {
        A.sum->overflow = 1;
        return;
    }
    A.cn_adj[(size_t)c * KC + d] = v;
    A.cn_deg[c] = d + 1;
    A.vn_adj[(size_t)v * KV + A.vn_deg[v]++] = c;
    A.sum->winner = c;
}

// One expansion of the BFS: the slots i = q * K + k of level `from` (q its
// position, k < K an adjacency slot) discover the unvisited nodes they point
// to; the first slot in order wins (atomicMin of the key), as in the
// reference's sequential walk.  Blocks own contiguous slot segments and
// write their discoverers, in slot order, to out[b * seg ...]; out_cnt[b]
// gets the count.  `grid_mode` false: block 0 alone (small levels).
template <class Nbr>
__device__ __forceinline__ void expand(const PegArgs& A, int token, int hl, const Level& from, int K, Nbr nbr,
                                       unsigned long long* key, int* vis, int* out, int* out_cnt,
                                       long long* out_seg, bool grid_mode, int* sh)
{
    const long long items = (long long)from.total * K;
    const int nb = grid_mode ? gridDim.x : 1;
    const int bid = grid_mode ? blockIdx.x : 0;
    const long long seg = (items + nb - 1) / nb;
    const long long s0 = min(items, (long long)bid * seg), s1 = min(items, s0 + seg);
    for (long long c0 = s0; c0 < s1; c0 += PB) {
        from.tile(c0 / K);
        const long long i = c0 + threadIdx.x;
        if (i < s1) {
            const int x = nbr(from.at(i / K), (int)(i % K));
            if (x >= 0 && ld_cg(vis + x) != token) atomicMin(key + x, mk(token, hl, i));
        }
        __syncthreads();
    }
    if (grid_mode) grid_barrier(A.bar); else __syncthreads();
    int pos = 0;
    for (long long c0 = s0; c0 < s1; c0 += PB) {
        from.tile(c0 / K);
        const long long i = c0 + threadIdx.x;
        int x = -1;
        const bool d = i < s1 && (x = nbr(from.at(i / K), (int)(i % K))) >= 0 && ld_cg(key + x) == mk(token, hl, i);
        int tot;
        const int r = block_excl_sum(d ? 1 : 0, sh, &tot);
        if (d) {
            out[(long long)bid * seg + pos + r] = x;
            vis[x] = token;
        }
        pos += tot;
    }
    if (threadIdx.x == 0) out_cnt[bid] = pos;
    if (!grid_mode) {
        for (int b = 1 + threadIdx.x; b < (int)gridDim.x; b += PB) out_cnt[b] = 0;
    }
    if (bid == 0 && threadIdx.x == 0) *out_seg = seg;
    if (grid_mode) grid_barrier(A.bar); else __syncthreads();
}

// A level of at most 32 slots on warp 0 alone (the long, thin BFSs of a
// graph near its percolation point): lane = slot, the first lane holding a
// node discovers it (__match_any_sync), ballots keep slot order.  The level
// is read from and written to region 0 of the global level arrays, so block
// and grid expansions can follow.  All threads call it; returns the count.
template <class Nbr>
__device__ __forceinline__ int expand_warp(int token, const int* from, int items, int K, Nbr nbr, int* vis,
                                           int* out, int* out_cnt, long long* out_seg, int* s_cnt)
{
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int x = -1;
        if (lane < items) {
            x = nbr(ld_cg(from + lane / K), lane % K);
            if (x >= 0 && ld_cg(vis + x) == token) x = -1;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, x >= 0 ? x : -1 - lane);
        const bool win = x >= 0 && lane == __ffs(peers) - 1;
        const unsigned wins = __ballot_sync(0xffffffffu, win);
        if (win) {
            out[__popc(wins & ((1u << lane) - 1u))] = x;
            vis[x] = token;
        }
        if (lane == 0) {
            *out_cnt = __popc(wins);
            *out_seg = items;
            *s_cnt = __popc(wins);
        }
    }
    __syncthreads();
    return *s_cnt;
}

// One edge, one cooperative launch:
//  1. block 0 attaches the previous edge's winner (it owns the candidate
//     sequence the previous summary left) and runs the BFS from v while its
//     levels are small (block barriers only);
//  2. the whole grid takes over for the large levels (two grid barriers per
//     expansion);
//  3. the candidate-scan summary: per-block degree histograms and first
//     positions, one grid barrier, then dmin, p0, K* and the running-minimum
//     ties before p0.
__global__ void __launch_bounds__(PB) peg_step_kernel(PegArgs A, int v, int token, int attach_v,
                                                      unsigned long long attach_j, int do_bfs, int kc)
{
    __shared__ int sh[72];
    __shared__ int s_i[2 * ND + 4];
    __shared__ int s_pre[PB + 1];
    __shared__ int s_hint;
    const int m = A.m;
    Level F{A.fr, 0, s_pre, &s_hint, 0}, L{A.lvl, 0, s_pre, &s_hint, 0};
    auto nbr_v2c = [&](int w, int k) {
        return k < ld_cg(A.vn_deg + w) ? ld_cg(A.vn_adj + (size_t)w * KV + k) : -1;
    };
    auto nbr_c2v = [&](int c, int k) {
        return k < ld_cg(A.cn_deg + c) ? ld_cg(A.cn_adj + (size_t)c * KC + k) : -1;
    };

    if (blockIdx.x == 0) {
        // ---- 1a. attach the previous edge's winner ---------------------------
        if (attach_v >= 0) {
            const PegSummary S = *A.sum;
            if (S.mode == 1) {
                L.seg = ld_cg(A.lvl_seg);
                L.total = load_prefix(A.lvl_cnt, s_pre, sh);
            }
            if (attach_j == 0) {
                if (S.mode == 1) L.tile(S.p0);
                if (threadIdx.x == 0) attach(A, S.mode == 0 ? S.p0 : L.at(S.p0), attach_v);
            } else {
                // owner segment of the attach_j-th degree-dmin candidate after p0
                const int cnt = threadIdx.x < (int)gridDim.x ? ld_cg(A.blk_k + threadIdx.x) : 0;
                int tot;
                const int pre = block_excl_sum(cnt, sh, &tot);
                if ((unsigned long long)pre < attach_j && attach_j <= (unsigned long long)(pre + cnt)) {
                    s_i[0] = threadIdx.x;
                    s_i[1] = pre;
                }
                __syncthreads();
                const int b = s_i[0];
                const long long seg = ((long long)S.count + gridDim.x - 1) / gridDim.x;
                const long long s0 = min((long long)S.count, (long long)b * seg);
                const long long s1 = min((long long)S.count, s0 + seg);
                int pos = s_i[1];
                for (long long c0 = s0; c0 < s1; c0 += PB) {
                    if (S.mode == 1) L.tile(c0);
                    const long long i = c0 + threadIdx.x;
                    bool q = false;
                    int c = -1;
                    if (i < s1 && i > S.p0) {
                        c = S.mode == 0 ? (int)i : L.at(i);
                        q = (S.mode == 1 || ld_cg(A.vis_c + c) != token - 1) && ld_cg(A.cn_deg + c) == S.dmin;
                    }
                    const int r = block_excl_sum(q ? 1 : 0, sh, &tot);
                    if (q && (unsigned long long)(pos + r + 1) == attach_j) attach(A, c, attach_v);
                    pos += tot;
                }
            }
            __syncthreads();
        }
        // ---- 1b. BFS from v while the levels are small ------------------------
        if (do_bfs) {
            if (threadIdx.x == 0) {
                A.vis_v[v] = token;
                A.fr[0] = v;
                A.fr_cnt[0] = 1;
                *A.fr_seg = 1;
                A.sum->t_pre = 0;
            }
            for (int b = 1 + threadIdx.x; b < (int)gridDim.x; b += PB) {
                A.fr_cnt[b] = 0;   // small levels live in region 0 only
                A.lvl_cnt[b] = 0;
            }
            __syncthreads();
            int nF = 1, nL = 0, reached = 0, hl = 0, stage = 0, done = 0;
            for (;;) {
                if (stage == 0) {
                    const long long items = (long long)nF * KV;
                    if (items > kSmallLevel) break;
                    if (items <= 32) {
                        nL = expand_warp(token, A.fr, (int)items, KV, nbr_v2c, A.vis_c, A.lvl, A.lvl_cnt, A.lvl_seg,
                                         &s_i[2 * ND + 1]);
                    } else {
                        F.seg = ld_cg(A.fr_seg);
                        F.total = load_prefix(A.fr_cnt, s_pre, sh);
                        expand(A, token, hl, F, KV, nbr_v2c, A.key_c, A.vis_c, A.lvl, A.lvl_cnt, A.lvl_seg, false,
                               sh);
                        nL = ld_cg(A.lvl_cnt);
                    }
                    ++hl;
                    if (nL == 0) { done = 1; break; }
                    reached += nL;
                    if (reached == m) { done = 1; break; }
                    stage = 1;
                } else {
                    const long long items = (long long)nL * kc;
                    if (items > kSmallLevel) break;
                    if (items <= 32) {
                        nF = expand_warp(token, A.lvl, (int)items, kc, nbr_c2v, A.vis_v, A.fr, A.fr_cnt, A.fr_seg,
                                         &s_i[2 * ND + 1]);
                    } else {
                        L.seg = ld_cg(A.lvl_seg);
                        L.total = load_prefix(A.lvl_cnt, s_pre, sh);
                        expand(A, token, hl, L, kc, nbr_c2v, A.key_v, A.vis_v, A.fr, A.fr_cnt, A.fr_seg, false, sh);
                        nF = ld_cg(A.fr_cnt);
                    }
                    ++hl;
                    if (nF == 0) { done = 1; break; }
                    stage = 0;
                }
                if (hl >= kMaxHalfLevels) { done = 1; if (threadIdx.x == 0) A.sum->overflow = 1; break; }
            }
            if (threadIdx.x == 0) {
                A.bfs[0] = nF; A.bfs[1] = nL; A.bfs[2] = reached; A.bfs[3] = hl; A.bfs[4] = stage; A.bfs[5] = done;
            }
        }
    }
    if (!do_bfs) return;
    grid_barrier(A.bar);

    // ---- 2. the large levels on the whole grid ---------------------------------
    int nF = ld_cg(A.bfs + 0), nL = ld_cg(A.bfs + 1), reached = ld_cg(A.bfs + 2), hl = ld_cg(A.bfs + 3);
    int stage = ld_cg(A.bfs + 4);
    bool done = ld_cg(A.bfs + 5) != 0;
    while (!done) {
        if (stage == 0) {
            F.seg = ld_cg(A.fr_seg);
            F.total = load_prefix(A.fr_cnt, s_pre, sh);
            expand(A, token, hl, F, KV, nbr_v2c, A.key_c, A.vis_c, A.lvl, A.lvl_cnt, A.lvl_seg, true, sh);
            nL = load_prefix(A.lvl_cnt, s_pre, sh);
            ++hl;
            if (nL == 0) break;           // saturation
            reached += nL;
            if (reached == m) break;      // everything reachable: this level is the deepest
            stage = 1;
        } else {
            L.seg = ld_cg(A.lvl_seg);
            L.total = load_prefix(A.lvl_cnt, s_pre, sh);
            expand(A, token, hl, L, kc, nbr_c2v, A.key_v, A.vis_v, A.fr, A.fr_cnt, A.fr_seg, true, sh);
            nF = load_prefix(A.fr_cnt, s_pre, sh);
            ++hl;
            if (nF == 0) break;
            stage = 0;
        }
        if (hl >= kMaxHalfLevels) {
            if (blockIdx.x == 0 && threadIdx.x == 0) A.sum->overflow = 1;
            break;
        }
    }

    // ---- 3. candidate-scan summary ---------------------------------------------
    const int mode = reached < m ? 0 : 1;
    if (mode == 1) {   // the sequence is the deepest check level
        L.seg = ld_cg(A.lvl_seg);
        L.total = load_prefix(A.lvl_cnt, s_pre, sh);
    }
    const int count = mode == 0 ? m : L.total;
    auto cand_deg = [&](long long i) -> int {   // degree at sequence position i, INF if not a candidate
        if (mode == 0) return ld_cg(A.vis_c + i) == token ? INF : ld_cg(A.cn_deg + i);
        return ld_cg(A.cn_deg + L.at(i));
    };
    const long long seg = ((long long)count + gridDim.x - 1) / gridDim.x;
    const long long s0 = min((long long)count, (long long)blockIdx.x * seg), s1 = min((long long)count, s0 + seg);
    int* s_cnt = s_i;          // [ND] candidates per degree in this block's segment
    int* s_first = s_i + ND;   // [ND] first position per degree
    for (int d = threadIdx.x; d < ND; d += PB) {
        s_cnt[d] = 0;
        s_first[d] = INF;
    }
    __syncthreads();
    for (long long c0 = s0; c0 < s1; c0 += PB) {
        if (mode == 1) L.tile(c0);
        const long long i = c0 + threadIdx.x;
        if (i < s1) {
            const int d = cand_deg(i);
            if (d < ND) {
                atomicAdd(&s_cnt[d], 1);
                atomicMin(&s_first[d], (int)i);
            }
        }
    }
    __syncthreads();
    int bmin = INF;
    for (int d = ND - 1; d >= 0; --d)
        if (s_cnt[d]) bmin = d;
    for (int d = threadIdx.x; d < ND; d += PB) {
        A.st_cnt[blockIdx.x * ND + d] = s_cnt[d];
        A.st_first[blockIdx.x * ND + d] = s_first[d];
    }
    if (threadIdx.x == 0) A.blk_min[blockIdx.x] = bmin;
    grid_barrier(A.bar);
    // every block: dmin, p0, and the incoming running minimum of its segment
    // (thread t reads block t's entries; grid <= PB)
    int dmin, rin;
    {
        const int x = threadIdx.x < (int)gridDim.x ? ld_cg(A.blk_min + threadIdx.x) : INF;
        const int ex = block_excl_min(x, sh, &dmin);
        if (threadIdx.x == blockIdx.x) s_i[2 * ND] = ex;
        __syncthreads();
        rin = s_i[2 * ND];
        __syncthreads();
    }
    if (dmin >= INF) {   // no candidate at all
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            A.sum->mode = mode; A.sum->count = count; A.sum->dmin = INF; A.sum->p0 = INF; A.sum->kstar = 0;
        }
        return;
    }
    int p0, total;
    {
        const bool in = threadIdx.x < (int)gridDim.x;
        block_excl_min(in ? ld_cg(A.st_first + threadIdx.x * ND + dmin) : INF, sh, &p0);
        block_excl_sum(in ? ld_cg(A.st_cnt + threadIdx.x * ND + dmin) : 0, sh, &total);
    }
    // degree-dmin candidates after p0 per block (p0 is the first one overall)
    if (threadIdx.x == 0) {
        const int c = s_cnt[dmin];
        A.blk_k[blockIdx.x] = (s0 <= p0 && p0 < s1) ? c - 1 : c;
    }
    // running-minimum ties before p0 (draws whose outcome p0 overwrites)
    int tb = 0;
    for (long long c0 = s0; c0 < s1 && c0 < p0; c0 += PB) {
        if (mode == 1) L.tile(c0);
        const long long i = c0 + threadIdx.x;
        const int dd = (i < s1 && i < p0) ? cand_deg(i) : INF;
        int tmin;
        const int pm = min(rin, block_excl_min(dd, sh, &tmin));
        tb += __syncthreads_count(dd < INF && pm < INF && dd == pm);
        rin = min(rin, tmin);
    }
    if (threadIdx.x == 0 && tb) atomicAdd(&A.sum->t_pre, (unsigned long long)tb);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.sum->mode = mode;
        A.sum->count = count;
        A.sum->dmin = dmin;
        A.sum->p0 = p0;
        A.sum->kstar = (unsigned long long)(total - 1);
    }
}

inline uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline uint64_t xorshift64star(uint64_t x)
{
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x * 0x2545F4914F6CDD1Dull;
}

// t | s without a division: t = 2^z * o (o odd), t | s <=> the low z bits of
// s are zero and s * o^-1 (mod 2^64) <= (2^64 - 1) / o
struct DivTab {
    std::vector<uint64_t> inv, lim;
    std::vector<uint8_t> tz;
    explicit DivTab(size_t cap) : inv(cap + 1), lim(cap + 1), tz(cap + 1)
    {
        for (size_t t = 1; t <= cap; ++t) {
            const int z = __builtin_ctzll(t);
            const uint64_t o = t >> z;
            uint64_t x = o;   // Newton iteration for o^-1 mod 2^64
            for (int k = 0; k < 6; ++k) x *= 2 - o * x;
            inv[t] = x;
            lim[t] = ~0ull / o;
            tz[t] = (uint8_t)z;
        }
    }
    bool divides(uint64_t t, uint64_t s) const
    {
        if (t >= inv.size()) return s % t == 0;
        return (s & ((1ull << tz[t]) - 1)) == 0 && s * inv[t] <= lim[t];
    }
};

struct DevMem {
    std::vector<void*> ptrs;
    ~DevMem() { for (void* p : ptrs) cudaFree(p); }
    template <class T> cudaError_t alloc(T** p, size_t count, int fill)
    {
        cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(1, count * sizeof(T)));
        if (e != cudaSuccess) return e;
        ptrs.push_back(*p);
        return cudaMemset(*p, fill, count * sizeof(T));
    }
};

#define PEG_CUDA(call)                                                                               \
    do {                                                                                             \
        cudaError_t e__ = (call);                                                                    \
        if (e__ != cudaSuccess) {                                                                    \
            cudaGetLastError();                                                                      \
            return mbp::set_error(MBP_ECUDA, (std::string(#call) + ": " + cudaGetErrorString(e__)).c_str()); \
        }                                                                                            \
    } while (0)

}  // namespace

namespace {

// Variables [v_begin, v_end) of the construction on GPU `device`.  vn_adj
// (host, [n][KV], -1 = no edge) holds the graph of variables < v_begin in
// edge order and receives the rows up to v_end; *state is the tie-break
// stream's state at v_begin (derived from `seed` when v_begin == 0) and at
// v_end on return.  Check rows list their variables in attachment order,
// which is ascending variable order, so the device graph is rebuilt from
// vn_adj alone: a construction can stop and resume anywhere.
int peg_device_run(int32_t n, int32_t m, const int32_t* col_deg, uint64_t seed, uint64_t* state_io, int32_t v_begin,
                   int32_t v_end, int32_t* vn_adj_host, int device)
{
    if (!col_deg || !vn_adj_host || !state_io) return mbp::set_error(MBP_EINVAL, "null pointer argument");
    if (!(0 < m && m < n)) return mbp::set_error(MBP_EINVAL, "need 0 < m < n");
    if (v_begin < 0 || v_end < v_begin || v_end > n) return mbp::set_error(MBP_EINVAL, "bad variable range");
    int64_t E = 0;
    for (int i = 0; i < n; ++i) {
        if (col_deg[i] < 1 || col_deg[i] > std::min(m, KV))
            return mbp::set_error(MBP_EUNSUPPORTED, "column degree outside [1, min(m, 4)] (device PEG)");
        E += col_deg[i];
    }
    if (E >= (1 << 22)) return mbp::set_error(MBP_EUNSUPPORTED, "device PEG supports < 2^22 edges");
    if ((long long)n * KV >= (1 << 24) || (long long)m * KC >= (1 << 24))
        return mbp::set_error(MBP_EUNSUPPORTED, "device PEG supports n < 2^22 and m < 2^20");
    // the graph so far, rebuilt on the host
    std::vector<int> vdeg(n, 0), cdeg(m, 0), cadj((size_t)m * KC, -1);
    int kc = 1;   // effective check-adjacency slots: the largest check degree so far
    for (int v = 0; v < v_begin; ++v) {
        for (int k = 0; k < KV; ++k) {
            const int c = vn_adj_host[(size_t)v * KV + k];
            if (c < 0) break;
            if (c >= m || k >= col_deg[v]) return mbp::set_error(MBP_EINVAL, "resume graph does not fit (n, m, degrees)");
            if (cdeg[c] >= KC) return mbp::set_error(MBP_EUNSUPPORTED, "resume graph exceeds the check capacity");
            cadj[(size_t)c * KC + cdeg[c]++] = v;
            kc = std::max(kc, cdeg[c]);
            vdeg[v] = k + 1;
        }
        if (vdeg[v] != col_deg[v]) return mbp::set_error(MBP_EINVAL, "resume graph: a variable before v_begin is incomplete");
    }
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    PEG_CUDA(cudaSetDevice(device));
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev_dev};
    cudaDeviceProp prop;
    PEG_CUDA(cudaGetDeviceProperties(&prop, device));
    int per_sm = 0;
    PEG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peg_step_kernel, PB, 0));
    if (per_sm < 1) return mbp::set_error(MBP_ECUDA, "device PEG kernel does not fit on an SM");
    const int grid = std::min(prop.multiProcessorCount, PB);   // one block per SM: two builds can share the GPU

    DevMem mem;
    PegArgs A{};
    A.n = n;
    A.m = m;
    PEG_CUDA(mem.alloc(&A.vn_adj, (size_t)n * KV, 0xff));
    PEG_CUDA(mem.alloc(&A.vn_deg, n, 0));
    PEG_CUDA(mem.alloc(&A.cn_adj, (size_t)m * KC, 0xff));
    PEG_CUDA(mem.alloc(&A.cn_deg, m, 0));
    PEG_CUDA(cudaMemcpy(A.vn_adj, vn_adj_host, sizeof(int) * (size_t)n * KV, cudaMemcpyHostToDevice));
    PEG_CUDA(cudaMemcpy(A.vn_deg, vdeg.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    PEG_CUDA(cudaMemcpy(A.cn_adj, cadj.data(), sizeof(int) * (size_t)m * KC, cudaMemcpyHostToDevice));
    PEG_CUDA(cudaMemcpy(A.cn_deg, cdeg.data(), sizeof(int) * m, cudaMemcpyHostToDevice));
    PEG_CUDA(mem.alloc(&A.vis_c, m, 0));
    PEG_CUDA(mem.alloc(&A.vis_v, n, 0));
    PEG_CUDA(mem.alloc(&A.key_c, m, 0xff));
    PEG_CUDA(mem.alloc(&A.key_v, n, 0xff));
    // regions: a level's slots can outnumber its nodes, and each block owns
    // a segment of ceil(slots / grid) entries
    const size_t reg_c = (size_t)n * KV + grid, reg_v = (size_t)m * KC + grid;
    PEG_CUDA(mem.alloc(&A.lvl, reg_c, 0));
    PEG_CUDA(mem.alloc(&A.fr, std::max(reg_v, (size_t)n), 0));
    PEG_CUDA(mem.alloc(&A.lvl_cnt, grid, 0));
    PEG_CUDA(mem.alloc(&A.fr_cnt, grid, 0));
    PEG_CUDA(mem.alloc(&A.lvl_seg, 1, 0));
    PEG_CUDA(mem.alloc(&A.fr_seg, 1, 0));
    PEG_CUDA(mem.alloc(&A.blk_k, grid, 0));
    PEG_CUDA(mem.alloc(&A.blk_min, grid, 0));
    PEG_CUDA(mem.alloc(&A.st_cnt, (size_t)grid * ND, 0));
    PEG_CUDA(mem.alloc(&A.st_first, (size_t)grid * ND, 0));
    PEG_CUDA(mem.alloc(&A.bfs, 8, 0));
    PEG_CUDA(mem.alloc(&A.bar, 2, 0));
    PEG_CUDA(mem.alloc(&A.sum, 1, 0));
    PegSummary* hs = nullptr;
    PEG_CUDA(cudaHostAlloc((void**)&hs, sizeof(PegSummary), cudaHostAllocDefault));
    struct FreeHost { void* p; ~FreeHost() { if (p) cudaFreeHost(p); } } fh{hs};
    cudaStream_t s;
    PEG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct FreeStream { cudaStream_t s; ~FreeStream() { cudaStreamDestroy(s); } } fs{s};

    DivTab dt((size_t)m + 2);
    uint64_t state = *state_io;
    if (v_begin == 0) {
        state = splitmix64(seed);
        if (state == 0) state = 0x9E3779B97F4A7C15ull;
    }
    const int debug = std::getenv("MBP_PEG_DEBUG") ? std::atoi(std::getenv("MBP_PEG_DEBUG")) : 0;
    double t_rng = 0.0, t_wait = 0.0;
    unsigned long long draws = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t_start = now();
    int token = 0;
    int attach_v = -1;
    unsigned long long attach_j = 0;
    auto launch = [&](int v, int tok, int do_bfs) -> cudaError_t {
        void* args[] = {(void*)&A, (void*)&v, (void*)&tok, (void*)&attach_v, (void*)&attach_j, (void*)&do_bfs,
                        (void*)&kc};
        return cudaLaunchCooperativeKernel((const void*)peg_step_kernel, dim3(grid), dim3(PB), args, 0, s);
    };
    for (int v = v_begin; v < v_end; ++v) {
        if (debug >= 2 && v > v_begin && (v & 0xffff) == 0)
            fprintf(stderr, "peg_gpu seed=%llu: %d/%d variables, %.0f s, %.1f s GPU, %.1f s stream\n",
                    (unsigned long long)seed, v, n, std::chrono::duration<double>(now() - t_start).count(), t_wait,
                    t_rng);
        for (int e = 0; e < col_deg[v]; ++e) {
            ++token;
            const auto t0 = now();
            PEG_CUDA(launch(v, token, 1));
            PEG_CUDA(cudaMemcpyAsync(hs, A.sum, sizeof(PegSummary), cudaMemcpyDeviceToHost, s));
            PEG_CUDA(cudaStreamSynchronize(s));
            const auto t1 = now();
            t_wait += std::chrono::duration<double>(t1 - t0).count();
            if (hs->overflow)
                return mbp::set_error(MBP_EUNSUPPORTED, "device PEG capacity exceeded (check degree > 16 or BFS depth > 2^18)");
            if (hs->dmin >= INF) return mbp::set_error(MBP_EUNSUPPORTED, "PEG found no attachable check node");
            // the tie-break stream: T_pre draws whose outcome p0 overwrites,
            // then one draw per degree-dmin candidate after p0 (ties 2, 3, ...)
            for (unsigned long long k = 0; k < hs->t_pre; ++k) state = xorshift64star(state);
            unsigned long long win = 0;
            for (unsigned long long k = 1; k <= hs->kstar; ++k) {
                state = xorshift64star(state);
                if (dt.divides(k + 1, state)) win = k;
            }
            draws += hs->t_pre + hs->kstar;
            t_rng += std::chrono::duration<double>(now() - t1).count();
            if (debug == 1)
                fprintf(stderr, "peg v=%d e=%d mode=%d count=%d dmin=%d p0=%d t_pre=%llu kstar=%llu win=%llu prev_winner=%d\n",
                        v, e, hs->mode, hs->count, hs->dmin, hs->p0, hs->t_pre, hs->kstar, win, hs->winner);
            attach_v = v;
            attach_j = win;
            kc = std::min(KC, std::max(kc, hs->dmin + 1));   // the winner's new degree
        }
    }
    if (debug >= 2)
        fprintf(stderr, "peg_gpu n=%d m=%d seed=%llu [%d, %d): %.1f s total, %.1f s waiting for the GPU (%.1f us/edge), "
                        "%.1f s tie-break stream (%.3e draws, %.2f ns/draw)\n",
                n, m, (unsigned long long)seed, v_begin, v_end, std::chrono::duration<double>(now() - t_start).count(),
                t_wait, 1e6 * t_wait / std::max(1, token), t_rng, (double)draws,
                1e9 * t_rng / std::max(1.0, (double)draws));
    if (attach_v >= 0) {   // the last edge's winner
        PEG_CUDA(launch(0, token + 1, 0));
        PEG_CUDA(cudaMemcpyAsync(hs, A.sum, sizeof(PegSummary), cudaMemcpyDeviceToHost, s));
    }
    PEG_CUDA(cudaMemcpyAsync(vn_adj_host, A.vn_adj, sizeof(int) * (size_t)n * KV, cudaMemcpyDeviceToHost, s));
    PEG_CUDA(cudaStreamSynchronize(s));
    if (hs->overflow) return mbp::set_error(MBP_EUNSUPPORTED, "a check exceeded the device PEG's degree capacity");
    *state_io = state;
    return MBP_OK;
}

}  // namespace

int mbp_peg_build_device_range(int32_t n, int32_t m, const int32_t* col_deg, uint64_t seed, uint64_t* state,
                               int32_t v_begin, int32_t v_end, int32_t* vn_adj, int device)
{
    return peg_device_run(n, m, col_deg, seed, state, v_begin, v_end, vn_adj, device);
}

int mbp_peg_build_device(int32_t n, int32_t m, const int32_t* col_deg, uint64_t seed, int64_t* chk_ptr,
                         int32_t* chk_var, int device)
{
    if (!chk_ptr || !chk_var) return mbp::set_error(MBP_EINVAL, "null pointer argument");
    if (!(0 < n)) return mbp::set_error(MBP_EINVAL, "need 0 < m < n");
    std::vector<int32_t> vadj((size_t)n * KV, -1);
    uint64_t state = 0;
    int rc = peg_device_run(n, m, col_deg, seed, &state, 0, n, vadj.data(), device);
    if (rc) return rc;
    // check rows in attachment order = ascending variable order
    std::vector<int64_t> cnt(m + 1, 0);
    for (size_t i = 0; i < vadj.size(); ++i)
        if (vadj[i] >= 0) ++cnt[vadj[i] + 1];
    for (int c = 0; c < m; ++c) cnt[c + 1] += cnt[c];
    for (int c = 0; c <= m; ++c) chk_ptr[c] = cnt[c];
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int v = 0; v < n; ++v)
        for (int k = 0; k < KV; ++k) {
            const int c = vadj[(size_t)v * KV + k];
            if (c >= 0) chk_var[fill[c]++] = v;
        }
    return MBP_OK;
}
