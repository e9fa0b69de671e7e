// peg.cpp -- progressive edge growth, restating the reference's
// _kernels.peg_build (pkg/src/mmrecon/_kernels.py:57-161) and
// matrix.peg_construct (matrix.py:215-234) so that a seed gives the SAME
// matrix: the same BFS discovery order, candidate scan
// order and xorshift64* tie-break stream (seeded through splitmix64).
//
// For each new edge of variable v a BFS over the current graph splits the
// checks into unreached ones (preferred) or, when all are reachable, the
// deepest BFS level; among those the lowest-degree check wins, exact ties
// broken by a reservoir draw.  The unreached scan walks per-degree bitsets
// (ascending check order, reached checks masked out) instead of all m
// checks, with the reference's exact draw sequence (see the running-minimum
// note below).  Host code, single threaded: the
// construction is inherently sequential (every edge depends on the graph so
// far).
#include "../../include/mbp.h"

#include <cstdint>
#include <vector>

namespace mbp {
int set_error(int code, const char* msg);   // mbp.cu: thread-local mbp_last_error()
}

namespace {

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

struct DegreeSets {
    // bit c of sets[d] <=> check c has degree d
    int words;
    std::vector<std::vector<uint64_t>> sets;
    std::vector<int> count;
    DegreeSets(int m) : words((m + 63) / 64) {}
    void ensure(int d)
    {
        while ((int)sets.size() <= d) {
            sets.emplace_back(words, 0ull);
            count.push_back(0);
        }
    }
    void add(int c, int d) { ensure(d); sets[d][c >> 6] |= 1ull << (c & 63); ++count[d]; }
    void remove(int c, int d) { sets[d][c >> 6] &= ~(1ull << (c & 63)); --count[d]; }
};

}  // namespace

int mbp_peg_build(int32_t n, int32_t m, const int32_t* col_deg, uint64_t seed, int64_t* chk_ptr, int32_t* chk_var)
{
    if (!col_deg || !chk_ptr || !chk_var) return mbp::set_error(MBP_EINVAL, "null pointer argument");
    if (!(0 < m && m < n)) return mbp::set_error(MBP_EINVAL, "need 0 < m < n");
    int64_t E = 0;
    int dmax = 0;
    for (int i = 0; i < n; ++i) {
        if (col_deg[i] < 1 || col_deg[i] > m) return mbp::set_error(MBP_EINVAL, "column degree outside [1, m]");
        E += col_deg[i];
        dmax = col_deg[i] > dmax ? col_deg[i] : dmax;
    }
    std::vector<std::vector<int>> cn_adj(m);
    std::vector<int> vn_adj((size_t)n * dmax, -1), vn_deg(n, 0), cn_deg(m, 0);
    std::vector<int> chk_stamp(m, 0), var_stamp(n, 0), frontier, next_frontier, level;
    frontier.reserve(n);
    next_frontier.reserve(n);
    level.reserve(m);
    std::vector<uint64_t> reached_bits((m + 63) / 64, 0);
    DegreeSets ds(m);
    for (int c = 0; c < m; ++c) ds.add(c, 0);
    std::vector<int> reached_list;   // checks stamped in the current BFS (to clear reached_bits)
    reached_list.reserve(m);
    int token = 0;
    uint64_t state = splitmix64(seed);
    if (state == 0) state = 0x9E3779B97F4A7C15ull;

    for (int v = 0; v < n; ++v) {
        for (int e = 0; e < col_deg[v]; ++e) {
            ++token;
            var_stamp[v] = token;
            frontier.assign(1, v);
            int reached = 0;
            reached_list.clear();
            level.clear();
            for (;;) {
                level.clear();
                for (int w : frontier)
                    for (int k = 0; k < vn_deg[w]; ++k) {
                        const int c = vn_adj[(size_t)w * dmax + k];
                        if (chk_stamp[c] != token) {
                            chk_stamp[c] = token;
                            level.push_back(c);
                        }
                    }
                if (level.empty()) break;   // saturation: the rest is unreachable
                for (int c : level) {
                    reached_bits[c >> 6] |= 1ull << (c & 63);
                    reached_list.push_back(c);
                }
                reached += (int)level.size();
                if (reached == m) break;    // all reachable: this level is the deepest
                next_frontier.clear();
                for (int c : level)
                    for (int w : cn_adj[c])
                        if (var_stamp[w] != token) {
                            var_stamp[w] = token;
                            next_frontier.push_back(w);
                        }
                if (next_frontier.empty()) break;
                frontier.swap(next_frontier);
            }
            int best = -1;
            uint64_t ties = 0;
            if (reached < m) {
                // The reference scans every unreached check in ascending order
                // with a running minimum degree; a draw is taken for each
                // check tying the running minimum.  Let dmin be the lowest
                // unreached degree and p0 its first check: before p0 the
                // running minimum is above dmin (scanned literally, usually a
                // short prefix); from p0 on only degree-dmin checks tie.
                int dmin = -1;
                for (int d = 0; d < (int)ds.sets.size() && dmin < 0; ++d) {
                    if (ds.count[d] == 0) continue;
                    for (int wdx = 0; wdx < ds.words; ++wdx)
                        if (ds.sets[d][wdx] & ~reached_bits[wdx]) { dmin = d; break; }
                }
                if (dmin >= 0) {
                    const std::vector<uint64_t>& bits = ds.sets[dmin];
                    int p0 = -1, w0 = 0;
                    for (; w0 < ds.words; ++w0) {
                        const uint64_t x = bits[w0] & ~reached_bits[w0];
                        if (x) { p0 = w0 * 64 + __builtin_ctzll(x); break; }
                    }
                    int best_deg = 1 << 30;
                    for (int c = 0; c < p0; ++c) {
                        if ((reached_bits[c >> 6] >> (c & 63)) & 1ull) continue;
                        const int d = cn_deg[c];
                        if (d < best_deg) {
                            best = c;
                            best_deg = d;
                            ties = 1;
                        } else if (d == best_deg) {
                            ++ties;
                            state = xorshift64star(state);
                            if (state % ties == 0) best = c;
                        }
                    }
                    best = p0;   // dmin < best_deg: the running minimum resets here
                    ties = 1;
                    uint64_t x = (bits[w0] & ~reached_bits[w0]) & ~((2ull << (p0 & 63)) - 1ull);
                    for (int wdx = w0;;) {
                        while (x) {
                            const int c = wdx * 64 + __builtin_ctzll(x);
                            x &= x - 1;
                            ++ties;
                            state = xorshift64star(state);
                            if (state % ties == 0) best = c;
                        }
                        if (++wdx >= ds.words) break;
                        x = bits[wdx] & ~reached_bits[wdx];
                    }
                }
            } else {
                int best_deg = 1 << 30;
                for (int c : level) {
                    const int d = cn_deg[c];
                    if (d < best_deg) {
                        best = c;
                        best_deg = d;
                        ties = 1;
                    } else if (d == best_deg) {
                        ++ties;
                        state = xorshift64star(state);
                        if (state % ties == 0) best = c;
                    }
                }
            }
            for (int c : reached_list) reached_bits[c >> 6] &= ~(1ull << (c & 63));
            if (best < 0) return mbp::set_error(MBP_EUNSUPPORTED, "PEG found no attachable check node");
            ds.remove(best, cn_deg[best]);
            ++cn_deg[best];
            ds.add(best, cn_deg[best]);
            cn_adj[best].push_back(v);
            vn_adj[(size_t)v * dmax + vn_deg[v]++] = best;
        }
    }
    // rows in insertion order = ascending variable index (from_check_adjacency sorts)
    chk_ptr[0] = 0;
    for (int c = 0; c < m; ++c) {
        chk_ptr[c + 1] = chk_ptr[c] + (int64_t)cn_adj[c].size();
        int64_t o = chk_ptr[c];
        for (int w : cn_adj[c]) chk_var[o++] = w;
    }
    return chk_ptr[m] == E ? MBP_OK : mbp::set_error(MBP_EINVAL, "internal: edge count mismatch");
}
