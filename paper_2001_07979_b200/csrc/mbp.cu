// mbp.cu -- host side of libmbp_b200.so: the C ABI of include/mbp.h.
//
// Owns device copies of the stacked graph (mbp_ensemble) and per-batch
// device buffers (mbp_workspace); enqueues the transposes and the persistent
// cooperative decode kernel of kernels.cuh.  No torch, no Python: callers
// bind it with ctypes (paper_2001_07979_b200/_native.py) or any FFI.
#include "../../include/mbp.h"
#include "launch.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg)
{
    g_last_error = msg;
    return code;
}

#define MBP_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t err__ = (call);                                                             \
        if (err__ != cudaSuccess)                                                               \
            return fail(MBP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(err__));      \
    } while (0)

// Smallest double x with tanh(x/2) == 1.0 under the host libm -- where the
// reference's float64 product saturates (_kernels.py:242, 249-252) -- rounded
// up to float (the fp32 path compares float messages against it).
float saturation_threshold()
{
    double lo = 1.0, hi = 100.0;
    for (int k = 0; k < 200; ++k) {
        const double mid = 0.5 * (lo + hi);
        if (std::tanh(0.5 * mid) == 1.0) hi = mid; else lo = mid;
    }
    float f = (float)hi;
    if ((double)f < hi) f = std::nextafter(f, INFINITY);
    return f;
}

}  // namespace

// error reporting for the host-only translation units (peg.cpp)
namespace mbp {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace mbp

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() { if (p) cudaFree(p); }
    int alloc(size_t b)
    {
        if (p) { cudaFree(p); p = nullptr; }
        bytes = b;
        if (!b) return MBP_OK;
        if (cudaMalloc(&p, b) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(MBP_ENOMEM, "cudaMalloc of " + std::to_string(b) + " bytes failed");
        }
        return MBP_OK;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) { cudaGetDevice(&prev); if (prev != dev) cudaSetDevice(dev); }
    ~DeviceGuard() { int cur; cudaGetDevice(&cur); if (prev >= 0 && cur != prev) cudaSetDevice(prev); }
};

int pick_degree(int dmax)
{
    if (dmax <= 8) return 8;
    if (dmax <= 16) return 16;
    if (dmax <= 32) return 32;
    if (dmax <= 64) return 64;
    return 0;
}

}  // namespace

struct mbp_ensemble {
    int n = 0, m = 0, u = 0, C = 0;
    long long E = 0;
    int dmax_c = 0, dmax_v = 0;
    int Ds = 0;       // ELL row stride = max check degree
    int dv_reg = 0;   // regular column degree (0 if irregular)
    int device = 0, sm_count = 0;
    float sat = 0.f;
    std::vector<long long> edge_off;  // [u+1] reference edge offsets
    // reference CSR (single-phase kernels)
    DevBuf chk_ptr, chk_var, var_ptr, var_edge;  // int32
    // decode layout: padded ELL rows + slot ids per variable
    DevBuf deg, chk_ell, var_slot, ref2slot;
    DevBuf var_chk;   // stacked check id of each variable's edges (ascending edge order)
    // stream of the single-phase ABI (mbp_c2v_pass & co.): never the legacy
    // default stream, so they do not serialise against other streams
    cudaStream_t op_stream = nullptr;
    ~mbp_ensemble() { if (op_stream) cudaStreamDestroy(op_stream); }
};

struct mbp_workspace {
    mbp_ensemble* ens = nullptr;
    mbp_decoder_config cfg{};
    int cap = 0, G = 0;
    size_t real_size = 4;
    DevBuf c2v, post, v2c, Lmag, noisy_w, syn_w, hard_w, hist_w, cnt, any_bad, iters, barrier,
        sweeps, ts, work, tmp_in,
        c2v_b, post_b, v2c_b, Lmag_b, noisy_b, syn_b, hard_b, cnt_b, fid_b, src_b, newslot, grp_cnt, ctrl, tmp_out, tmp_conv, tmp_iters, tmp_mism, tmp_e;
    // scatter path (scatter.cuh)
    DevBuf sc_vb, sc_mis, sc_Mtab, sc_Lfix, sc_Mfix, sc_Lmax, sc_vb_b, sc_Mtab_b, sc_Lfix_b, sc_mis_b;
    bool scatter = false;   // path of the current configuration
    int ts_cap = 0;
    int Gb = 0;        // compaction capacity (groups), 0 = disabled
    cudaStream_t own_stream = nullptr;
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;   // host-path pipeline
    static constexpr int kMaxSub = 8;
    cudaEvent_t ev_in[kMaxSub] = {}, ev_out[kMaxSub] = {}, ev_fin[kMaxSub] = {}, ev_d2h = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
    int last_B = 0;
    bool timed = false, e2e_timed = false;
    // pinned staging of the host path's crossover probabilities: an async
    // copy from pageable memory would block the issuing thread until the
    // copy stream drains, serialising the staging ring
    double* e_host = nullptr;
    size_t e_host_cap = 0;
    ~mbp_workspace()
    {
        if (e_host) cudaFreeHost(e_host);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (ev2) cudaEventDestroy(ev2);
        if (ev3) cudaEventDestroy(ev3);
        for (int i = 0; i < kMaxSub; ++i) {
            if (ev_in[i]) cudaEventDestroy(ev_in[i]);
            if (ev_out[i]) cudaEventDestroy(ev_out[i]);
            if (ev_fin[i]) cudaEventDestroy(ev_fin[i]);
        }
        if (ev_d2h) cudaEventDestroy(ev_d2h);
        if (own_stream) cudaStreamDestroy(own_stream);
        if (h2d_stream) cudaStreamDestroy(h2d_stream);
        if (d2h_stream) cudaStreamDestroy(d2h_stream);
    }
};

// Exported functions take C linkage from their declarations in mbp.h.

const char* mbp_last_error(void) { return g_last_error.c_str(); }

const char* mbp_version(void) { return "mbp_b200 0.1.0 (sm_100a)"; }

int mbp_device_count(int* count)
{
    if (!count) return fail(MBP_EINVAL, "count is null");
    MBP_CUDA(cudaGetDeviceCount(count));
    return MBP_OK;
}

int mbp_ensemble_create(int32_t n, int32_t m, int32_t u, const int64_t* chk_ptr,
                        const int32_t* chk_var, int device, mbp_ensemble** out)
{
    if (!out || !chk_ptr || !chk_var) return fail(MBP_EINVAL, "null pointer argument");
    *out = nullptr;
    if (!(0 < m && 0 < n)) return fail(MBP_EINVAL, "need m > 0 and n > 0, got m=" + std::to_string(m) + ", n=" + std::to_string(n));
    if (u < 1 || u > MBP_MAX_MATRICES) return fail(MBP_EINVAL, "u must be in [1, " + std::to_string(MBP_MAX_MATRICES) + "]");
    const long long C = (long long)u * m;
    const long long E = chk_ptr[C];
    if (chk_ptr[0] != 0 || E <= 0 || E >= (1LL << 31) / 32)
        return fail(MBP_EINVAL, "bad stacked chk_ptr (edge count " + std::to_string(E) + ")");
    auto* ens = new mbp_ensemble;
    ens->n = n; ens->m = m; ens->u = u; ens->C = (int)C; ens->E = E; ens->device = device;
    std::vector<int> cp(C + 1), cv(E), col_deg(n, 0);
    int dmax_c = 0;
    for (long long j = 0; j < C; ++j) {
        if (chk_ptr[j + 1] < chk_ptr[j]) { delete ens; return fail(MBP_EINVAL, "chk_ptr not monotone"); }
        dmax_c = std::max<int>(dmax_c, (int)(chk_ptr[j + 1] - chk_ptr[j]));
        cp[j] = (int)chk_ptr[j];
    }
    cp[C] = (int)E;
    for (long long e = 0; e < E; ++e) {
        const int v = chk_var[e];
        if (v < 0 || v >= n) { delete ens; return fail(MBP_EINVAL, "variable index out of range at edge " + std::to_string(e)); }
        cv[e] = v;
        ++col_deg[v];
    }
    // edge_off: matrix l owns edges [chk_ptr[l*m], chk_ptr[(l+1)*m])
    ens->edge_off.resize(u + 1);
    for (int l = 0; l <= u; ++l) ens->edge_off[l] = chk_ptr[(long long)l * m];
    // variable side: stable counting sort of edges by variable (ascending ids)
    std::vector<int> vp(n + 1, 0), ve(E);
    int dmax_v = 0;
    for (int i = 0; i < n; ++i) {
        if (col_deg[i] == 0) { delete ens; return fail(MBP_EINVAL, "variable " + std::to_string(i) + " has degree 0"); }
        vp[i + 1] = vp[i] + col_deg[i];
        dmax_v = std::max(dmax_v, col_deg[i]);
    }
    {
        std::vector<int> fill(vp.begin(), vp.end() - 1);
        for (long long e = 0; e < E; ++e) ve[fill[cv[e]]++] = (int)e;
    }
    ens->dmax_c = dmax_c;
    ens->dmax_v = dmax_v;
    ens->sat = saturation_threshold();
    ens->Ds = std::max(dmax_c, 1);
    ens->dv_reg = dmax_v;
    for (int i = 0; i < n; ++i)
        if (col_deg[i] != dmax_v) { ens->dv_reg = 0; break; }
    // padded ELL: edge k of check j -> slot j*Ds + k (monotone in the reference edge id)
    const int D = ens->Ds;
    std::vector<uint8_t> rowdeg(C);
    std::vector<int> ell((size_t)C * D, 0), r2s(E), vs(E);
    for (long long j = 0; j < C; ++j) {
        const int d = (int)(chk_ptr[j + 1] - chk_ptr[j]);
        rowdeg[j] = (uint8_t)std::min(d, 255);
        for (int k = 0; k < d && k < D; ++k) {
            ell[(size_t)j * D + k] = cv[chk_ptr[j] + k];
            r2s[chk_ptr[j] + k] = (int)((size_t)j * D + k);
        }
    }
    for (long long t = 0; t < E; ++t) vs[t] = r2s[ve[t]];
    std::vector<int> vchk(E);
    for (long long t = 0; t < E; ++t) vchk[t] = vs[t] / D;
    int rc;
    {
        DeviceGuard dg(device);
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
            delete ens;
            cudaGetLastError();
            return fail(MBP_ECUDA, "no CUDA device " + std::to_string(device));
        }
        ens->sm_count = prop.multiProcessorCount;
        if (cudaStreamCreateWithFlags(&ens->op_stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete ens;
            cudaGetLastError();
            return fail(MBP_ECUDA, "stream creation failed");
        }
        if ((rc = ens->chk_ptr.alloc(sizeof(int) * (C + 1))) || (rc = ens->chk_var.alloc(sizeof(int) * E)) ||
            (rc = ens->var_ptr.alloc(sizeof(int) * (n + 1))) || (rc = ens->var_edge.alloc(sizeof(int) * E)) ||
            (rc = ens->deg.alloc(C)) || (rc = ens->chk_ell.alloc(sizeof(int) * (size_t)C * D)) ||
            (rc = ens->var_slot.alloc(sizeof(int) * E)) || (rc = ens->ref2slot.alloc(sizeof(int) * E)) ||
            (rc = ens->var_chk.alloc(sizeof(int) * E))) {
            delete ens;
            return rc;
        }
        cudaError_t err = cudaMemcpy(ens->chk_ptr.p, cp.data(), sizeof(int) * (C + 1), cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->chk_var.p, cv.data(), sizeof(int) * E, cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->var_ptr.p, vp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->var_edge.p, ve.data(), sizeof(int) * E, cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->deg.p, rowdeg.data(), C, cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->chk_ell.p, ell.data(), sizeof(int) * (size_t)C * D, cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->var_slot.p, vs.data(), sizeof(int) * E, cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->ref2slot.p, r2s.data(), sizeof(int) * E, cudaMemcpyHostToDevice);
        if (err == cudaSuccess) err = cudaMemcpy(ens->var_chk.p, vchk.data(), sizeof(int) * E, cudaMemcpyHostToDevice);
        if (err != cudaSuccess) { delete ens; return fail(MBP_ECUDA, std::string("ensemble upload: ") + cudaGetErrorString(err)); }
    }
    *out = ens;
    return MBP_OK;
}

int mbp_ensemble_destroy(mbp_ensemble* ens)
{
    if (ens) { DeviceGuard dg(ens->device); delete ens; }
    return MBP_OK;
}

int mbp_ensemble_get_info(const mbp_ensemble* ens, mbp_ensemble_info* info)
{
    if (!ens || !info) return fail(MBP_EINVAL, "null pointer argument");
    info->n = ens->n; info->m = ens->m; info->u = ens->u; info->edges = ens->E;
    info->max_check_degree = ens->dmax_c; info->max_var_degree = ens->dmax_v;
    info->device = ens->device; info->sm_count = ens->sm_count;
    return MBP_OK;
}

static int validate_cfg(const mbp_decoder_config* cfg)
{
    if (!cfg) return fail(MBP_EINVAL, "config is null");
    if (cfg->max_iterations < 1) return fail(MBP_EINVAL, "max_iterations must be >= 1, got " + std::to_string(cfg->max_iterations));
    if (!(cfg->llr_clamp > 0)) return fail(MBP_EINVAL, "llr_clamp must be positive");
    if (!(cfg->damping >= 0.0 && cfg->damping <= 1.0)) return fail(MBP_EINVAL, "damping must be in [0, 1]");
    if (cfg->combining_mode != MBP_JOINT_GRAPH && cfg->combining_mode != MBP_ISOLATED_PER_MATRIX)
        return fail(MBP_EINVAL, "combining_mode must be joint-graph or isolated-per-matrix");
    if (cfg->precision != MBP_FP32_PHI && cfg->precision != MBP_FP64_TANH)
        return fail(MBP_EINVAL, "precision must be MBP_FP32_PHI or MBP_FP64_TANH");
    return MBP_OK;
}

// Degree bound of a scatter-kernel instance (k_scatter.cu), 0 if none.
static int scatter_degree(int Ds)
{
    if (Ds <= 16) return std::max(Ds, 3);
    for (int d : {20, 24, 32, 48, 64}) if (Ds <= d) return d;
    return 0;
}

// The scatter kernel (scatter.cuh) runs fp32, joint-graph, undamped decodes
// whose fixed-point range stays fine: |acc| <= L + dv_max * clamp must leave
// >= 19 fractional bits (L <= 745 for any double e).
static bool scatter_eligible(const mbp_ensemble* ens, const mbp_decoder_config& cfg)
{
    return cfg.precision == MBP_FP32_PHI && cfg.combining_mode == MBP_JOINT_GRAPH && cfg.damping == 0.0 &&
           !(cfg.flags & MBP_EXPLICIT_MESSAGES) && scatter_degree(ens->Ds) != 0 &&
           (double)ens->n * mbp::kVB * 4 < 4294967296.0 &&   // 32-bit byte offsets of variable blocks
           (double)ens->dmax_v * cfg.llr_clamp <= 1024.0;
}

static int fit(DevBuf& b, size_t bytes)
{
    return b.bytes == bytes ? MBP_OK : b.alloc(bytes);
}

// (Re)allocate the buffers whose shape depends on cfg.
static int ws_alloc(mbp_workspace* ws)
{
    const mbp_ensemble* ens = ws->ens;
    const size_t F = (size_t)ws->G * 32, R = ws->real_size;
    const size_t P = ws->cfg.combining_mode == MBP_ISOLATED_PER_MATRIX ? (size_t)ens->u + 1 : 1;
    int rc;
    const size_t slots = (size_t)ens->C * ens->Ds;
    ws->scatter = scatter_eligible(ens, ws->cfg);
    if (ws->c2v.bytes != ws->G * slots * 32 * R && (rc = ws->c2v.alloc(ws->G * slots * 32 * R))) return rc;
    const size_t post_bytes = ws->scatter ? 0 : ws->G * P * ens->n * 32 * R;
    if ((rc = fit(ws->post, post_bytes))) return rc;
    const size_t v2c_bytes = ws->cfg.damping != 0.0 ? ws->G * slots * 32 * R : 0;
    if (ws->v2c.bytes != v2c_bytes && (rc = ws->v2c.alloc(v2c_bytes))) return rc;
    const size_t hist_bytes = (ws->cfg.flags & MBP_RECORD_HISTORY)
        ? (size_t)(ws->cfg.max_iterations + 1) * ws->G * ens->n * 4 : 0;
    if (ws->hist_w.bytes != hist_bytes && (rc = ws->hist_w.alloc(hist_bytes))) return rc;
    // frame compaction (decode.cuh): secondary layout of ceil(G/2) groups;
    // off for the diagnostic modes, which read state by original frame index
    // off when recording histories (written by original frame index); kept
    // state stays readable through the slot map (moved_slot)
    const bool compaction = ws->G >= 2 && !(ws->cfg.flags & (MBP_RECORD_HISTORY | MBP_NO_COMPACTION));
    ws->Gb = compaction ? (ws->G + 1) / 2 : 0;
    {
        const size_t Gb = ws->Gb, Fb = Gb * 32;
        if (ws->c2v_b.bytes != Gb * slots * 32 * R && (rc = ws->c2v_b.alloc(Gb * slots * 32 * R))) return rc;
        if (ws->post_b.bytes != Gb * P * ens->n * 32 * R && (rc = ws->post_b.alloc(Gb * P * ens->n * 32 * R))) return rc;
        const size_t vb = ws->cfg.damping != 0.0 ? Gb * slots * 32 * R : 0;
        if (ws->v2c_b.bytes != vb && (rc = ws->v2c_b.alloc(vb))) return rc;
        if (ws->Lmag_b.bytes != Fb * R && (rc = ws->Lmag_b.alloc(Fb * R))) return rc;
        if (ws->noisy_b.bytes != Gb * ens->n * 4 && (rc = ws->noisy_b.alloc(Gb * ens->n * 4))) return rc;
        if (ws->hard_b.bytes != Gb * ens->n * 4 && (rc = ws->hard_b.alloc(Gb * ens->n * 4))) return rc;
        if (ws->syn_b.bytes != Gb * ens->C * 4 && (rc = ws->syn_b.alloc(Gb * ens->C * 4))) return rc;
        if (ws->cnt_b.bytes != 2 * Fb * 4 && (rc = ws->cnt_b.alloc(2 * Fb * 4))) return rc;
        if (ws->fid_b.bytes != Fb * 4 && (rc = ws->fid_b.alloc(Fb * 4))) return rc;
        if (ws->src_b.bytes != Fb * 4 && (rc = ws->src_b.alloc(Fb * 4))) return rc;
        const size_t F = (size_t)ws->G * 32;
        if (ws->newslot.bytes != (Gb ? F * 4 : 0) && (rc = ws->newslot.alloc(Gb ? F * 4 : 0))) return rc;
        if (ws->grp_cnt.bytes != (Gb ? (size_t)ws->G * 4 : 0) && (rc = ws->grp_cnt.alloc(Gb ? (size_t)ws->G * 4 : 0))) return rc;
        const size_t cb = (size_t)(2 * (ws->cfg.max_iterations + 2)) * 4;
        if (ws->ctrl.bytes != cb && (rc = ws->ctrl.alloc(cb))) return rc;
    }
    {   // scatter-path state (sized 0 when the explicit kernel runs)
        const bool sc = ws->scatter;
        const size_t G = ws->G, Gb = ws->Gb, n = ens->n, C = ens->C, Dm1 = ens->Ds + 1;
        if ((rc = fit(ws->sc_vb, sc ? G * n * mbp::kVB * 4 : 0)) ||
            (rc = fit(ws->sc_mis, sc ? G * C * 4 : 0)) || (rc = fit(ws->sc_Mtab, sc ? Dm1 * G * 32 * 4 : 0)) ||
            (rc = fit(ws->sc_Lfix, sc ? G * 32 * 4 : 0)) || (rc = fit(ws->sc_Mfix, sc ? Dm1 * G * 32 * 4 : 0)) ||
            (rc = fit(ws->sc_Lmax, sc ? 4 : 0)) || (rc = fit(ws->sc_vb_b, sc ? Gb * n * mbp::kVB * 4 : 0)) ||
            (rc = fit(ws->sc_Mtab_b, sc ? Dm1 * Gb * 32 * 4 : 0)) ||
            (rc = fit(ws->sc_Lfix_b, sc ? Gb * 32 * 4 : 0)) || (rc = fit(ws->sc_mis_b, sc ? Gb * C * 4 : 0)))
            return rc;
        if (sc && (rc = fit(ws->post_b, 0))) return rc;
    }
    const size_t work_bytes = (size_t)(3 * (ws->cfg.max_iterations + 1) + 2) * 4;
    if (ws->work.bytes != work_bytes && (rc = ws->work.alloc(work_bytes))) return rc;
    ws->ts_cap = (ws->cfg.flags & MBP_PROFILE_PHASES) ? 3 * (ws->cfg.max_iterations + 1) + 8 : 0;
    if (ws->ts.bytes != (size_t)ws->ts_cap * 8 && (rc = ws->ts.alloc((size_t)ws->ts_cap * 8))) return rc;
    if (!ws->Lmag.p) {
        if ((rc = ws->Lmag.alloc(F * R)) || (rc = ws->noisy_w.alloc((size_t)ws->G * ens->n * 4)) ||
            (rc = ws->syn_w.alloc((size_t)ws->G * ens->C * 4)) || (rc = ws->hard_w.alloc((size_t)ws->G * ens->n * 4)) ||
            (rc = ws->cnt.alloc(2 * F * 4)) || (rc = ws->any_bad.alloc(2 * 4)) || (rc = ws->iters.alloc(F * 4)) ||
            (rc = ws->barrier.alloc(2 * 4)) || (rc = ws->sweeps.alloc(16 * 4)))
            return rc;
    }
    return MBP_OK;
}

int mbp_workspace_create(mbp_ensemble* ens, int32_t max_frames, const mbp_decoder_config* cfg,
                         mbp_workspace** out)
{
    if (!ens || !out) return fail(MBP_EINVAL, "null pointer argument");
    *out = nullptr;
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (max_frames < 1) return fail(MBP_EINVAL, "max_frames must be >= 1");
    if (!pick_degree(ens->dmax_c))
        return fail(MBP_EUNSUPPORTED, "check degree " + std::to_string(ens->dmax_c) + " exceeds MBP_MAX_CHECK_DEGREE");
    DeviceGuard dg(ens->device);
    auto* ws = new mbp_workspace;
    ws->ens = ens;
    ws->cfg = *cfg;
    ws->cap = max_frames;
    ws->G = (max_frames + 31) / 32;
    ws->real_size = cfg->precision == MBP_FP64_TANH ? 8 : 4;
    if ((rc = ws_alloc(ws))) { delete ws; return rc; }
    bool ok = cudaStreamCreateWithFlags(&ws->h2d_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&ws->d2h_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&ws->ev_d2h, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < mbp_workspace::kMaxSub; ++i)
        ok = cudaEventCreateWithFlags(&ws->ev_in[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&ws->ev_out[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&ws->ev_fin[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok || cudaStreamCreateWithFlags(&ws->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&ws->ev0) != cudaSuccess || cudaEventCreate(&ws->ev1) != cudaSuccess ||
        cudaEventCreate(&ws->ev2) != cudaSuccess || cudaEventCreate(&ws->ev3) != cudaSuccess) {
        delete ws;
        cudaGetLastError();
        return fail(MBP_ECUDA, "stream/event creation failed");
    }
    *out = ws;
    return MBP_OK;
}

int mbp_workspace_destroy(mbp_workspace* ws)
{
    if (ws) { DeviceGuard dg(ws->ens->device); delete ws; }
    return MBP_OK;
}

int mbp_workspace_configure(mbp_workspace* ws, const mbp_decoder_config* cfg)
{
    if (!ws) return fail(MBP_EINVAL, "workspace is null");
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (cfg->precision != ws->cfg.precision || cfg->combining_mode != ws->cfg.combining_mode)
        return fail(MBP_EINVAL, "precision and combining_mode are fixed at workspace creation");
    DeviceGuard dg(ws->ens->device);
    ws->cfg = *cfg;
    return ws_alloc(ws);
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
static int launch_rows_to_words(const uint8_t* rows, long long row_bytes, int B, int G, int nseg,
                                int seg_bits, long long seg_bytes, unsigned* words, unsigned* words2,
                                long long wpg, cudaStream_t s)
{
    const long long tiles = (long long)G * nseg * ((seg_bytes + mbp::kTileBytes - 1) / mbp::kTileBytes);
    const int grid = (int)std::max(1LL, std::min(tiles, 148LL * 8));
    mbp::rows_to_words_kernel<<<grid, 256, 0, s>>>(rows, row_bytes, B, G, nseg, seg_bits, seg_bytes, words,
                                                   words2, wpg);
    MBP_CUDA(cudaGetLastError());
    return MBP_OK;
}

static int launch_words_to_rows(const unsigned* words, long long wpg, int B, int G, int nseg,
                                int seg_bits, long long seg_bytes, uint8_t* rows, long long row_bytes,
                                cudaStream_t s)
{
    const long long tiles = (long long)G * nseg * ((seg_bytes + mbp::kTileBytes - 1) / mbp::kTileBytes);
    const int grid = (int)std::max(1LL, std::min(tiles, 148LL * 8));
    mbp::words_to_rows_kernel<<<grid, 256, 0, s>>>(words, wpg, B, G, nseg, seg_bits, seg_bytes, rows, row_bytes);
    MBP_CUDA(cudaGetLastError());
    return MBP_OK;
}

template <class Real>
static int dispatch_decode(mbp_workspace* ws, mbp::DecodeArgs<Real>& A, cudaStream_t s)
{
    const bool damp = ws->cfg.damping != 0.0;
    const bool iso = ws->cfg.combining_mode == MBP_ISOLATED_PER_MATRIX;
    const int D = pick_degree(ws->ens->Ds);
    MBP_CUDA(cudaEventRecord(ws->ev0, s));
    cudaError_t err = sizeof(Real) == 8
        ? mbp::launch_explicit_f64(reinterpret_cast<mbp::DecodeArgs<double>&>(A), D, damp, iso, ws->ens->sm_count, s)
        : mbp::launch_explicit_f32(reinterpret_cast<mbp::DecodeArgs<float>&>(A), D, damp, iso, ws->ens->sm_count, s);
    if (err == cudaErrorNotSupported) return fail(MBP_EUNSUPPORTED, "check degree too large");
    MBP_CUDA(err);
    MBP_CUDA(cudaEventRecord(ws->ev1, s));
    ws->timed = true;
    return MBP_OK;
}

// Hot/tail split (scatter.cuh): the hot instance runs sweeps 1..3 and, when
// frames remain, leaves its loop state in ws->sweeps[8..15] for the full
// instance launched behind it (which returns at once otherwise).  Saturating
// inputs (clamp >= sat) and wide rows run the full instance alone.
// MBP_NO_HOT=1 in the environment forces the single full launch (A/B runs).
static bool hot_split_enabled()
{
    static const bool on = [] {
        const char* v = std::getenv("MBP_NO_HOT");
        return !(v && std::atoi(v) != 0);
    }();
    return on;
}

static int dispatch_scatter(mbp_workspace* ws, mbp::ScatterArgs A, cudaStream_t s)
{
    const int D = scatter_degree(ws->ens->Ds);
    const int sm = ws->ens->sm_count;
    const bool split = D <= 16 && A.clamp < A.sat && hot_split_enabled();
    MBP_CUDA(cudaEventRecord(ws->ev0, s));
    cudaError_t err = cudaSuccess;
    A.resume = split ? ws->sweeps.as<int>() + 8 : nullptr;
    if (split) {
        err = D <= 8 ? mbp::launch_scatter_small(A, D, true, sm, s) : mbp::launch_scatter_mid(A, D, true, sm, s);
        if (err == cudaSuccess)
            err = D <= 8 ? mbp::launch_scatter_small(A, D, false, sm, s) : mbp::launch_scatter_mid(A, D, false, sm, s);
    } else {
        err = D <= 8 ? mbp::launch_scatter_small(A, D, false, sm, s)
            : D <= 16 ? mbp::launch_scatter_mid(A, D, false, sm, s)
                      : mbp::launch_scatter_large(A, D, sm, s);
    }
    if (err == cudaErrorNotSupported) return fail(MBP_EUNSUPPORTED, "check degree too large");
    MBP_CUDA(err);
    MBP_CUDA(cudaEventRecord(ws->ev1, s));
    ws->timed = true;
    return MBP_OK;
}

template <class Real>
static __global__ void fill_post_prior_kernel(const unsigned* __restrict__ noisy_w, const Real* __restrict__ L,
                                              int G, int n, int P, Real* __restrict__ post)
{
    const long long total = (long long)G * P * n * 32;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const int lane = (int)(k & 31);
        const int i = (int)((k >> 5) % n);
        const int g = (int)((k >> 5) / ((long long)n * P));
        const unsigned w = noisy_w[(long long)g * n + i];
        const Real l = L[g * 32 + lane];
        post[k] = ((w >> lane) & 1u) ? -l : l;
    }
}

// scatter-path state is kept in the noisy-relative domain (scatter.cuh):
// post' = (-1)^y post.  Prior fill and readback convert.
static __global__ void fill_rel_prior_kernel(const float* __restrict__ L, int G, int n, float* __restrict__ vb)
{
    const long long total = (long long)G * n * 32;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x)
        vb[(k >> 5) * mbp::kVB + (k & 31)] = L[(k >> 5) / n * 32 + (k & 31)];   // line 0 of the block
}

static __global__ void gather_rel_post_kernel(const float* __restrict__ vb_g, const unsigned* __restrict__ noisy_g,
                                              int n, int lane, double* __restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double v = vb_g[(long long)i * mbp::kVB + lane] * 0.69314718055994530942;   // log2 -> natural units
        dst[i] = ((noisy_g[i] >> lane) & 1u) ? -v : v;
    }
}

// The per-chunk control state (counters, flags, slot maps) reset by one
// launch instead of a dozen small memsets.
struct FillSpan {
    unsigned* p;
    long long words;
    unsigned v;
};
struct FillArgs {
    FillSpan s[12];
    int n;
};

static __global__ void fill_spans_kernel(FillArgs a)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    for (int k = 0; k < a.n; ++k)
        for (long long i = t; i < a.s[k].words; i += st) a.s[k].p[i] = a.s[k].v;
}

static int reset_chunk_state(mbp_workspace* ws, int F, cudaStream_t s, bool lmax)
{
    FillArgs a{};
    auto add = [&](const DevBuf& b, size_t bytes, unsigned v) {
        if (bytes) a.s[a.n++] = FillSpan{(unsigned*)b.p, (long long)(bytes / 4), v};
    };
    add(ws->cnt, 2 * (size_t)F * 4, 0u);
    add(ws->any_bad, 8, 0u);
    add(ws->iters, (size_t)F * 4, ~0u);
    add(ws->barrier, 8, 0u);
    add(ws->work, ws->work.bytes, 0u);
    add(ws->sweeps, 16 * 4, 0u);   // sweeps_run[2] + the hot instance's resume block [8..15]
    if (ws->Gb) {
        add(ws->ctrl, ws->ctrl.bytes, 0u);
        add(ws->fid_b, ws->fid_b.bytes, ~0u);
        add(ws->src_b, ws->src_b.bytes, ~0u);
        add(ws->newslot, ws->newslot.bytes, ~0u);
    }
    if (lmax) add(ws->sc_Lmax, 4, 0u);
    fill_spans_kernel<<<64, 256, 0, s>>>(a);
    MBP_CUDA(cudaGetLastError());
    return MBP_OK;
}

// Scatter path (scatter.cuh) for one chunk of <= ws->cap frames.
static int decode_chunk_scatter(mbp_workspace* ws, const uint8_t* noisy, const uint8_t* syn, const double* e,
                                int e_stride, int B, uint8_t* corrected, uint8_t* conv, int* iters, int* mism,
                                cudaStream_t s)
{
    const mbp_ensemble* ens = ws->ens;
    const int G = (B + 31) / 32, F = G * 32;
    const long long nb = (ens->n + 7) / 8, mb = (ens->m + 7) / 8;
    const mbp_decoder_config& cfg = ws->cfg;
    const int Dm = ens->Ds;
    int rc;
    // tables are laid out with the chunk's own frame stride F = 32 G
    if ((rc = reset_chunk_state(ws, F, s, true))) return rc;
    mbp::scatter_setup_kernel<<<(F + 127) / 128, 128, 0, s>>>(e, e_stride, B, F, Dm, (double)(float)cfg.llr_clamp,
                                                               ws->Lmag.as<float>(), ws->sc_Mtab.as<float>(),
                                                               ws->sc_Lmax.as<float>());
    MBP_CUDA(cudaGetLastError());
    if ((rc = launch_rows_to_words(noisy, nb, B, G, 1, ens->n, nb, ws->noisy_w.as<unsigned>(),
                                   ws->hard_w.as<unsigned>(), ens->n, s)))
        return rc;
    if ((rc = launch_rows_to_words(syn, (long long)ens->u * mb, B, G, ens->u, ens->m, mb,
                                   ws->syn_w.as<unsigned>(), nullptr, ens->C, s)))
        return rc;
    const bool record = (cfg.flags & MBP_RECORD_HISTORY) != 0;
    if (record)
        MBP_CUDA(cudaMemcpyAsync(ws->hist_w.p, ws->noisy_w.p, (size_t)G * ens->n * 4, cudaMemcpyDeviceToDevice, s));
    if (cfg.flags & MBP_KEEP_STATE) {
        // slot 0 holds the prior (+L in the noisy-relative domain) for frames
        // that stop at iteration 0
        fill_rel_prior_kernel<<<1024, 256, 0, s>>>(ws->Lmag.as<float>(), G, ens->n, ws->sc_vb.as<float>());
        MBP_CUDA(cudaGetLastError());
    }
    mbp::ScatterArgs A;
    std::memset(&A, 0, sizeof A);
    A.n = ens->n; A.m = ens->m; A.u = ens->u; A.C = ens->C; A.Ds = ens->Ds;
    A.slots = (long long)ens->C * ens->Ds;
    A.deg = ens->deg.as<uint8_t>(); A.chk_ell = ens->chk_ell.as<int>();
    A.var_ptr = ens->var_ptr.as<int>(); A.var_chk = ens->var_chk.as<int>();
    A.dv_max = ens->dmax_v; A.var_ptr_regular = ens->dv_reg == ens->dmax_v; A.Dm = Dm;
    A.G = G; A.B = B;
    A.vb = ws->sc_vb.as<float>(); A.c2v = ws->c2v.as<float>();
    A.Lmag = ws->Lmag.as<float>(); A.Mtab = ws->sc_Mtab.as<float>();
    A.Lfix = ws->sc_Lfix.as<int>(); A.Mfix = ws->sc_Mfix.as<int>();
    A.noisy_w = ws->noisy_w.as<unsigned>(); A.syn_w = ws->syn_w.as<unsigned>(); A.mis_w = ws->sc_mis.as<unsigned>();
    A.hard_w = ws->hard_w.as<unsigned>(); A.hist_w = record ? ws->hist_w.as<unsigned>() : nullptr;
    A.cnt = ws->cnt.as<int>();
    A.Gb = G >= 2 ? std::min(ws->Gb, (G + 1) / 2) : 0;
    A.vb_b = ws->sc_vb_b.as<float>(); A.c2v_b = ws->c2v_b.as<float>();
    A.Mtab_b = ws->sc_Mtab_b.as<float>(); A.Lfix_b = ws->sc_Lfix_b.as<int>();
    A.noisy_b = ws->noisy_b.as<unsigned>(); A.syn_b = ws->syn_b.as<unsigned>(); A.mis_b = ws->sc_mis_b.as<unsigned>();
    A.hard_b = ws->hard_b.as<unsigned>(); A.cnt_b = ws->cnt_b.as<int>(); A.fid_b = ws->fid_b.as<int>();
    A.src_b = ws->src_b.as<int>(); A.newslot = ws->newslot.as<int>(); A.grp_cnt = ws->grp_cnt.as<int>();
    A.ctrl = ws->ctrl.as<int>();
    A.any_bad = ws->any_bad.as<int>(); A.iters = ws->iters.as<int>();
    A.barrier = ws->barrier.as<unsigned>(); A.work = ws->work.as<unsigned>(); A.sweeps_run = ws->sweeps.as<int>();
    A.ts = ws->ts_cap ? ws->ts.as<unsigned long long>() : nullptr; A.ts_cap = ws->ts_cap;
    if (ws->ts_cap)   // compaction stamps are written only when a compaction happens
        MBP_CUDA(cudaMemsetAsync(ws->ts.as<unsigned long long>() + ws->ts_cap - 4, 0, 32, s));
    A.Lmax = ws->sc_Lmax.as<float>();
    A.out_conv = conv; A.out_iters = iters; A.out_mism = mism;
    // the scatter kernel works in log2 units (scatter.cuh)
    A.max_it = cfg.max_iterations;
    A.clamp = (float)((double)(float)cfg.llr_clamp * 1.4426950408889634074);
    A.sat = (float)((double)ens->sat * 1.4426950408889634074);
    if ((rc = dispatch_scatter(ws, A, s))) return rc;
    if ((rc = launch_words_to_rows(ws->hard_w.as<unsigned>(), ens->n, B, G, 1, ens->n, nb, corrected, nb, s)))
        return rc;
    ws->last_B = B;
    return MBP_OK;
}

template <class Real>
static int decode_chunk(mbp_workspace* ws, const uint8_t* noisy, const uint8_t* syn, const double* e,
                        int e_stride, int B, uint8_t* corrected, uint8_t* conv, int* iters, int* mism,
                        cudaStream_t s)
{
    const mbp_ensemble* ens = ws->ens;
    const int G = (B + 31) / 32, F = G * 32;
    const long long nb = (ens->n + 7) / 8, mb = (ens->m + 7) / 8;
    const mbp_decoder_config& cfg = ws->cfg;
    int rc;
    if (sizeof(Real) == 4 && ws->scatter)
        return decode_chunk_scatter(ws, noisy, syn, e, e_stride, B, corrected, conv, iters, mism, s);
    mbp::prior_kernel<Real><<<(F + 255) / 256, 256, 0, s>>>(e, e_stride, B, F, ws->Lmag.as<Real>());
    MBP_CUDA(cudaGetLastError());
    if ((rc = launch_rows_to_words(noisy, nb, B, G, 1, ens->n, nb, ws->noisy_w.as<unsigned>(),
                                   ws->hard_w.as<unsigned>(), ens->n, s)))
        return rc;
    if ((rc = launch_rows_to_words(syn, (long long)ens->u * mb, B, G, ens->u, ens->m, mb,
                                   ws->syn_w.as<unsigned>(), nullptr, ens->C, s)))
        return rc;
    const bool record = (cfg.flags & MBP_RECORD_HISTORY) != 0;
    if (record)
        MBP_CUDA(cudaMemcpyAsync(ws->hist_w.p, ws->noisy_w.p, (size_t)G * ens->n * 4, cudaMemcpyDeviceToDevice, s));
    if (cfg.flags & MBP_KEEP_STATE) {
        const int P = cfg.combining_mode == MBP_ISOLATED_PER_MATRIX ? ens->u + 1 : 1;
        fill_post_prior_kernel<Real><<<1024, 256, 0, s>>>(ws->noisy_w.as<unsigned>(), ws->Lmag.as<Real>(), G,
                                                          ens->n, P, ws->post.as<Real>());
        MBP_CUDA(cudaGetLastError());
        MBP_CUDA(cudaMemsetAsync(ws->c2v.p, 0, (size_t)G * ens->C * ens->Ds * 32 * sizeof(Real), s));
    }
    if ((rc = reset_chunk_state(ws, F, s, false))) return rc;

    mbp::DecodeArgs<Real> A;
    std::memset(&A, 0, sizeof A);
    A.n = ens->n; A.m = ens->m; A.u = ens->u; A.C = ens->C;
    A.Ds = ens->Ds;
    A.slots = (long long)ens->C * ens->Ds;
    A.deg = ens->deg.as<uint8_t>(); A.chk_ell = ens->chk_ell.as<int>();
    A.var_ptr = ens->var_ptr.as<int>(); A.var_edge = ens->var_slot.as<int>();
    A.dv = ens->dv_reg;
    for (int l = 0; l <= ens->u; ++l) A.edge_off[l] = (long long)l * ens->m * ens->Ds;
    A.G = G;
    A.c2v = ws->c2v.as<Real>(); A.post = ws->post.as<Real>(); A.v2c = ws->v2c.as<Real>();
    A.Lmag = ws->Lmag.as<Real>();
    A.noisy_w = ws->noisy_w.as<unsigned>(); A.syn_w = ws->syn_w.as<unsigned>();
    A.hard_w = ws->hard_w.as<unsigned>(); A.hist_w = record ? ws->hist_w.as<unsigned>() : nullptr;
    A.cnt = ws->cnt.as<int>(); A.any_bad = ws->any_bad.as<int>(); A.iters = ws->iters.as<int>();
    // compaction only pays when the chunk has at least two groups
    A.Gb = G >= 2 ? std::min(ws->Gb, (G + 1) / 2) : 0;
    A.c2v_b = ws->c2v_b.as<Real>(); A.post_b = ws->post_b.as<Real>(); A.v2c_b = ws->v2c_b.as<Real>();
    A.Lmag_b = ws->Lmag_b.as<Real>(); A.noisy_b = ws->noisy_b.as<unsigned>(); A.syn_b = ws->syn_b.as<unsigned>();
    A.hard_b = ws->hard_b.as<unsigned>(); A.cnt_b = ws->cnt_b.as<int>(); A.fid_b = ws->fid_b.as<int>();
    A.src_b = ws->src_b.as<int>(); A.newslot = ws->newslot.as<int>(); A.grp_cnt = ws->grp_cnt.as<int>();
    A.ctrl = ws->ctrl.as<int>();
    A.barrier = ws->barrier.as<unsigned>(); A.work = ws->work.as<unsigned>(); A.sweeps_run = ws->sweeps.as<int>();
    A.ts = ws->ts_cap ? ws->ts.as<unsigned long long>() : nullptr; A.ts_cap = ws->ts_cap;
    if (ws->ts_cap)   // compaction stamps are written only when a compaction happens
        MBP_CUDA(cudaMemsetAsync(ws->ts.as<unsigned long long>() + ws->ts_cap - 4, 0, 32, s));
    A.B = B; A.out_conv = conv; A.out_iters = iters; A.out_mism = mism;
    A.max_it = cfg.max_iterations; A.clamp = (Real)cfg.llr_clamp; A.damping = (Real)cfg.damping;
    A.sat = ens->sat;
    if (A.Ds < 1 || A.slots < A.C) return fail(MBP_EINVAL, "internal: bad ELL stride");
    if ((rc = dispatch_decode<Real>(ws, A, s))) return rc;
    if ((rc = launch_words_to_rows(ws->hard_w.as<unsigned>(), ens->n, B, G, 1, ens->n, nb, corrected, nb, s)))
        return rc;
    ws->last_B = B;
    return MBP_OK;
}

int mbp_decode_batch_device(mbp_workspace* ws, const uint8_t* noisy, const uint8_t* syn, const double* e,
                            int32_t e_stride, int64_t batch, uint8_t* corrected, uint8_t* converged,
                            int32_t* iterations, int32_t* mismatches, void* stream)
{
    if (!ws || !noisy || !syn || !e || !corrected || !converged || !iterations || !mismatches)
        return fail(MBP_EINVAL, "null pointer argument");
    if (batch < 0) return fail(MBP_EINVAL, "negative batch");
    if (e_stride != 0 && e_stride != 1) return fail(MBP_EINVAL, "e_stride must be 0 or 1");
    if (batch == 0) return MBP_OK;
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    cudaStream_t s = (cudaStream_t)stream;
    const long long nb = (ens->n + 7) / 8, sb = (long long)ens->u * ((ens->m + 7) / 8);
    for (int64_t off = 0; off < batch; off += ws->cap) {
        const int B = (int)std::min<int64_t>(ws->cap, batch - off);
        int rc = ws->real_size == 8
            ? decode_chunk<double>(ws, noisy + off * nb, syn + off * sb, e + off * e_stride, e_stride, B,
                                   corrected + off * nb, converged + off, iterations + off, mismatches + off, s)
            : decode_chunk<float>(ws, noisy + off * nb, syn + off * sb, e + off * e_stride, e_stride, B,
                                  corrected + off * nb, converged + off, iterations + off, mismatches + off, s);
        if (rc) return rc;
    }
    return MBP_OK;
}

// host-buffer variant: stage through the workspace's device scratch
static int ensure(DevBuf& b, size_t bytes)
{
    return b.bytes >= bytes ? MBP_OK : b.alloc(bytes);
}

// Host-buffer path.
//
// Streams (batch > workspace capacity): the batch is decoded in chunks of
// `cap` frames through a two-slot device staging ring.  Chunk c's H2D copy
// (h2d_stream) overlaps chunk c-1's decode (workspace stream) and chunk
// c-2's D2H copy (d2h_stream): the decode kernel owns every SM, the copies
// only the copy engines, so a long stream runs at the decode rate.
//
// Single batches (batch <= cap) may be split into sub-batches that overlap
// the same way (MBP_HOST_SUBBATCHES; by default only above 1024 frames: the
// decode kernel's efficiency falls below ~1024 frames per launch).  The
// diagnostic modes (kept state, decision history, phase stamps) read the
// last decode's buffers, so they decode a batch as one piece.
static bool diagnostic(const mbp_workspace* ws)
{
    return (ws->cfg.flags & (MBP_KEEP_STATE | MBP_RECORD_HISTORY | MBP_PROFILE_PHASES)) != 0;
}

static int host_subbatches(const mbp_workspace* ws, int64_t batch)
{
    if (diagnostic(ws)) return 1;
    if (const char* v = std::getenv("MBP_HOST_SUBBATCHES"))
        return (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)std::atoi(v), mbp_workspace::kMaxSub, batch / 32}));
    return (int)std::max<int64_t>(1, std::min<int64_t>(mbp_workspace::kMaxSub, batch / 1024));
}

// e (1 or batch values) copied into the workspace's pinned staging buffer
static int stage_e(mbp_workspace* ws, const double* e, size_t ne, const double** staged)
{
    if (ws->e_host_cap < ne) {
        // the previous staging may still feed an in-flight copy of this workspace
        MBP_CUDA(cudaStreamSynchronize(ws->h2d_stream));
        if (ws->e_host) cudaFreeHost(ws->e_host);
        ws->e_host = nullptr;
        ws->e_host_cap = 0;
        MBP_CUDA(cudaHostAlloc((void**)&ws->e_host, std::max<size_t>(ne, 1024) * 8, cudaHostAllocPortable));
        ws->e_host_cap = std::max<size_t>(ne, 1024);
    } else {
        MBP_CUDA(cudaStreamSynchronize(ws->h2d_stream));
    }
    std::memcpy(ws->e_host, e, ne * 8);
    *staged = ws->e_host;
    return MBP_OK;
}

static int decode_host_stream(mbp_workspace* ws, const uint8_t* noisy, const uint8_t* syn, const double* e,
                              int32_t e_stride, int64_t batch, uint8_t* corrected, uint8_t* converged,
                              int32_t* iterations, int32_t* mismatches)
{
    const mbp_ensemble* ens = ws->ens;
    cudaStream_t s = ws->own_stream;
    const size_t nb = (ens->n + 7) / 8, sb = (size_t)ens->u * ((ens->m + 7) / 8);
    const int64_t cap = ws->cap;
    const size_t ne = e_stride ? (size_t)cap : 1;
    int rc;
    if ((rc = ensure(ws->tmp_in, 2 * cap * (nb + sb))) || (rc = ensure(ws->tmp_out, 2 * cap * nb)) ||
        (rc = ensure(ws->tmp_conv, 2 * cap)) || (rc = ensure(ws->tmp_iters, 2 * cap * 4)) ||
        (rc = ensure(ws->tmp_mism, 2 * cap * 4)) || (rc = ensure(ws->tmp_e, 2 * ne * 8)))
        return rc;
    if ((rc = stage_e(ws, e, e_stride ? (size_t)batch : 1, &e))) return rc;
    MBP_CUDA(cudaEventRecord(ws->ev2, s));
    MBP_CUDA(cudaStreamWaitEvent(ws->h2d_stream, ws->ev2, 0));
    MBP_CUDA(cudaStreamWaitEvent(ws->d2h_stream, ws->ev2, 0));
    const int64_t chunks = (batch + cap - 1) / cap;
    for (int64_t c = 0; c < chunks; ++c) {
        const int k = (int)(c & 1);
        const int64_t a = c * cap, n = std::min<int64_t>(cap, batch - a);
        uint8_t* in_noisy = ws->tmp_in.as<uint8_t>() + k * cap * (nb + sb);
        uint8_t* in_syn = in_noisy + cap * nb;
        double* in_e = ws->tmp_e.as<double>() + k * ne;
        uint8_t* out_rows = ws->tmp_out.as<uint8_t>() + k * cap * nb;
        uint8_t* out_conv = ws->tmp_conv.as<uint8_t>() + k * cap;
        int* out_it = ws->tmp_iters.as<int>() + k * cap;
        int* out_mis = ws->tmp_mism.as<int>() + k * cap;
        // input slot k is free once chunk c-2's decode has run
        if (c >= 2) MBP_CUDA(cudaStreamWaitEvent(ws->h2d_stream, ws->ev_out[k], 0));
        MBP_CUDA(cudaMemcpyAsync(in_noisy, noisy + a * nb, n * nb, cudaMemcpyHostToDevice, ws->h2d_stream));
        MBP_CUDA(cudaMemcpyAsync(in_syn, syn + a * sb, n * sb, cudaMemcpyHostToDevice, ws->h2d_stream));
        MBP_CUDA(cudaMemcpyAsync(in_e, e + (e_stride ? a : 0), (e_stride ? n : 1) * 8, cudaMemcpyHostToDevice,
                                 ws->h2d_stream));
        MBP_CUDA(cudaEventRecord(ws->ev_in[k], ws->h2d_stream));
        MBP_CUDA(cudaStreamWaitEvent(s, ws->ev_in[k], 0));
        // output slot k is free once chunk c-2's results reached the host
        if (c >= 2) MBP_CUDA(cudaStreamWaitEvent(s, ws->ev_fin[k], 0));
        if ((rc = mbp_decode_batch_device(ws, in_noisy, in_syn, in_e, e_stride, n, out_rows, out_conv, out_it,
                                          out_mis, s)))
            return rc;
        MBP_CUDA(cudaEventRecord(ws->ev_out[k], s));
        MBP_CUDA(cudaStreamWaitEvent(ws->d2h_stream, ws->ev_out[k], 0));
        MBP_CUDA(cudaMemcpyAsync(corrected + a * nb, out_rows, n * nb, cudaMemcpyDeviceToHost, ws->d2h_stream));
        MBP_CUDA(cudaMemcpyAsync(converged + a, out_conv, n, cudaMemcpyDeviceToHost, ws->d2h_stream));
        MBP_CUDA(cudaMemcpyAsync(iterations + a, out_it, n * 4, cudaMemcpyDeviceToHost, ws->d2h_stream));
        MBP_CUDA(cudaMemcpyAsync(mismatches + a, out_mis, n * 4, cudaMemcpyDeviceToHost, ws->d2h_stream));
        MBP_CUDA(cudaEventRecord(ws->ev_fin[k], ws->d2h_stream));
    }
    MBP_CUDA(cudaEventRecord(ws->ev_d2h, ws->d2h_stream));
    MBP_CUDA(cudaStreamWaitEvent(s, ws->ev_d2h, 0));
    MBP_CUDA(cudaEventRecord(ws->ev3, s));
    MBP_CUDA(cudaStreamSynchronize(s));
    ws->e2e_timed = true;
    return MBP_OK;
}

int mbp_decode_batch(mbp_workspace* ws, const uint8_t* noisy, const uint8_t* syn, const double* e,
                     int32_t e_stride, int64_t batch, uint8_t* corrected, uint8_t* converged,
                     int32_t* iterations, int32_t* mismatches)
{
    if (!ws || !noisy || !syn || !e || !corrected || !converged || !iterations || !mismatches)
        return fail(MBP_EINVAL, "null pointer argument");
    if (e_stride != 0 && e_stride != 1) return fail(MBP_EINVAL, "e_stride must be 0 or 1");
    if (batch <= 0) return batch == 0 ? MBP_OK : fail(MBP_EINVAL, "negative batch");
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    if (batch > ws->cap && !diagnostic(ws))
        return decode_host_stream(ws, noisy, syn, e, e_stride, batch, corrected, converged, iterations, mismatches);
    cudaStream_t s = ws->own_stream;
    const size_t nb = (ens->n + 7) / 8, sb = (size_t)ens->u * ((ens->m + 7) / 8);
    const size_t ne = e_stride ? (size_t)batch : 1;
    int rc;
    if ((rc = ensure(ws->tmp_in, batch * (nb + sb))) || (rc = ensure(ws->tmp_out, batch * nb)) ||
        (rc = ensure(ws->tmp_conv, batch)) || (rc = ensure(ws->tmp_iters, batch * 4)) ||
        (rc = ensure(ws->tmp_mism, batch * 4)) || (rc = ensure(ws->tmp_e, ne * 8)))
        return rc;
    if ((rc = stage_e(ws, e, ne, &e))) return rc;
    uint8_t* d_noisy = ws->tmp_in.as<uint8_t>();
    uint8_t* d_syn = d_noisy + batch * nb;
    const int nsub = host_subbatches(ws, batch);
    // sub-batch k = frames [off[k], off[k+1]), offsets multiples of 32
    int64_t off[mbp_workspace::kMaxSub + 1];
    const int64_t per = ((batch + nsub - 1) / nsub + 31) / 32 * 32;
    for (int k = 0; k <= nsub; ++k) off[k] = std::min<int64_t>(batch, per * k);
    MBP_CUDA(cudaEventRecord(ws->ev2, s));
    MBP_CUDA(cudaStreamWaitEvent(ws->h2d_stream, ws->ev2, 0));
    MBP_CUDA(cudaStreamWaitEvent(ws->d2h_stream, ws->ev2, 0));
    MBP_CUDA(cudaMemcpyAsync(ws->tmp_e.p, e, ne * 8, cudaMemcpyHostToDevice, ws->h2d_stream));
    for (int k = 0; k < nsub; ++k) {
        const int64_t a = off[k], n = off[k + 1] - off[k];
        if (n <= 0) continue;
        MBP_CUDA(cudaMemcpyAsync(d_noisy + a * nb, noisy + a * nb, n * nb, cudaMemcpyHostToDevice, ws->h2d_stream));
        MBP_CUDA(cudaMemcpyAsync(d_syn + a * sb, syn + a * sb, n * sb, cudaMemcpyHostToDevice, ws->h2d_stream));
        MBP_CUDA(cudaEventRecord(ws->ev_in[k], ws->h2d_stream));
    }
    for (int k = 0; k < nsub; ++k) {
        const int64_t a = off[k], n = off[k + 1] - off[k];
        if (n <= 0) continue;
        MBP_CUDA(cudaStreamWaitEvent(s, ws->ev_in[k], 0));
        if ((rc = mbp_decode_batch_device(ws, d_noisy + a * nb, d_syn + a * sb,
                                          ws->tmp_e.as<double>() + (e_stride ? a : 0), e_stride, n,
                                          ws->tmp_out.as<uint8_t>() + a * nb, ws->tmp_conv.as<uint8_t>() + a,
                                          ws->tmp_iters.as<int>() + a, ws->tmp_mism.as<int>() + a, s)))
            return rc;
        MBP_CUDA(cudaEventRecord(ws->ev_out[k], s));
        MBP_CUDA(cudaStreamWaitEvent(ws->d2h_stream, ws->ev_out[k], 0));
        MBP_CUDA(cudaMemcpyAsync(corrected + a * nb, ws->tmp_out.as<uint8_t>() + a * nb, n * nb,
                                 cudaMemcpyDeviceToHost, ws->d2h_stream));
        MBP_CUDA(cudaMemcpyAsync(converged + a, ws->tmp_conv.as<uint8_t>() + a, n, cudaMemcpyDeviceToHost,
                                 ws->d2h_stream));
        MBP_CUDA(cudaMemcpyAsync(iterations + a, ws->tmp_iters.as<int>() + a, n * 4, cudaMemcpyDeviceToHost,
                                 ws->d2h_stream));
        MBP_CUDA(cudaMemcpyAsync(mismatches + a, ws->tmp_mism.as<int>() + a, n * 4, cudaMemcpyDeviceToHost,
                                 ws->d2h_stream));
    }
    MBP_CUDA(cudaEventRecord(ws->ev_d2h, ws->d2h_stream));
    MBP_CUDA(cudaStreamWaitEvent(s, ws->ev_d2h, 0));
    MBP_CUDA(cudaEventRecord(ws->ev3, s));
    MBP_CUDA(cudaStreamSynchronize(s));
    ws->e2e_timed = true;
    return MBP_OK;
}

int mbp_syndrome_batch_device(mbp_workspace* ws, const uint8_t* keys, int64_t batch, uint8_t* syn, void* stream)
{
    if (!ws || !keys || !syn) return fail(MBP_EINVAL, "null pointer argument");
    if (batch < 0) return fail(MBP_EINVAL, "negative batch");
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    cudaStream_t s = (cudaStream_t)stream;
    const long long nb = (ens->n + 7) / 8, mb = (ens->m + 7) / 8, sb = (long long)ens->u * mb;
    for (int64_t off = 0; off < batch; off += ws->cap) {
        const int B = (int)std::min<int64_t>(ws->cap, batch - off);
        const int G = (B + 31) / 32;
        int rc;
        if ((rc = launch_rows_to_words(keys + off * nb, nb, B, G, 1, ens->n, nb, ws->noisy_w.as<unsigned>(),
                                       nullptr, ens->n, s)))
            return rc;
        const long long items = (long long)G * ens->C;
        mbp::syndrome_words_kernel<<<(int)std::min<long long>((items + 255) / 256, 148LL * 32), 256, 0, s>>>(
            ens->deg.as<uint8_t>(), ens->chk_ell.as<int>(), ens->Ds, ens->n, ens->C, G, ws->noisy_w.as<unsigned>(),
            ws->syn_w.as<unsigned>());
        MBP_CUDA(cudaGetLastError());
        if ((rc = launch_words_to_rows(ws->syn_w.as<unsigned>(), ens->C, B, G, ens->u, ens->m, mb,
                                       syn + off * sb, sb, s)))
            return rc;
    }
    return MBP_OK;
}

int mbp_syndrome_batch(mbp_workspace* ws, const uint8_t* keys, int64_t batch, uint8_t* syn)
{
    if (!ws || !keys || !syn) return fail(MBP_EINVAL, "null pointer argument");
    if (batch <= 0) return batch == 0 ? MBP_OK : fail(MBP_EINVAL, "negative batch");
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    cudaStream_t s = ws->own_stream;
    const size_t nb = (ens->n + 7) / 8, sb = (size_t)ens->u * ((ens->m + 7) / 8);
    int rc;
    if ((rc = ensure(ws->tmp_in, batch * nb)) || (rc = ensure(ws->tmp_out, batch * sb))) return rc;
    MBP_CUDA(cudaMemcpyAsync(ws->tmp_in.p, keys, batch * nb, cudaMemcpyHostToDevice, s));
    if ((rc = mbp_syndrome_batch_device(ws, ws->tmp_in.as<uint8_t>(), batch, ws->tmp_out.as<uint8_t>(), s)))
        return rc;
    MBP_CUDA(cudaMemcpyAsync(syn, ws->tmp_out.p, batch * sb, cudaMemcpyDeviceToHost, s));
    MBP_CUDA(cudaStreamSynchronize(s));
    return MBP_OK;
}

// ---------------------------------------------------------------------------
// state readback
// ---------------------------------------------------------------------------
// Where the last chunk left `frame`'s state: its slot in the compacted
// layout (frames still undecided when the chunk compacted, decode.cuh /
// scatter.cuh sc_compact) or -1 (primary layout, lane = frame).
static int moved_slot(mbp_workspace* ws, int64_t frame, int* slot)
{
    *slot = -1;
    if (!ws->Gb) return MBP_OK;
    int v[2] = {0, 0};
    MBP_CUDA(cudaMemcpy(v, ws->sweeps.p, 8, cudaMemcpyDeviceToHost));
    if (v[1] == 0) return MBP_OK;   // no compaction in the last chunk
    MBP_CUDA(cudaMemcpy(slot, ws->newslot.as<int>() + frame, 4, cudaMemcpyDeviceToHost));
    return MBP_OK;
}

static int read_lane(mbp_workspace* ws, const void* base, long long count, int64_t frame, double* out,
                     const int* map = nullptr)
{
    DevBuf tmp;
    int rc;
    if ((rc = tmp.alloc(count * 8))) return rc;
    const int lane = (int)(frame & 31);   // frame's lane (or compacted slot's)
    cudaStream_t s = ws->own_stream;
    if (ws->real_size == 8)
        mbp::gather_lane_kernel<double><<<(int)((count + 255) / 256), 256, 0, s>>>((const double*)base, count, lane, map, tmp.as<double>());
    else
        mbp::gather_lane_kernel<float><<<(int)((count + 255) / 256), 256, 0, s>>>((const float*)base, count, lane, map, tmp.as<double>());
    MBP_CUDA(cudaGetLastError());
    MBP_CUDA(cudaMemcpyAsync(out, tmp.p, count * 8, cudaMemcpyDeviceToHost, s));
    MBP_CUDA(cudaStreamSynchronize(s));
    return MBP_OK;
}

int mbp_workspace_read_posterior(mbp_workspace* ws, int64_t frame, double* posterior)
{
    if (!ws || !posterior) return fail(MBP_EINVAL, "null pointer argument");
    if (!(ws->cfg.flags & MBP_KEEP_STATE)) return fail(MBP_EINVAL, "workspace was not configured with MBP_KEEP_STATE");
    if (frame < 0 || frame >= ws->last_B) return fail(MBP_EINVAL, "frame outside the last batch");
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    MBP_CUDA(cudaStreamSynchronize(ws->own_stream));
    MBP_CUDA(cudaDeviceSynchronize());
    int rc, s2;
    if ((rc = moved_slot(ws, frame, &s2))) return rc;
    const size_t g = s2 >= 0 ? (size_t)s2 / 32 : frame / 32;
    const int lane = s2 >= 0 ? (s2 & 31) : (int)(frame & 31);
    if (ws->scatter) {
        // post_t lives in slot t & 1; a frame's last sweep is its converged
        // iteration (0: the prior, kept in slot 0) or max_iterations
        int it = -1;
        MBP_CUDA(cudaMemcpy(&it, ws->iters.as<int>() + frame, 4, cudaMemcpyDeviceToHost));
        const int last = it >= 0 ? it : ws->cfg.max_iterations;
        const float* vb = s2 >= 0 ? ws->sc_vb_b.as<float>() : ws->sc_vb.as<float>();
        const unsigned* nw = s2 >= 0 ? ws->noisy_b.as<unsigned>() : ws->noisy_w.as<unsigned>();
        const float* base = vb + g * ens->n * mbp::kVB + (size_t)(last & 1) * 32;
        DevBuf tmp;
        if ((rc = tmp.alloc((size_t)ens->n * 8))) return rc;
        gather_rel_post_kernel<<<(ens->n + 255) / 256, 256, 0, ws->own_stream>>>(
            base, nw + g * ens->n, ens->n, lane, tmp.as<double>());
        MBP_CUDA(cudaGetLastError());
        MBP_CUDA(cudaMemcpyAsync(posterior, tmp.p, (size_t)ens->n * 8, cudaMemcpyDeviceToHost, ws->own_stream));
        MBP_CUDA(cudaStreamSynchronize(ws->own_stream));
        return MBP_OK;
    }
    const size_t P = ws->cfg.combining_mode == MBP_ISOLATED_PER_MATRIX ? (size_t)ens->u + 1 : 1;
    const char* base = (s2 >= 0 ? ws->post_b : ws->post).as<char>() + ((g * P + (P - 1)) * ens->n * 32) * ws->real_size;
    return read_lane(ws, base, ens->n, lane, posterior);
}

int mbp_workspace_read_c2v(mbp_workspace* ws, int64_t frame, double* c2v)
{
    if (!ws || !c2v) return fail(MBP_EINVAL, "null pointer argument");
    if (!(ws->cfg.flags & MBP_KEEP_STATE)) return fail(MBP_EINVAL, "workspace was not configured with MBP_KEEP_STATE");
    if (ws->scatter)
        return fail(MBP_EINVAL, "the scatter decode path does not keep messages; configure MBP_EXPLICIT_MESSAGES");
    if (frame < 0 || frame >= ws->last_B) return fail(MBP_EINVAL, "frame outside the last batch");
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    MBP_CUDA(cudaDeviceSynchronize());
    int rc, s2;
    if ((rc = moved_slot(ws, frame, &s2))) return rc;
    const size_t g = s2 >= 0 ? (size_t)s2 / 32 : frame / 32;
    const char* base = (s2 >= 0 ? ws->c2v_b : ws->c2v).as<char>() + (g * ens->C * ens->Ds * 32) * ws->real_size;
    return read_lane(ws, base, ens->E, s2 >= 0 ? s2 : frame, c2v, ens->ref2slot.as<int>());
}

int mbp_workspace_read_v2c(mbp_workspace* ws, int64_t frame, double* v2c)
{
    if (!ws || !v2c) return fail(MBP_EINVAL, "null pointer argument");
    if (!(ws->cfg.flags & MBP_KEEP_STATE)) return fail(MBP_EINVAL, "workspace was not configured with MBP_KEEP_STATE");
    if (!ws->v2c.p) return fail(MBP_EINVAL, "workspace keeps no v2c buffer (damping == 0)");
    if (frame < 0 || frame >= ws->last_B) return fail(MBP_EINVAL, "frame outside the last batch");
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    MBP_CUDA(cudaDeviceSynchronize());
    int rc, s2;
    if ((rc = moved_slot(ws, frame, &s2))) return rc;
    const size_t g = s2 >= 0 ? (size_t)s2 / 32 : frame / 32;
    const char* base = (s2 >= 0 ? ws->v2c_b : ws->v2c).as<char>() + (g * ens->C * ens->Ds * 32) * ws->real_size;
    return read_lane(ws, base, ens->E, s2 >= 0 ? s2 : frame, v2c, ens->ref2slot.as<int>());
}

int mbp_workspace_read_history(mbp_workspace* ws, int64_t frame, int32_t rows, uint8_t* out)
{
    if (!ws || !out) return fail(MBP_EINVAL, "null pointer argument");
    if (!(ws->cfg.flags & MBP_RECORD_HISTORY)) return fail(MBP_EINVAL, "workspace was not configured with MBP_RECORD_HISTORY");
    if (frame < 0 || frame >= ws->last_B) return fail(MBP_EINVAL, "frame outside the last batch");
    if (rows < 0 || rows > ws->cfg.max_iterations + 1) return fail(MBP_EINVAL, "rows out of range");
    const mbp_ensemble* ens = ws->ens;
    DeviceGuard dg(ens->device);
    MBP_CUDA(cudaDeviceSynchronize());
    const size_t n = ens->n, nb = (n + 7) / 8, g = frame / 32;
    const int lane = (int)(frame & 31);
    std::vector<unsigned> w(n);
    for (int t = 0; t < rows; ++t) {
        MBP_CUDA(cudaMemcpy(w.data(), ws->hist_w.as<unsigned>() + ((size_t)t * ws->G + g) * n, n * 4,
                            cudaMemcpyDeviceToHost));
        uint8_t* r = out + t * nb;
        std::memset(r, 0, nb);
        for (size_t i = 0; i < n; ++i) r[i >> 3] |= (uint8_t)(((w[i] >> lane) & 1u) << (i & 7));
    }
    return MBP_OK;
}

int mbp_workspace_read_phase_times(mbp_workspace* ws, uint64_t* ns, int32_t cap, int32_t* count)
{
    if (!ws || !ns || !count) return fail(MBP_EINVAL, "null pointer argument");
    if (!ws->ts_cap) return fail(MBP_EINVAL, "workspace was not configured with MBP_PROFILE_PHASES");
    DeviceGuard dg(ws->ens->device);
    MBP_CUDA(cudaDeviceSynchronize());
    int sweeps = 0;
    MBP_CUDA(cudaMemcpy(&sweeps, ws->sweeps.p, 4, cudaMemcpyDeviceToHost));
    // stamps: start, 3 per executed sweep, the final check's barrier, end
    const int k = std::min(ws->ts_cap - 4, 3 * sweeps + 3);
    *count = k;
    MBP_CUDA(cudaMemcpy(ns, ws->ts.p, (size_t)std::min(k, cap) * 8, cudaMemcpyDeviceToHost));
    // the last 4 slots: compaction stamps (start, maps built, moved, done)
    if (cap >= k + 4) MBP_CUDA(cudaMemcpy(ns + k, ws->ts.as<char>() + (size_t)(ws->ts_cap - 4) * 8, 32, cudaMemcpyDeviceToHost));
    return MBP_OK;
}

int mbp_workspace_last_stats(mbp_workspace* ws, int32_t* sweeps, int32_t* compaction_sweep)
{
    if (!ws) return fail(MBP_EINVAL, "workspace is null");
    DeviceGuard dg(ws->ens->device);
    int v[2] = {0, 0};
    MBP_CUDA(cudaDeviceSynchronize());
    MBP_CUDA(cudaMemcpy(v, ws->sweeps.p, 8, cudaMemcpyDeviceToHost));
    if (sweeps) *sweeps = v[0];
    if (compaction_sweep) *compaction_sweep = v[1];
    return MBP_OK;
}

int mbp_workspace_last_timing(mbp_workspace* ws, float* ms, float* e2e_ms, int32_t* sweeps)
{
    if (!ws) return fail(MBP_EINVAL, "workspace is null");
    DeviceGuard dg(ws->ens->device);
    if (ms) {
        if (!ws->timed) return fail(MBP_EINVAL, "no decode has run");
        MBP_CUDA(cudaEventSynchronize(ws->ev1));
        MBP_CUDA(cudaEventElapsedTime(ms, ws->ev0, ws->ev1));
    }
    if (e2e_ms) {
        if (!ws->e2e_timed) return fail(MBP_EINVAL, "no host-buffer decode has run");
        MBP_CUDA(cudaEventSynchronize(ws->ev3));
        MBP_CUDA(cudaEventElapsedTime(e2e_ms, ws->ev2, ws->ev3));
    }
    if (sweeps) MBP_CUDA(cudaMemcpy(sweeps, ws->sweeps.p, 4, cudaMemcpyDeviceToHost));
    return MBP_OK;
}

// ---------------------------------------------------------------------------
// single phases (c2v_update / v2c_update / soft_decision)
// ---------------------------------------------------------------------------
template <class Real>
static int phase_c2v(mbp_ensemble* ens, int l, const uint8_t* syn_bits, double clamp, const double* v2c, double* c2v)
{
    const size_t E = ens->E;
    std::vector<Real> hv(E), hc(E);
    for (size_t k = 0; k < E; ++k) { hv[k] = (Real)v2c[k]; hc[k] = (Real)c2v[k]; }
    DevBuf dv, dc, ds;
    int rc;
    if ((rc = dv.alloc(E * sizeof(Real))) || (rc = dc.alloc(E * sizeof(Real))) || (rc = ds.alloc(ens->m))) return rc;
    MBP_CUDA(cudaMemcpyAsync(dv.p, hv.data(), E * sizeof(Real), cudaMemcpyHostToDevice, ens->op_stream));
    MBP_CUDA(cudaMemcpyAsync(dc.p, hc.data(), E * sizeof(Real), cudaMemcpyHostToDevice, ens->op_stream));
    MBP_CUDA(cudaMemcpyAsync(ds.p, syn_bits, ens->m, cudaMemcpyHostToDevice, ens->op_stream));
    const int lo = l * ens->m, hi = lo + ens->m, grid = (ens->m + 127) / 128;
#define MBP_C2V(D) mbp::c2v_phase_kernel<Real, D><<<grid, 128, 0, ens->op_stream>>>(ens->chk_ptr.as<int>(), lo, hi, ds.as<uint8_t>(), (Real)clamp, ens->sat, dv.as<Real>(), dc.as<Real>())
    switch (pick_degree(ens->dmax_c)) {
    case 8: MBP_C2V(8); break;
    case 16: MBP_C2V(16); break;
    case 32: MBP_C2V(32); break;
    case 64: MBP_C2V(64); break;
    default: return fail(MBP_EUNSUPPORTED, "check degree too large");
    }
#undef MBP_C2V
    MBP_CUDA(cudaGetLastError());
    MBP_CUDA(cudaMemcpyAsync(hc.data(), dc.p, E * sizeof(Real), cudaMemcpyDeviceToHost, ens->op_stream));
    MBP_CUDA(cudaStreamSynchronize(ens->op_stream));
    for (size_t k = 0; k < E; ++k) c2v[k] = (double)hc[k];
    return MBP_OK;
}

int mbp_c2v_pass(mbp_ensemble* ens, int32_t precision, int32_t matrix_index, const uint8_t* syn_bits,
                 double clamp, const double* v2c, double* c2v)
{
    if (!ens || !syn_bits || !v2c || !c2v) return fail(MBP_EINVAL, "null pointer argument");
    if (matrix_index < 0 || matrix_index >= ens->u) return fail(MBP_EINVAL, "matrix_index out of range");
    DeviceGuard dg(ens->device);
    return precision == MBP_FP64_TANH ? phase_c2v<double>(ens, matrix_index, syn_bits, clamp, v2c, c2v)
                                      : phase_c2v<float>(ens, matrix_index, syn_bits, clamp, v2c, c2v);
}

template <class Real>
static int phase_v2c(mbp_ensemble* ens, int l, int joint, double damping, double clamp, const double* c2v,
                     const double* priors, double* v2c)
{
    const size_t E = ens->E, n = ens->n;
    std::vector<Real> hc(E), hv(E), hp(n);
    for (size_t k = 0; k < E; ++k) { hc[k] = (Real)c2v[k]; hv[k] = (Real)v2c[k]; }
    for (size_t k = 0; k < n; ++k) hp[k] = (Real)priors[k];
    DevBuf dc, dv, dp;
    int rc;
    if ((rc = dc.alloc(E * sizeof(Real))) || (rc = dv.alloc(E * sizeof(Real))) || (rc = dp.alloc(n * sizeof(Real)))) return rc;
    MBP_CUDA(cudaMemcpyAsync(dc.p, hc.data(), E * sizeof(Real), cudaMemcpyHostToDevice, ens->op_stream));
    MBP_CUDA(cudaMemcpyAsync(dv.p, hv.data(), E * sizeof(Real), cudaMemcpyHostToDevice, ens->op_stream));
    MBP_CUDA(cudaMemcpyAsync(dp.p, hp.data(), n * sizeof(Real), cudaMemcpyHostToDevice, ens->op_stream));
    mbp::v2c_phase_kernel<Real><<<(int)((n + 127) / 128), 128, 0, ens->op_stream>>>(
        ens->var_ptr.as<int>(), ens->var_edge.as<int>(), (int)n, (int)ens->edge_off[l], (int)ens->edge_off[l + 1],
        joint, (Real)damping, (Real)clamp, dc.as<Real>(), dp.as<Real>(), dv.as<Real>());
    MBP_CUDA(cudaGetLastError());
    MBP_CUDA(cudaMemcpyAsync(hv.data(), dv.p, E * sizeof(Real), cudaMemcpyDeviceToHost, ens->op_stream));
    MBP_CUDA(cudaStreamSynchronize(ens->op_stream));
    for (size_t k = 0; k < E; ++k) v2c[k] = (double)hv[k];
    return MBP_OK;
}

int mbp_v2c_pass(mbp_ensemble* ens, int32_t precision, int32_t matrix_index, int32_t joint, double damping,
                 double clamp, const double* c2v, const double* priors, double* v2c)
{
    if (!ens || !c2v || !priors || !v2c) return fail(MBP_EINVAL, "null pointer argument");
    if (matrix_index < 0 || matrix_index >= ens->u) return fail(MBP_EINVAL, "matrix_index out of range");
    DeviceGuard dg(ens->device);
    return precision == MBP_FP64_TANH ? phase_v2c<double>(ens, matrix_index, joint, damping, clamp, c2v, priors, v2c)
                                      : phase_v2c<float>(ens, matrix_index, joint, damping, clamp, c2v, priors, v2c);
}

template <class Real>
static int phase_post(mbp_ensemble* ens, const double* c2v, const double* priors, double* post)
{
    const size_t E = ens->E, n = ens->n;
    std::vector<Real> hc(E), hp(n), ho(n);
    for (size_t k = 0; k < E; ++k) hc[k] = (Real)c2v[k];
    for (size_t k = 0; k < n; ++k) hp[k] = (Real)priors[k];
    DevBuf dc, dp, dout;
    int rc;
    if ((rc = dc.alloc(E * sizeof(Real))) || (rc = dp.alloc(n * sizeof(Real))) || (rc = dout.alloc(n * sizeof(Real)))) return rc;
    MBP_CUDA(cudaMemcpyAsync(dc.p, hc.data(), E * sizeof(Real), cudaMemcpyHostToDevice, ens->op_stream));
    MBP_CUDA(cudaMemcpyAsync(dp.p, hp.data(), n * sizeof(Real), cudaMemcpyHostToDevice, ens->op_stream));
    mbp::posterior_phase_kernel<Real><<<(int)((n + 127) / 128), 128, 0, ens->op_stream>>>(ens->var_ptr.as<int>(), ens->var_edge.as<int>(),
                                                                       (int)n, dc.as<Real>(), dp.as<Real>(), dout.as<Real>());
    MBP_CUDA(cudaGetLastError());
    MBP_CUDA(cudaMemcpyAsync(ho.data(), dout.p, n * sizeof(Real), cudaMemcpyDeviceToHost, ens->op_stream));
    MBP_CUDA(cudaStreamSynchronize(ens->op_stream));
    for (size_t k = 0; k < n; ++k) post[k] = (double)ho[k];
    return MBP_OK;
}

int mbp_posterior_pass(mbp_ensemble* ens, int32_t precision, const double* c2v, const double* priors, double* posterior)
{
    if (!ens || !c2v || !priors || !posterior) return fail(MBP_EINVAL, "null pointer argument");
    DeviceGuard dg(ens->device);
    return precision == MBP_FP64_TANH ? phase_post<double>(ens, c2v, priors, posterior)
                                      : phase_post<float>(ens, c2v, priors, posterior);
}

void* mbp_host_alloc(size_t bytes)
{
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        g_last_error = "cudaHostAlloc failed";
        return nullptr;
    }
    return p;
}

void mbp_host_free(void* p)
{
    if (p) cudaFreeHost(p);
}

