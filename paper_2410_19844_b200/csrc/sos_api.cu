// sos_api.cu -- the C ABI declared in include/sos_b200.h (host side).
// Argument checking, device memory ownership, launch sequencing.  Every
// arithmetic step of the path runs in the kernels of sos_index.cu,
// sos_pointwise.cu and sos_gemmq.cu; there is no host or CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstddef>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/sos_b200.h"
#include "sos_internal.cuh"

using namespace sos;

struct sos_index {
    Index ix;
};
struct sos_plan {
    Plan P;
};

static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return fail(SOS_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

static int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SOS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return SOS_OK;
}

static int require_device(int* num_sms) {
    int dev = 0, count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(SOS_ERR_DEVICE, "no CUDA device");
    }
    CK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) return fail(SOS_ERR_DEVICE, "device %s is sm_%d%d, need sm_100", prop.name, prop.major, prop.minor);
    if (num_sms) *num_sms = prop.multiProcessorCount;
    return SOS_OK;
}

static uint64_t binom_u64(int x, int k) {
    if (k < 0 || k > x) return 0;
    unsigned __int128 c = 1;
    for (int t = 1; t <= k; ++t) {
        c = c * (unsigned)(x - k + t) / (unsigned)t;
        if (c > (unsigned __int128)UINT64_MAX) return UINT64_MAX;
    }
    return (uint64_t)c;
}

#ifdef SOS_EXPERIMENTS
// Experiment build only: every device allocation of the library sits between
// two kGuardBytes margins of 0xFF bytes (NaN as fp32, so a read past a float
// buffer poisons the result it feeds); sos_exp_check_guards() reports the
// allocations whose margins changed, i.e. writes past plan- or index-owned
// scratch (tests/test_gpu_guard.py).  The shipped library allocates plainly.
constexpr size_t kGuardBytes = 1 << 16;  // keeps cudaMalloc's 256-byte alignment
struct GuardRec { char* base; size_t bytes; };
static std::mutex g_guard_mu;
static std::map<void*, GuardRec> g_guards;
#endif

template <class T>
static int dalloc(T** p, size_t bytes) {
#ifdef SOS_EXPERIMENTS
    char* base = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuardBytes) != cudaSuccess ||
        cudaMemset(base, 0xFF, bytes + 2 * kGuardBytes) != cudaSuccess) {
        cudaGetLastError();
        if (base) cudaFree(base);
        *p = nullptr;
        return fail(SOS_ERR_NOMEM, "cudaMalloc(%zu) failed", bytes);
    }
    *p = reinterpret_cast<T*>(base + kGuardBytes);
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guards[*p] = GuardRec{base, bytes};
    return SOS_OK;
#else
    if (cudaMalloc(reinterpret_cast<void**>(p), bytes) != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return fail(SOS_ERR_NOMEM, "cudaMalloc(%zu) failed", bytes);
    }
    return SOS_OK;
#endif
}

// frees what dalloc returned (nullptr is fine)
static void dfree(void* p) {
#ifdef SOS_EXPERIMENTS
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_guard_mu);
    auto it = g_guards.find(p);
    if (it == g_guards.end()) return;
    cudaFree(it->second.base);
    g_guards.erase(it);
#else
    cudaFree(p);
#endif
}

extern "C" {

const char* sos_last_error(void) { return g_err; }
int sos_version(void) { return 2; }

// ------------------------------------------------------------------ index --
int sos_build_index(int n, int d, sos_index** out) {
    if (!out) return fail(SOS_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (n < 1 || d < 1 || 2 * d > kMaxDeg2 || n + 2 * d > kMaxVars)
        return fail(SOS_ERR_ARG, "need n>=1, 1<=d<=%d, n+2d<=%d", kMaxDeg2 / 2, kMaxVars);
    const uint64_t N = binom_u64(n + d - 1, d), M = binom_u64(n + 2 * d - 1, 2 * d);
    if (N > 65536) return fail(SOS_ERR_ARG, "N=%llu > 65536", (unsigned long long)N);
    if (M >= 0xFFFFFFFFull) return fail(SOS_ERR_ARG, "M=%llu does not fit uint32 ranks", (unsigned long long)M);
    int sms = 0;
    int rc = require_device(&sms);
    if (rc) return rc;

    sos_index* h = new sos_index();
    Index& ix = h->ix;
    ix.n = n;
    ix.d = d;
    ix.N = (int64_t)N;
    ix.M = (int64_t)M;
    ix.Np = ((ix.N + kPad - 1) / kPad) * kPad;
    ix.nb = n + 2 * d;
    const int bstride = 2 * d + 1;
    std::vector<uint32_t> hb((size_t)ix.nb * bstride);
    for (int x = 0; x < ix.nb; ++x)
        for (int k = 0; k < bstride; ++k) {
            uint64_t c = binom_u64(x, k);
            hb[(size_t)x * bstride + k] = c > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c;
        }
    if ((rc = dalloc(&ix.d_binom, hb.size() * 4)) || (rc = dalloc(&ix.d_ms, (size_t)ix.N * d)) ||
        (rc = dalloc(&ix.d_alpha, (size_t)ix.N * n)) ||
        (rc = dalloc(&ix.d_pt, (size_t)pt_entries(ix.Np) * 4))) {
        sos_index_destroy(h);
        return rc;
    }
    if (cudaMemcpy(ix.d_binom, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        sos_index_destroy(h);
        return fail(SOS_ERR_CUDA, "copy binomial table");
    }
    launch_index_build(ix, 0);
    if ((rc = check_launch("index build")) || (cudaDeviceSynchronize() != cudaSuccess)) {
        if (!rc) rc = fail(SOS_ERR_CUDA, "index build: %s", cudaGetErrorString(cudaGetLastError()));
        sos_index_destroy(h);
        return rc;
    }
    *out = h;
    return SOS_OK;
}

int sos_index_destroy(sos_index* h) {
    if (!h) return SOS_OK;
    dfree(h->ix.d_binom);
    dfree(h->ix.d_ms);
    dfree(h->ix.d_alpha);
    dfree(h->ix.d_pt);
    delete h;
    return SOS_OK;
}

int sos_index_dims(const sos_index* h, int64_t* N, int64_t* M) {
    if (!h) return fail(SOS_ERR_ARG, "index is NULL");
    if (N) *N = h->ix.N;
    if (M) *M = h->ix.M;
    return SOS_OK;
}

int sos_index_alpha(const sos_index* h, uint8_t* alpha_dev, void* stream) {
    if (!h || !alpha_dev) return fail(SOS_ERR_ARG, "NULL argument");
    CK(cudaMemcpyAsync(alpha_dev, h->ix.d_alpha, (size_t)h->ix.N * h->ix.n, cudaMemcpyDeviceToDevice,
                       (cudaStream_t)stream));
    return SOS_OK;
}

int sos_index_beta(const sos_index* h, uint8_t* beta_dev, void* stream) {
    if (!h || !beta_dev) return fail(SOS_ERR_ARG, "NULL argument");
    launch_beta_table(h->ix, beta_dev, (cudaStream_t)stream);
    return check_launch("beta table");
}

int sos_index_pair_ranks(const sos_index* h, const int64_t* i_dev, const int64_t* j_dev, int64_t count,
                         uint32_t* out_dev, void* stream) {
    if (!h || count < 0 || (count > 0 && (!i_dev || !j_dev || !out_dev))) return fail(SOS_ERR_ARG, "bad argument");
    launch_pair_lookup(h->ix, i_dev, j_dev, count, out_dev, (cudaStream_t)stream);
    return check_launch("pair lookup");
}

// scratch of the lattice DP for the R row maxima: degrees d+1 .. 2d-1
static size_t rlev_floats(const Index& ix) {
    size_t s = 0;
    for (int D = ix.d + 1; D <= 2 * ix.d - 1; ++D) s += (size_t)rmax_level_count(ix.n, D);
    return s;
}

// ------------------------------------------------------------------- plan --
// CTA-pair tiles: a = 256-row block, b = 160-col block, grouped raster (8 row
// blocks per group) so a wave of CTAs shares A and B panels in L2
static int64_t tile_group() {
#ifdef SOS_EXPERIMENTS
    const char* ga = getenv("SOS_TILE_GROUP");
    if (ga && atoi(ga) > 0) return atoi(ga);
#endif
    return 8;
}
// MMA N of a tile: its live columns rounded up to 16 (UMMA M = 256 takes N % 16 == 0,
// 16 <= N <= 256; each CTA then supplies N/2 B rows, whole 8-row swizzle atoms).
// Never past the next multiple of 16: the next tile may start there.
static int round_up16(int64_t x) { return (int)std::max<int64_t>(16, (x + 15) / 16 * 16); }

// forward: upper triangle of the Gram matrix (columns j >= rows' block start);
// backward: all of R V.  Columns tiled on a W grid (W = 160, or narrower for
// small problems, see pick_tile_width); see TileCoord for the narrow tiles
static void build_tiles(int64_t row_blocks, int64_t ncols, bool upper, bool narrow, int W, std::vector<TileCoord>& out) {
    const int64_t GA = tile_group();
    const int64_t col_blocks = (ncols + W - 1) / W;
    for (int64_t g0 = 0; g0 < row_blocks; g0 += GA) {
        const int64_t g1 = std::min(row_blocks, g0 + GA);
        for (int64_t b = 0; b < col_blocks; ++b)
            for (int64_t a = g0; a < g1; ++a) {
                int64_t c_start = b * W, c_end = std::min(ncols, c_start + W);
                if (upper) {
                    if (c_end <= a * kPairM) continue;              // wholly below the diagonal block
                    c_start = std::max(c_start, a * kPairM);        // skip columns left of it
                }
                if (!narrow) c_start = b * W, c_end = c_start + W;  // A/B: full grid tiles
                out.push_back(TileCoord{(int)a, (int)c_start, round_up16(c_end - c_start), 0});
            }
    }
}

// Column tile width.  A GEMM of T tiles on P CTA pairs runs ceil(T / P) waves,
// and a wave of W-wide tiles takes ~W of MMA time plus a per-wave cost that does
// not shrink with W (measured ~10 us at config 2b: 4 waves of 112 lose to 3 of
// 160).  So the plan takes the narrowest width that does not add a wave to the
// 160-wide tiling: config 2 backward 104 tiles of 160 -> 144 tiles of 112, both
// 2 waves; forward 56 tiles of 160 -> 72 of 128, both one wave; config 1 one
// wave at 160 or at 96.  The int8 pair MMA runs at full rate down to N = 128 and
// loses little at 96 (profiles/r1_mma2_pair_N_sweep.log), so widths stop at 96
// (multiples of 16: UMMA N with M = 256); only problems of at most 4 waves are
// considered (more tiles re-read their A panels more often).  A/B:
// profiles/r2_tile_width16_ab.log.  forced: sos_plan_opts.tile_w.
static int pick_tile_width(int64_t row_blocks, int64_t ncols, bool upper, bool narrow, int pairs, int forced) {
    if (forced > 0) return forced;
    auto waves = [&](int W) {
        std::vector<TileCoord> t;
        build_tiles(row_blocks, ncols, upper, narrow, W, t);
        return ((int64_t)t.size() + pairs - 1) / pairs;
    };
    const int64_t w160 = waves(kTileN);
    if (w160 > 4) return kTileN;
    int bestW = kTileN;
    for (int W = kTileN - 16; W >= 16; W -= 16)
        if (waves(W) <= w160) bestW = W;
    return bestW;
}

int sos_plan_create(const sos_index* h, int64_t r, sos_plan** out) {
    return sos_plan_create_ex(h, r, nullptr, out);
}

static bool pick(int opt, bool dflt) { return opt < 0 ? dflt : opt != 0; }

int sos_plan_create_ex(const sos_index* h, int64_t r, const sos_plan_opts* opts, sos_plan** out) {
    if (!h || !out || r < 1) return fail(SOS_ERR_ARG, "bad argument");
    sos_plan_opts o = {-1, -1, -1, -1, -1, -1, -1, -1};
    if (opts) o = *opts;
    for (int v : {o.split, o.vtq_from_update, o.vtq_in_aux, o.rmax_direct, o.narrow_tiles, o.r_headroom, o.tiny})
        if (v < -1 || v > 1) return fail(SOS_ERR_ARG, "sos_plan_opts fields must be -1, 0 or 1");
    if (!(o.tile_w == -1 || o.tile_w == 0 || (o.tile_w >= 16 && o.tile_w <= kTileN && o.tile_w % 16 == 0)))
        return fail(SOS_ERR_ARG, "sos_plan_opts.tile_w must be -1 / 0 (auto) or a multiple of 16 in [16, 160]");
    *out = nullptr;
    int sms = 0;
    int rc = require_device(&sms);
    if (rc) return rc;
    sos_plan* pl = new sos_plan();
    Plan& P = pl->P;
    P.idx = &h->ix;
    P.r = r;
    P.num_sms = sms;
    {
        int dev = 0, l2 = 0;
        cudaGetDevice(&dev);
        P.l2_bytes = cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) == cudaSuccess ? l2 : 0;
    }
    const int64_t Np = h->ix.Np, N = h->ix.N, M = h->ix.M;
    const int64_t colBlocksV = (N + kTileN - 1) / kTileN;
    P.rowsV = std::max(Np, colBlocksV * kTileN);
    P.nkbV = (r + kQK - 1) / kQK;
    P.rowsVT = ((r + kTileN - 1) / kTileN) * kTileN;
    P.nkbN = (N + kQK - 1) / kQK;  // K = j runs over the N monomials (rows stay padded to Np)
    P.narrow = pick(o.narrow_tiles, true);
    // short K: a tile's MMAs (~nkbN x 0.5 us) cannot hide the fused update
    // (~25 us per tile), so the split step stores the gradient and updates
    // with all SMs (profiles/r1_update_split_ab.log, r2_split_vs_fused_shapes.log)
    P.split = pick(o.split, P.nkbN < kSplitKb);
    {
        // the fused update assumes every tile but a matrix-edge one is 160 wide, so
        // narrower backward tiles only with the split step (gradient stored)
        const int pairs = resident_gemm_pairs(sms);
        P.tile_w_fwd = pick_tile_width(Np / kPairM, N, true, P.narrow, pairs, o.tile_w);
        P.tile_w_bwd = P.split ? pick_tile_width(Np / kPairM, r, false, P.narrow, pairs, o.tile_w) : kTileN;
    }
    std::vector<TileCoord> tf, tb;
    build_tiles(Np / kPairM, N, true, P.narrow, P.tile_w_fwd, tf);
    build_tiles(Np / kPairM, r, false, P.narrow, P.tile_w_bwd, tb);
    P.ntiles_fwd = (int)tf.size();
    P.ntiles_bwd = (int)tb.size();
    // sos_descend: the update can write the next step's V^T slices when its
    // extra slicing work hides under a tile's MMAs (long K); for short K it
    // would lengthen the update-bound backward (profiles/r1_vtq_next_ab.log)
    P.vtq_from_update = !P.split && pick(o.vtq_from_update, P.nkbN >= 128);
    P.r_headroom = !P.split && pick(o.r_headroom, true);
    P.vtq_in_aux = pick(o.vtq_in_aux, vtq_fits_aux(P));
    P.rmax_direct = pick(o.rmax_direct, rmax_direct_default(h->ix));
    if (P.split) P.mid_grid = mid_grid_for(P.nkbN, P.rowsVT, M, sms, &P.mid_tiles, &P.mid_hold_v);
    // tiny plans: the whole descent in one cooperative kernel (sos_tiny.cu) for
    // small N and r, where the split step's four launches are latency-bound
    P.tiny_grid = tiny_grid_for(sms);
    P.tiny = P.tiny_grid > 0 && pick(o.tiny, (double)N * N * r <= kTinyMaxWork);
    // row chunks of the last step's V release = the raster's row groups
    P.sig_blocks = (int)tile_group();
    P.sig_expect.assign((size_t)((Np / kPairM + P.sig_blocks - 1) / P.sig_blocks), 0u);
    for (const TileCoord& t : tb) P.sig_expect[t.a / P.sig_blocks] += 2;  // one per CTA of the pair

    if ((rc = dalloc(&P.d_vq, (size_t)kSlices * P.nkbV * P.rowsV * 64)) ||
        (rc = dalloc(&P.d_vtq, (size_t)kSlices * P.nkbN * P.rowsVT * 64)) ||
        (rc = dalloc(&P.d_rq, (size_t)kSlices * P.nkbN * Np * 64)) ||
        (rc = dalloc(&P.d_vrow, (size_t)P.rowsV * 4)) || (rc = dalloc(&P.d_vcol, (size_t)P.rowsVT * 4)) ||
        (rc = dalloc(&P.d_rrow, (size_t)Np * 4)) || (rc = dalloc(&P.d_coef, (size_t)M * 4)) ||
        (rc = dalloc(&P.d_dbuf, (size_t)(4 * P.rowsV + 4 * P.rowsVT) * 4)) ||
        (rc = dalloc(&P.d_opt, sizeof(DevOpt))) ||
        (rc = dalloc(&P.d_rlev, std::max<size_t>(1, rlev_floats(h->ix)) * sizeof(float))) ||
        (rc = dalloc(&P.d_res, (size_t)M * 4)) || (rc = dalloc(&P.d_scal, sizeof(Scalars))) ||
        (rc = dalloc(&P.d_ring, (size_t)sms * 128 * kTileN * 4)) ||
        (rc = dalloc(&P.d_progress, 2 * sizeof(unsigned long long))) ||
        (rc = dalloc(&P.d_tiles_fwd, std::max<size_t>(1, tf.size()) * sizeof(TileCoord))) ||
        (rc = dalloc(&P.d_tiles_bwd, std::max<size_t>(1, tb.size()) * sizeof(TileCoord))) ||
        (rc = dalloc(&P.d_rowsig, std::max<size_t>(1, P.sig_expect.size()) * sizeof(unsigned))) ||
        ((P.split || P.tiny) && (rc = dalloc(&P.d_grad, (size_t)N * r * sizeof(float)))) ||
        ((P.split || P.tiny) &&
         (rc = dalloc(&P.d_part, (size_t)2 * std::max({P.mid_grid, P.tiny_grid, 1}) * sizeof(double)))) ||
        (P.r_headroom && (rc = dalloc(&P.d_rrowx, (size_t)2 * Np * sizeof(unsigned)))) ||
        (P.r_headroom && (rc = dalloc(&P.d_urowr, (size_t)Np * sizeof(unsigned))))) {
        sos_plan_destroy(pl);
        return rc;
    }
    if (cudaMemcpy(P.d_tiles_fwd, tf.data(), tf.size() * sizeof(TileCoord), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(P.d_tiles_bwd, tb.data(), tb.size() * sizeof(TileCoord), cudaMemcpyHostToDevice) != cudaSuccess) {
        sos_plan_destroy(pl);
        return fail(SOS_ERR_CUDA, "tile list upload");
    }
    // zero-initialised maxima: the GEMMs read them for padding rows too
    if (cudaMemset(P.d_vrow, 0, (size_t)P.rowsV * 4) != cudaSuccess ||
        cudaMemset(P.d_vcol, 0, (size_t)P.rowsVT * 4) != cudaSuccess ||
        cudaMemset(P.d_rrow, 0, (size_t)Np * 4) != cudaSuccess ||
        cudaMemset(P.d_rq, 0, (size_t)kSlices * P.nkbN * Np * 64) != cudaSuccess ||  // padding rows stay 0
        cudaMemset(P.d_progress, 0, 2 * sizeof(unsigned long long)) != cudaSuccess ||  // GEMMs reset it themselves
        cudaMemset(P.d_dbuf, 0, (size_t)(4 * P.rowsV + 4 * P.rowsVT) * 4) != cudaSuccess ||
        cudaMemset(P.d_opt, 0, sizeof(DevOpt)) != cudaSuccess ||
        (P.r_headroom && (cudaMemset(P.d_rrowx, 0, (size_t)2 * Np * 4) != cudaSuccess ||
                          cudaMemset(P.d_urowr, 0, (size_t)Np * 4) != cudaSuccess))) {
        sos_plan_destroy(pl);
        return fail(SOS_ERR_CUDA, "workspace init");
    }
    if (!make_q_tmap(P.tmap_vq_a, P.d_vq, P.rowsV, P.nkbV, 128) ||
        !make_q_tmap(P.tmap_vq_b, P.d_vq, P.rowsV, P.nkbV, kHalfN) ||
        !make_q_tmap(P.tmap_vtq_b, P.d_vtq, P.rowsVT, P.nkbN, kHalfN) ||
        !make_q_tmap(P.tmap_rq_a, P.d_rq, Np, P.nkbN, 128)) {
        sos_plan_destroy(pl);
        return fail(SOS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    }
    P.timing = new Timing();
    P.opt_kind = SOS_OPT_GD;
    P.lr = 0.f;
    P.opt_ready = false;
    *out = pl;
    return SOS_OK;
}

int sos_plan_destroy(sos_plan* pl) {
    if (!pl) return SOS_OK;
    Plan& P = pl->P;
    dfree(P.d_vq);
    dfree(P.d_vtq);
    dfree(P.d_vtq2);
    dfree(P.d_rq);
    dfree(P.d_vrow);
    dfree(P.d_vcol);
    dfree(P.d_rrow);
    dfree(P.d_dbuf);
    dfree(P.d_opt);
    dfree(P.d_rlev);
    dfree(P.d_hV);
    dfree(P.d_hp);
    dfree(P.d_hl);
    if (P.gexec) cudaGraphExecDestroy(P.gexec);
    for (cudaGraphExec_t& g : P.gexec_long)
        if (g) cudaGraphExecDestroy(g);
    dfree(P.d_coef);
    dfree(P.d_res);
    dfree(P.d_m);
    dfree(P.d_v);
    dfree(P.d_scal);
    dfree(P.d_ring);
    dfree(P.d_progress);
    dfree(P.d_tiles_fwd);
    dfree(P.d_tiles_bwd);
    dfree(P.d_rowsig);
    dfree(P.d_grad);
    dfree(P.d_part);
    dfree(P.d_rrowx);
    dfree(P.d_urowr);
    if (P.copy_st) cudaStreamDestroy(P.copy_st);
    if (P.sig_ev) cudaEventDestroy(P.sig_ev);
    if (P.timing) {
        for (cudaEvent_t e : P.timing->pool) cudaEventDestroy(e);
        delete P.timing;
    }
    delete pl;
    return SOS_OK;
}

int64_t sos_plan_launch_count(const sos_plan* pl) { return pl ? pl->P.launches : -1; }

int sos_plan_timing(sos_plan* pl, int enable) {
    if (!pl || !pl->P.timing) return fail(SOS_ERR_ARG, "plan is NULL");
    Timing& T = *pl->P.timing;
    if (enable) {
        T.used = 0;
        T.recs.clear();
    }
    T.on = enable != 0;
    return SOS_OK;
}

int sos_plan_timing_read(sos_plan* pl, int kernel, double* total_ms, int64_t* launches) {
    if (!pl || !pl->P.timing || kernel < 0 || kernel >= KK_COUNT) return fail(SOS_ERR_ARG, "bad argument");
    double sum = 0.0;
    int64_t cnt = 0;
    for (const TimingRec& r : pl->P.timing->recs) {
        if (r.kind != kernel) continue;
        CK(cudaEventSynchronize(r.b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.a, r.b));
        sum += ms;
        cnt++;
    }
    if (total_ms) *total_ms = sum;
    if (launches) *launches = cnt;
    return SOS_OK;
}

// --------------------------------------------------------------- compute --
// forward; with_vtq also packs the V^T slices (the backward's B operand) in the
// forward GEMM's aux warps, hidden under its tensor-bound main loop
static int do_forward(Plan& P, const float* V, float* coef, bool with_vtq, cudaStream_t st) {
    CK(cudaMemsetAsync(P.d_scal, 0, sizeof(Scalars), st));
    CK(cudaMemsetAsync(coef, 0, (size_t)P.idx->M * 4, st));
    launch_pack_v(P, V, st);
    launch_gemm_fwd(P, coef, with_vtq ? V : nullptr, st);
    return check_launch("forward");
}

int sos_forward(sos_plan* pl, const float* V_dev, float* coef_dev, void* stream) {
    if (!pl || !V_dev || !coef_dev) return fail(SOS_ERR_ARG, "NULL argument");
    return do_forward(pl->P, V_dev, coef_dev, false, (cudaStream_t)stream);
}

int sos_backward(sos_plan* pl, const float* V_dev, const float* res_dev, float* grad_dev, void* stream) {
    if (!pl || !V_dev || !res_dev || !grad_dev) return fail(SOS_ERR_ARG, "NULL argument");
    Plan& P = pl->P;
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemsetAsync(P.d_scal, 0, sizeof(Scalars), st));
    launch_vmax(P, V_dev, st);
    launch_pack_vtq(P, V_dev, st);
    launch_pack_r(P, res_dev, st, 0);
    launch_gemm_bwd(P, grad_dev, st);
    return check_launch("backward");
}

static int do_loss_grad(Plan& P, const float* V, const float* p, double* loss, float* grad, float* res,
                        cudaStream_t st, bool pack_vtq_for_step = false) {
    int rc = do_forward(P, V, P.d_coef, grad != nullptr || pack_vtq_for_step, st);
    if (rc) return rc;
    float* r = res ? res : P.d_res;
    launch_residual(P, P.d_coef, p, r, st);
    if (grad) {
        launch_pack_r(P, r, st, 0);
        launch_gemm_bwd(P, grad, st);
    }
    if (loss) CK(cudaMemcpyAsync(loss, &P.d_scal->loss, sizeof(double), cudaMemcpyDeviceToDevice, st));
    return check_launch("loss_grad");
}

int sos_loss_grad(sos_plan* pl, const float* V_dev, const float* p_dev, double* loss_dev, float* grad_dev,
                  float* res_dev, void* stream) {
    if (!pl || !V_dev || !p_dev) return fail(SOS_ERR_ARG, "NULL argument");
    return do_loss_grad(pl->P, V_dev, p_dev, loss_dev, grad_dev, res_dev, (cudaStream_t)stream);
}

int sos_opt_init(sos_plan* pl, const sos_opt_params* prm, void* stream) {
    if (!pl || !prm) return fail(SOS_ERR_ARG, "NULL argument");
    if (prm->kind != SOS_OPT_GD && prm->kind != SOS_OPT_ADAM) return fail(SOS_ERR_ARG, "unknown optimiser %d", prm->kind);
    if (!(prm->lr > 0.f)) return fail(SOS_ERR_ARG, "lr must be > 0");
    Plan& P = pl->P;
    P.opt_kind = prm->kind;
    P.lr = prm->lr;
    P.b1 = prm->beta1;
    P.b2 = prm->beta2;
    P.eps = prm->eps;
    P.stop_tol = 0.0;
    if (P.gexec) {  // the captured steps bake in the optimiser kind and moment buffers
        cudaGraphExecDestroy(P.gexec);
        P.gexec = nullptr;
    }
    for (cudaGraphExec_t& g : P.gexec_long) {
        if (g) cudaGraphExecDestroy(g);
        g = nullptr;
    }
    if (prm->kind == SOS_OPT_ADAM) {
        if (!(prm->beta1 >= 0.f && prm->beta1 < 1.f && prm->beta2 >= 0.f && prm->beta2 < 1.f))
            return fail(SOS_ERR_ARG, "betas must be in [0,1)");
        const size_t bytes = (size_t)P.idx->N * P.r * 4;
        int rc;
        if (!P.d_m && ((rc = dalloc(&P.d_m, bytes)) || (rc = dalloc(&P.d_v, bytes)))) return rc;
        CK(cudaMemsetAsync(P.d_m, 0, bytes, (cudaStream_t)stream));
        CK(cudaMemsetAsync(P.d_v, 0, bytes, (cudaStream_t)stream));
    }
    CK(cudaMemsetAsync(P.d_opt, 0, sizeof(DevOpt), (cudaStream_t)stream));  // t = 0
    P.opt_ready = true;
    return SOS_OK;
}

// parameters of the optimiser as set on the host -> DevOpt (stream-ordered;
// t and loss_idx stay device-managed)
static int upload_opt(Plan& P, cudaStream_t st) {
    struct { float lr, b1, b2, eps; double stop_tol; } h{P.lr, P.b1, P.b2, P.eps, P.stop_tol};
    static_assert(sizeof(h) == offsetof(DevOpt, t), "DevOpt host-uploaded prefix");
    CK(cudaMemcpyAsync(P.d_opt, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    return SOS_OK;
}

int sos_opt_set_lr(sos_plan* pl, float lr) {
    if (!pl) return fail(SOS_ERR_ARG, "plan is NULL");
    if (!pl->P.opt_ready) return fail(SOS_ERR_ARG, "sos_opt_init not called");
    if (!(lr > 0.f)) return fail(SOS_ERR_ARG, "lr must be > 0");
    pl->P.lr = lr;
    return SOS_OK;
}

int sos_opt_set_stop(sos_plan* pl, double rel_tol) {
    if (!pl) return fail(SOS_ERR_ARG, "plan is NULL");
    if (!(rel_tol == rel_tol)) return fail(SOS_ERR_ARG, "rel_tol is NaN");
    pl->P.stop_tol = rel_tol > 0.0 ? rel_tol : 0.0;
    return SOS_OK;
}

int sos_step(sos_plan* pl, float* V_dev, const float* p_dev, double* loss_dev, void* stream) {
    if (!pl || !V_dev || !p_dev) return fail(SOS_ERR_ARG, "NULL argument");
    if (reinterpret_cast<uintptr_t>(V_dev) & 15) return fail(SOS_ERR_ARG, "V_dev must be 16-byte aligned");
    Plan& P = pl->P;
    if (!P.opt_ready) return fail(SOS_ERR_ARG, "sos_opt_init not called");
    cudaStream_t st = (cudaStream_t)stream;
    int rc = upload_opt(P, st);
    if (rc) return rc;
    if (P.split) {
        // split step: exact maxima + VQ of V, forward, k_mid (residual, loss into
        // loss_dev, R maxima, V^T and R slices), backward storing the gradient,
        // row-block update of V (no next-step slices: the next call packs V again)
        CK(cudaMemsetAsync(P.d_coef, 0, (size_t)P.idx->M * 4, st));
        launch_pack_v(P, V_dev, st, P.d_vrow, P.d_vcol);
        launch_gemm_fwd(P, P.d_coef, nullptr, st, P.d_vrow, P.d_vcol, true, true);
        launch_mid(P, p_dev, V_dev, P.d_vcol, false, nullptr, loss_dev, false, st);
        launch_gemm_bwd(P, P.d_grad, st, P.d_vcol, P.tmap_vtq_b, true);
        launch_update_rows(P, V_dev, nullptr, nullptr, nullptr, st);
        return check_launch("step");
    }
    // loss and residual of the current V, then the backward GEMM whose epilogue
    // warps apply the optimiser update to V in place, tile by tile
    rc = do_loss_grad(P, V_dev, p_dev, loss_dev, nullptr, nullptr, st, true);
    if (rc) return rc;
    launch_step_begin(P, nullptr, st);
    launch_pack_r(P, P.d_res, st, 1);
    launch_gemm_bwd_update(P, V_dev, st);
    return check_launch("step");
}

// one descent step of sos_descend on buffer parity b (see the header)
struct DescendPtrs {
    unsigned* vrowx[2];  // exact row maxima of V (current / next)
    unsigned* urow[2];   // row scales the slices in VQ were written with
    unsigned* vcol[2];   // exact column maxima of V
    unsigned* ucol[2];   // column scales the slices in VTQ[b] were written with
    uint8_t* vtq[2];     // VTQ buffers (step parity b reads vtq[b], its update writes vtq[b ^ 1])
    const uint8_t* tmap_vtq[2];
};
static DescendPtrs descend_ptrs(Plan& P) {
    DescendPtrs d;
    d.vrowx[0] = P.d_dbuf;
    d.vrowx[1] = P.d_dbuf + P.rowsV;
    d.urow[0] = P.d_dbuf + 2 * P.rowsV;
    d.urow[1] = P.d_dbuf + 3 * P.rowsV;
    d.vcol[0] = P.d_dbuf + 4 * P.rowsV;
    d.vcol[1] = P.d_dbuf + 4 * P.rowsV + P.rowsVT;
    d.ucol[0] = P.d_dbuf + 4 * P.rowsV + 2 * P.rowsVT;
    d.ucol[1] = P.d_dbuf + 4 * P.rowsV + 3 * P.rowsVT;
    d.vtq[0] = P.d_vtq;
    d.vtq[1] = P.d_vtq2;
    d.tmap_vtq[0] = P.tmap_vtq_b;
    d.tmap_vtq[1] = P.tmap_vtq2_b;
    return d;
}

// the second VTQ buffer of sos_descend, allocated on first use (zeroed: its
// K-padding rows j >= N are never written and must read as 0)
static int ensure_vtq2(Plan& P) {
    if (P.d_vtq2) return SOS_OK;
    const size_t bytes = (size_t)kSlices * P.nkbN * P.rowsVT * 64;
    int rc = dalloc(&P.d_vtq2, bytes);
    if (rc) return rc;
    if (cudaMemset(P.d_vtq2, 0, bytes) != cudaSuccess ||
        !make_q_tmap(P.tmap_vtq2_b, P.d_vtq2, P.rowsVT, P.nkbN, kHalfN)) {
        dfree(P.d_vtq2);
        P.d_vtq2 = nullptr;
        return fail(SOS_ERR_CUDA, "second VTQ buffer");
    }
    return SOS_OK;
}

static int descend_step(Plan& P, const DescendPtrs& d, int b, float* V, const float* p, double* losses,
                        cudaStream_t st, bool first = false) {
    // no memset nodes inside the replayed steps: the forward clears the loss
    // accumulators, step_begin / k_mid clear coef for the next forward and the
    // next step's maxima (the first step of a call starts from a clean coef)
    if (first) CK(cudaMemsetAsync(P.d_coef, 0, (size_t)P.idx->M * 4, st));
    if (P.split) {
        // split step (4 launches): VQ holds V_t sliced against its exact row
        // maxima vrowx[b] (the previous update, or the prologue's pack); k_mid
        // takes the column maxima of V_t into vcol[b] (cleared by the previous
        // k_mid; exact already after the prologue, where atomicMax keeps them)
        launch_gemm_fwd(P, P.d_coef, nullptr, st, d.vrowx[b], d.vcol[b], true, true);
        launch_mid(P, p, V, d.vcol[b], true, d.vcol[b ^ 1], nullptr, true, st);
        launch_gemm_bwd(P, P.d_grad, st, d.vcol[b], P.tmap_vtq_b, true);
        launch_update_rows(P, V, P.d_vq, d.vrowx[b], d.vrowx[b ^ 1], st);
        return check_launch("descend step");
    }
    const bool vu = P.vtq_from_update;
    // VTQ[b] came from the previous update; else (and in the first step of a call,
    // into VTQ[0] = P.d_vtq with the exact column maxima) the forward packs it
    launch_gemm_fwd(P, P.d_coef, vu && !first ? nullptr : V, st, d.urow[b], d.vcol[b], true);
    launch_residual(P, P.d_coef, p, P.d_res, st);
    // t += 1, losses[k] = L(V_t) (the call's array, from DevOpt); clear the next
    // maxima and the coefficient accumulator (read by the residual, done)
    // R slices: after the first step of a call with the previous step's exact R
    // row maxima (x kHeadroom, rare rows re-sliced: no DP on the step); the
    // first step computes them exactly (DP or direct pass) and keeps them
    const bool hr = P.r_headroom && !first;
    unsigned* rr_cur = P.d_rrowx + (size_t)b * P.idx->Np;
    unsigned* rr_prev = P.d_rrowx + (size_t)(b ^ 1) * P.idx->Np;
    launch_step_begin(P, nullptr, st, true, d.vrowx[b ^ 1], P.rowsV, d.vcol[b ^ 1], P.rowsVT, P.d_coef,
                      hr ? rr_cur : P.rmax_direct ? P.d_rrow : nullptr);
    if (hr) {
        launch_pack_r_headroom(P, P.d_res, rr_prev, rr_cur, P.d_urowr, st);
    } else {
        launch_pack_r(P, P.d_res, st, 1, P.rmax_direct);
        if (P.r_headroom)  // the next step's previous maxima
            CK(cudaMemcpyAsync(rr_cur, P.d_rrow, (size_t)P.idx->Np * 4, cudaMemcpyDeviceToDevice, st));
    }
    DescendBufs db = vu ? DescendBufs{d.vrowx[b], d.vcol[b], d.vrowx[b ^ 1], d.vcol[b ^ 1], d.ucol[b],
                                      d.tmap_vtq[b], d.vtq[b ^ 1], nullptr}
                        : DescendBufs{d.vrowx[b], d.vcol[b], d.vrowx[b ^ 1], d.vcol[b ^ 1], d.vcol[b],
                                      P.tmap_vtq_b, nullptr, nullptr};
    if (hr) db.urow_r = P.d_urowr;
    launch_gemm_bwd_update(P, V, st, &db);
    launch_descend_fixup(P, V, d.vrowx[b], d.vrowx[b ^ 1], d.urow[b], d.urow[b ^ 1], d.vcol[b], d.vcol[b ^ 1],
                         d.ucol[b ^ 1], vu ? d.vtq[b ^ 1] : nullptr, st);
    return check_launch("descend step");
}

constexpr int kLongGraphPairs[2] = {16, 4};  // pairs of steps per replay of a split plan's long graphs

// K descent steps; with sig_last the final step runs outside the graph with the
// row-chunk release of V on (P.d_rowsig zeroed, then P.sig_ev recorded, on st)
static int descend_impl(Plan& P, float* V_dev, const float* p_dev, int64_t steps, double* losses_dev, cudaStream_t st,
                        bool sig_last) {
    if (P.vtq_from_update) {
        const int rc0 = ensure_vtq2(P);
        if (rc0) return rc0;
    }
    const DescendPtrs d = descend_ptrs(P);
    auto plain_step = [&](int64_t t) -> int {
        const bool sig = sig_last && t == steps - 1;
        if (sig) {
            CK(cudaMemsetAsync(P.d_rowsig, 0, P.sig_expect.size() * sizeof(unsigned), st));
            CK(cudaEventRecord(P.sig_ev, st));
        }
        P.sig_on = sig;
        const int r = descend_step(P, d, (int)(t & 1), V_dev, p_dev, losses_dev, st, t == 0);
        P.sig_on = false;
        return r;
    };
    int rc = upload_opt(P, st);
    if (rc) return rc;
    CK(cudaMemsetAsync(&P.d_opt->loss_idx, 0, sizeof(long long), st));
    P.h_losses = losses_dev;  // pageable source: staged synchronously by the copy below
    CK(cudaMemcpyAsync(&P.d_opt->losses, &P.h_losses, sizeof(double*), cudaMemcpyHostToDevice, st));
    if (P.tiny) {  // every step in one cooperative kernel (sos_tiny.cu)
        CK(cudaMemsetAsync(P.d_coef, 0, (size_t)P.idx->M * 4, st));
        CK(cudaMemsetAsync(P.d_grad, 0, (size_t)P.idx->N * P.r * 4, st));
        if (launch_tiny_descend(P, V_dev, p_dev, steps, st))
            return fail(SOS_ERR_CUDA, "tiny descend launch: %s", cudaGetErrorString(cudaGetLastError()));
        return check_launch("tiny descend");
    }
    // step 0 starts from the exact maxima and slices of the caller's V
    launch_pack_v(P, V_dev, st, d.vrowx[0], d.vcol[0]);
    if (!P.split) CK(cudaMemcpyAsync(d.urow[0], d.vrowx[0], P.rowsV * 4, cudaMemcpyDeviceToDevice, st));
    if (P.vtq_from_update)  // step 0's forward packs VTQ[0] with the exact column maxima
        CK(cudaMemcpyAsync(d.ucol[0], d.vcol[0], P.rowsVT * 4, cudaMemcpyDeviceToDevice, st));
    if ((rc = plain_step(0))) return rc;
    int64_t left = steps - 1;
    const bool timing = P.timing && P.timing->on;  // per-kernel events need plain launches
    const int64_t keep_plain = sig_last ? 1 : 0;      // the signalling step is never replayed
    if (left >= 2 + keep_plain && !timing) {
        // steps 1, 2 (parities 1, 0) captured once as a graph, replayed for every pair;
        // split plans (a step of 4 short kernels chained by programmatic dependent
        // launch, which does not reach across graph launches) also keep a graph of
        // graphs of 16 and 4 pairs, so that a graph boundary (~3 us) falls on every 32nd
        // or 8th step instead of every 2nd
        const void* key[3] = {V_dev, p_dev, nullptr};  // the loss array is read from DevOpt
        if (memcmp(key, P.gkey, sizeof(key)) != 0) {
            if (P.gexec) cudaGraphExecDestroy(P.gexec);
            for (cudaGraphExec_t& g : P.gexec_long) {
                if (g) cudaGraphExecDestroy(g);
                g = nullptr;
            }
            P.gexec = nullptr;
            memcpy(P.gkey, key, sizeof(key));
        }
        auto capture = [&](cudaGraphExec_t* exec, int pairs) -> int {
            if (*exec) return SOS_OK;
            cudaStream_t cs;
            CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            const int64_t l0 = P.launches;
            cudaGraph_t graph = nullptr;
            cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
            int rcs = e == cudaSuccess ? SOS_OK : SOS_ERR_CUDA;
            for (int k = 0; k < 2 * pairs && !rcs; ++k)
                rcs = descend_step(P, d, (k + 1) & 1, V_dev, p_dev, losses_dev, cs);
            cudaError_t e2 = cudaStreamEndCapture(cs, &graph);
            P.glaunches = (P.launches - l0) / pairs;
            P.launches = l0;
            cudaStreamDestroy(cs);
            if (e != cudaSuccess || rcs || e2 != cudaSuccess || cudaGraphInstantiate(exec, graph, 0) != cudaSuccess) {
                if (graph) cudaGraphDestroy(graph);
                *exec = nullptr;
                return fail(SOS_ERR_CUDA, "descend graph capture failed: %s", cudaGetErrorString(cudaGetLastError()));
            }
            cudaGraphDestroy(graph);
            return SOS_OK;
        };
        if ((rc = capture(&P.gexec, 1))) return rc;
        for (int g = 0; g < 2 && P.split; ++g) {
            const int pairs = kLongGraphPairs[g];
            if (left < 2 * pairs + keep_plain) continue;
            if ((rc = capture(&P.gexec_long[g], pairs))) return rc;
            for (; left >= 2 * pairs + keep_plain; left -= 2 * pairs) {
                CK(cudaGraphLaunch(P.gexec_long[g], st));
                P.launches += P.glaunches * pairs;
            }
        }
        for (; left >= 2 + keep_plain; left -= 2) {
            CK(cudaGraphLaunch(P.gexec, st));
            P.launches += P.glaunches;
        }
    }
    for (int64_t t = steps - left; t < steps; ++t)
        if ((rc = plain_step(t))) return rc;
    return SOS_OK;
}

int sos_descend(sos_plan* pl, float* V_dev, const float* p_dev, int64_t steps, double* losses_dev, void* stream) {
    if (!pl || !V_dev || !p_dev || steps < 0 || (steps > 0 && !losses_dev)) return fail(SOS_ERR_ARG, "bad argument");
    if (reinterpret_cast<uintptr_t>(V_dev) & 15) return fail(SOS_ERR_ARG, "V_dev must be 16-byte aligned");
    Plan& P = pl->P;
    if (!P.opt_ready) return fail(SOS_ERR_ARG, "sos_opt_init not called");
    if (steps == 0) return SOS_OK;
    return descend_impl(P, V_dev, p_dev, steps, losses_dev, (cudaStream_t)stream, false);
}

// cuStreamWaitValue32 through the runtime's driver entry point (no -lcuda)
typedef CUresult (*PFN_wait_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_wait_value32 wait_value_fn() {
    static PFN_wait_value32 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_wait_value32>(p);
    }
    return fn;
}

int sos_solve_host(sos_plan* pl, float* V_host, const float* p_host, int64_t steps, double* losses_host) {
    if (!pl || !V_host || !p_host || steps < 0 || (steps > 0 && !losses_host)) return fail(SOS_ERR_ARG, "bad argument");
    Plan& P = pl->P;
    const size_t vb = (size_t)P.idx->N * P.r * 4, pb = (size_t)P.idx->M * 4;
    int rc;
    // device staging buffers live with the plan (no per-call cudaMalloc / cudaFree)
    if (!P.d_hV && ((rc = dalloc(&P.d_hV, vb)) || (rc = dalloc(&P.d_hp, pb)))) return rc;
    if (P.hl_cap < steps) {
        dfree(P.d_hl);
        P.d_hl = nullptr;
        P.hl_cap = 0;
        if ((rc = dalloc(&P.d_hl, sizeof(double) * steps))) return rc;
        P.hl_cap = steps;
    }
    if (steps > 0 && !P.opt_ready) return fail(SOS_ERR_ARG, "sos_opt_init not called");
    cudaStream_t st = 0;
    rc = SOS_OK;
    if (cudaMemcpyAsync(P.d_hV, V_host, vb, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(P.d_hp, p_host, pb, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return fail(SOS_ERR_CUDA, "H2D copy");
    // ship V back in row chunks while the last step's backward still runs (needs
    // stream memory operations; otherwise one copy after the last step)
    // (the split update of short-K plans does not release chunks: one copy at the end)
    const PFN_wait_value32 wait = steps > 0 && !P.split && !P.tiny ? wait_value_fn() : nullptr;
    bool overlap = wait != nullptr;
    if (overlap && !P.copy_st)
        overlap = cudaStreamCreateWithFlags(&P.copy_st, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreateWithFlags(&P.sig_ev, cudaEventDisableTiming) == cudaSuccess;
    if (steps > 0 && (rc = descend_impl(P, P.d_hV, P.d_hp, steps, P.d_hl, st, overlap))) return rc;
    const int64_t N = P.idx->N, chunk_rows = (int64_t)P.sig_blocks * kPairM;
    if (overlap) {
        if (cudaStreamWaitEvent(P.copy_st, P.sig_ev, 0) != cudaSuccess)
            return fail(SOS_ERR_CUDA, "copy stream wait");
        for (size_t c = 0; c < P.sig_expect.size(); ++c) {
            const int64_t r0 = (int64_t)c * chunk_rows, r1 = std::min(N, r0 + chunk_rows);
            if (r1 <= r0) break;
            if (wait(P.copy_st, (CUdeviceptr)(P.d_rowsig + c), P.sig_expect[c], CU_STREAM_WAIT_VALUE_GEQ) !=
                    CUDA_SUCCESS ||
                cudaMemcpyAsync(V_host + r0 * P.r, P.d_hV + r0 * P.r, (size_t)(r1 - r0) * P.r * 4,
                                cudaMemcpyDeviceToHost, P.copy_st) != cudaSuccess)
                return fail(SOS_ERR_CUDA, "chunked D2H of V");
        }
        // the fixup after the last update reads V only; the losses follow on st
    } else if (cudaMemcpyAsync(V_host, P.d_hV, vb, cudaMemcpyDeviceToHost, st) != cudaSuccess) {
        return fail(SOS_ERR_CUDA, "D2H copy");
    }
    if ((steps > 0 &&
         cudaMemcpyAsync(losses_host, P.d_hl, sizeof(double) * steps, cudaMemcpyDeviceToHost, st) != cudaSuccess) ||
        cudaStreamSynchronize(st) != cudaSuccess || (overlap && cudaStreamSynchronize(P.copy_st) != cudaSuccess))
        return fail(SOS_ERR_CUDA, "D2H copy: %s", cudaGetErrorString(cudaGetLastError()));
    return SOS_OK;
}

#ifdef SOS_EXPERIMENTS
// Experiment build only (not in include/sos_b200.h): number of live device
// allocations of the library whose guard margins are no longer all 0xFF; the
// first one is described in sos_last_error().  Synchronises the device.
int sos_exp_check_guards(int64_t* n_allocs) {
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(SOS_ERR_CUDA, "%s", cudaGetErrorString(cudaGetLastError()));
    std::lock_guard<std::mutex> lk(g_guard_mu);
    std::vector<unsigned char> h(kGuardBytes);
    int bad = 0;
    for (const auto& kv : g_guards) {
        const GuardRec& g = kv.second;
        for (int side = 0; side < 2; ++side) {
            const char* src = side ? g.base + kGuardBytes + g.bytes : g.base;
            if (cudaMemcpy(h.data(), src, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess)
                return fail(SOS_ERR_CUDA, "guard read: %s", cudaGetErrorString(cudaGetLastError()));
            size_t k = 0;
            while (k < kGuardBytes && h[k] == 0xFF) ++k;
            if (k < kGuardBytes) {
                if (!bad++)
                    fail(SOS_ERR_CUDA, "write %s a %zu-byte allocation (margin byte %zu)", side ? "past the end of" : "before",
                         g.bytes, k);
                break;
            }
        }
    }
    if (n_allocs) *n_allocs = (int64_t)g_guards.size();
    return bad ? -bad : SOS_OK;
}

// Experiment build only: negative control for the check above -- writes one
// zero byte just past the end of the largest live allocation.
int sos_exp_poke_guard(void) {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    const GuardRec* big = nullptr;
    for (const auto& kv : g_guards)
        if (!big || kv.second.bytes > big->bytes) big = &kv.second;
    if (!big) return fail(SOS_ERR_ARG, "no live allocation");
    return cudaMemset(big->base + kGuardBytes + big->bytes, 0, 1) == cudaSuccess ? SOS_OK : fail(SOS_ERR_CUDA, "poke");
}
#endif

}  // extern "C"
