// sos_internal.cuh -- shared definitions of the CUDA path (not part of the ABI).
//
// Precision scheme: every fp32 operand row x (a row of
// V, of V^T or of R) is stored as three signed-int8 slices against a per-row
// scale u = max|x| / 127 (sos_slice.cuh):
//     x / u = a1 + a2/256 + a3/65536 + e,   |a1| <= 127, |a2|,|a3| <= 128,  |e| <= 2^-16
// (about 23 significant bits relative to the row maximum).  A product of two
// such rows is accumulated EXACTLY in s32 on the tensor cores (kind::i8):
//     acc0 = sum a1 b1,  acc1 = sum a1 b2 + a2 b1,  acc2 = sum a1 b3 + a2 b2 + a3 b1
// and the epilogue forms u_x u_y (acc0 + acc1/256 + acc2/65536) in fp32.  The
// dropped slice products (2,3), (3,2), (3,3) are O(2^-24) of the leading term.
//
// HBM layouts:
//   * "Q-layout" of an operand X[rows][K] (int8 slices): K-blocks of 64, rows
//     of 64 bytes; byte (s, kb, row, k) at
//         ((s * nkb + kb) * rows_total + row) * 64 + ((c ^ ((row >> 1) & 3)) * 16) + k % 16,
//     c = (k % 64) / 16 -- the UMMA K-major SWIZZLE_64B image, so a box of
//     `rows` x 64 B x 3 slices is one TMA tensor copy into a pipeline stage.
//       VQ  = V   (rows = monomial i, K = square k)      fwd A and B operands
//       VTQ = V^T (rows = square k,   K = monomial j)    bwd B operand
//       RQ  = R   (rows = monomial i, K = monomial j)    bwd A operand
//   * per-row scales u = max / 127, kept as the float bits of the row maximum:
//     vrow[i] = max_k |V_ik|, vcol[k] = max_j |V_jk|, rrow[i] = max_j |R_ij|.
//   * pair-rank table PT (uint32, rank(alpha_i + alpha_j), 0xFFFFFFFF for
//     padding i >= N or j >= N): only the 64 x 64 blocks I <= J of the
//     symmetric table are stored, see pt_entry / pt_entries below.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

namespace sos {

// kernel kinds for per-launch event timing (sos_plan_timing_read)
enum KernelKind { KK_ABSMAX_V = 0, KK_PACK_V, KK_GEMM_FWD, KK_RESIDUAL, KK_ABSMAX_R, KK_PACK_R, KK_GEMM_BWD,
                  KK_UPDATE, KK_MID, KK_TINY, KK_COUNT };

struct TimingRec { int kind; cudaEvent_t a, b; };
struct Timing {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<TimingRec> recs;
    cudaEvent_t get() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
};

constexpr int kSlices = 3;        // int8 slices per operand value
constexpr int kQK = 64;           // K-elements per Q-layout row (64 bytes, SWIZZLE_64B)
constexpr int kPairM = 256;       // UMMA M over a CTA pair (128 rows per CTA)
constexpr int kTileN = 160;       // UMMA N (3 s32 accumulators x 160 columns fit TMEM's 512)
constexpr int kHalfN = kTileN / 2;  // B rows staged per CTA
constexpr int kPad = 256;         // Np = N rounded up to kPad (R rows, PT)
constexpr int kEpiWarps = 8;      // 4 TMEM lane quarters x 2 column halves
constexpr int kEpiCols = kTileN / 2;  // 80 output columns per epilogue thread
constexpr int kAuxWarps = 2;      // optimiser-update / V^T-pack warps of the GEMMs
constexpr int kGemmThreads = 64 + 32 * (kEpiWarps + kAuxWarps);  // producer, MMA, epilogue, aux
constexpr int kPtW = 64;          // pair-rank table block width (64 x 64 blocks, see pt_entry)
// bounded K-skew between the CTAs of a GEMM (see the producer in sos_gemmq.cu)
constexpr int kSkewEpoch = 8;     // K-blocks (of 64) per progress epoch (tools/gpu_skew2.sh)
constexpr int kSkewLag = 1;       // epochs a CTA may run ahead of the slowest
constexpr double kSkewMinBytes = 64.0 * (1 << 20);  // operand bytes (A + B slices) below which no pacing
constexpr int kSkewMaxSpin = 8192;  // bounded wait (polls): a locality hint, never a deadlock
constexpr uint32_t kInvalidRank = 0xFFFFFFFFu;
constexpr int kMaxVars = 255;     // n + 2d <= 255 (variable indices are uint8)
constexpr int kMaxDeg2 = 64;

// s32 accumulation stays exact while K * 3 * 128^2 < 2^31: K-blocks of 64 per
// TMEM segment (longer K is split into segments drained into fp32 sums)
constexpr int kSegKBMax = (int)(2147483647LL / (3LL * 128 * 128 * kQK));

struct Scalars {           // device-resident per-step scalars
    double loss;           // sum res^2
    double pnorm2;         // sum p^2
};

// optimiser state on the device, so that a captured step replays unchanged
// (CUDA graphs in sos_descend): the host uploads the parameters at the start of
// every sos_step / sos_descend call; k_step_begin advances t once per step
struct DevOpt {
    float lr, b1, b2, eps;  // uploaded by the host
    double stop_tol;        // sos_opt_set_stop (0 = off), uploaded by the host
    long long t;            // Adam step count (device-managed)
    long long loss_idx;     // sos_descend: next entry of the caller's loss array (device-managed)
    double* losses;         // sos_descend: the call's loss array (set per call, so the captured
                            // step graph does not depend on it)
    float lr_c1;            // Adam constants of step t (device-managed, advance_step):
    float inv_sqrt_c2;      //   lr / (1 - b1^t) and 1 / sqrt(1 - b2^t)
    double b1t, b2t;        // b1^t, b2^t as running products (device-managed; t = 0 after the
                            // memset of sos_opt_init, when they are not read)
};

// t += 1 and the bias-correction constants of the new step (one thread, once per
// step, before any update of that step reads them)
__device__ __forceinline__ void advance_step(DevOpt* opt) {
    const long long t = opt->t + 1;
    // b^t by one multiplication per step (two fp64 pow calls were ~2 us of one
    // thread on the step's critical path); relative drift <= t * 2^-53
    const double b1t = t == 1 ? (double)opt->b1 : opt->b1t * (double)opt->b1;
    const double b2t = t == 1 ? (double)opt->b2 : opt->b2t * (double)opt->b2;
    opt->t = t;
    opt->b1t = b1t;
    opt->b2t = b2t;
    opt->lr_c1 = (float)((double)opt->lr / (1.0 - b1t));
    opt->inv_sqrt_c2 = (float)(1.0 / sqrt(1.0 - b2t));
}

// the device-side stopping rule of sos_step (sos_opt_set_stop), read after
// the residual kernel completed the loss and |p|^2 reductions
__device__ __forceinline__ bool descent_stopped(const Scalars* sc, double tol) {
    return tol > 0.0 && sc->loss <= tol * sc->pnorm2;
}
__device__ __forceinline__ bool descent_stopped(const Scalars* sc, const DevOpt* opt, int use_stop) {
    return use_stop && descent_stopped(sc, opt->stop_tol);
}

// Pair-rank table layout: PT(i, j) = rank(alpha_i + alpha_j) = PT(j, i), stored
// only for 64-blocks I = i / 64 <= J = j / 64.  Block column J holds rows
// i < 64 (J + 1), 64 ranks (j % 64) per row: entry ((64 J (J+1) / 2 + i) 64 + j % 64).
// A 64 x 64 block (I <= J) is contiguous; a row i of block column J is 256 bytes.
__host__ __device__ inline int64_t pt_entry(int64_t i, int64_t j) {  // needs i / 64 <= j / 64
    const int64_t J = j >> 6;
    return ((J * (J + 1) / 2) * 64 + i) * 64 + (j & 63);
}
__host__ __device__ inline int64_t pt_entry_sym(int64_t i, int64_t j) {
    return (i >> 6) <= (j >> 6) ? pt_entry(i, j) : pt_entry(j, i);
}
__host__ __device__ inline int64_t pt_entries(int64_t Np) {
    const int64_t nb = Np / 64;
    return nb * (nb + 1) / 2 * 64 * 64;
}

struct Index {
    int n, d;
    int64_t N, M, Np;
    int nb;                    // rows of the binomial table = n + 2d
    uint32_t* d_binom;         // [nb][2d+1] C(x,k), x < nb, k <= 2d   (device)
    uint8_t* d_ms;             // [N][d] sorted variable indices of alpha_i
    uint8_t* d_alpha;          // [N][n] exponents of alpha_i
    uint32_t* d_pt;            // pair-rank table PT, one block triangle (pt_entries(Np))
};

// One CTA-pair output tile: rows [256a, 256a + 256) x columns [c0, c0 + nb).
// nb = 160 except where a narrower tile (multiple of 32) stops the MMAs from
// computing columns nobody needs: the last column block (r or N not a multiple
// of 160) and, in the forward, the diagonal tile of each row block (c0 = 256a
// instead of the 160-grid line below it).  The MMA N and the B rows each CTA
// supplies (nb / 2) follow nb; the epilogue ignores accumulator columns >= nb.
struct TileCoord { int a; int c0; int nb; int pad; };
// rowsig value that satisfies every chunk's wait (cyclic >= compare of stream waits)
constexpr unsigned kSigReleased = 0x40000000u;  // a: 256-row block (CTA pair), b: 160-col block

struct Plan {
    const Index* idx;
    int64_t r;
    int64_t rowsV;    // VQ rows_total: covers the 256-row A blocks and 160-row B blocks of N
    int64_t nkbV;     // VQ K-blocks: ceil(r / 64)
    int64_t rowsVT;   // VTQ rows_total: r rounded up to 160
    int64_t nkbN;     // VTQ / RQ K-blocks: ceil(N / 64) (RQ rows stay padded to Np)
    uint8_t* d_vq;    // VQ
    uint8_t* d_vtq;   // VTQ
    uint8_t* d_vtq2;  // sos_descend: second VTQ buffer (the update writes step t+1's while step t's is read)
    // implementation choices (sos_plan_opts, fixed at plan creation)
    bool split;            // split step: fwd, k_mid (cooperative), bwd storing the gradient,
                           // k_update_rows -- short K, where a tile's MMAs cannot hide the
                           // fused update (~25 us per tile in 8 warps per SM)
    bool vtq_from_update;  // sos_descend (fused step): the update writes the next VTQ (long K)
    bool vtq_in_aux;       // the forward's aux warps write VTQ (else k_pack_vtq before it)
    bool rmax_direct;      // R row maxima by one gather pass over PT (else the lattice DP)
    bool narrow;           // narrow tiles at ragged column blocks
    bool r_headroom;       // sos_descend, fused step: R slices with the previous step's scales (no DP)
    int tile_w_fwd;        // column tile width of the forward / backward GEMM (160, or 128 for
    int tile_w_bwd;        // small problems; the backward only in split plans)
    int mid_grid;          // cooperative grid of k_mid (co-resident blocks)
    int mid_tiles;         // R blocks each k_mid block holds in shared memory
    int mid_hold_v;        // V tiles each k_mid block holds from its phase A to B
    bool tiny;             // sos_descend runs all its steps in k_tiny_descend (small N, r)
    int tiny_grid;         // its cooperative grid (0: the problem is not tiny-capable)
    double* d_part;        // k_mid's per-block partial sums [mid_grid][2]
    unsigned* d_rrowx;     // sos_descend, long K: [2][Np] exact R row maxima (step parity)
    unsigned* d_urowr;     // [Np] scales the RQ rows were written with (headroom or exact)
    float* d_grad;         // N x r gradient buffer of the split step
    uint8_t* d_rq;    // RQ
    unsigned* d_vrow; // max_k |V_ik| (float bits), rowsV
    unsigned* d_vcol; // max_j |V_jk| (float bits), rowsVT
    unsigned* d_rrow; // max_j |R_ij| (float bits), Np
    float* d_rlev;    // lattice-DP levels for the R row maxima
    unsigned* d_dbuf; // sos_descend: [2][rowsV] exact row maxima, [2][rowsV] used row scales, [2][rowsVT] column
                      // maxima, [2][rowsVT] used column scales
    float* d_coef;    // M
    float* d_res;     // M
    float* d_m;       // Adam moments (lazy)
    float* d_v;
    Scalars* d_scal;
    float* d_ring;    // per-CTA staging of a finished gradient tile (fused backward + update)
    unsigned long long* d_progress;  // [2] K-skew counters (fwd, bwd)
    TileCoord* d_tiles_fwd; int ntiles_fwd;
    TileCoord* d_tiles_bwd; int ntiles_bwd;
    alignas(64) uint8_t tmap_vq_a[128];   // CUtensorMaps (3-D: 64 B x rows x slice planes)
    alignas(64) uint8_t tmap_vq_b[128];
    alignas(64) uint8_t tmap_vtq_b[128];
    alignas(64) uint8_t tmap_vtq2_b[128];
    alignas(64) uint8_t tmap_rq_a[128];
    int opt_kind; float lr, b1, b2, eps; bool opt_ready;
    double stop_tol;  // sos_opt_set_stop: skip backward + update once loss <= stop_tol * |p|^2
    DevOpt* d_opt;    // device copy of the optimiser parameters + step counter
    // sos_descend: a captured pair of steps, replayed with cudaGraphLaunch
    cudaGraphExec_t gexec;
    cudaGraphExec_t gexec_long[2];  // split plans: kLongGraphPairs[i] pairs per replay (fewer graph boundaries)
    const void* gkey[3];   // (V, p, -) the graphs were captured for
    double* h_losses;      // host copy of the current sos_descend call's loss array pointer
    int64_t glaunches;     // kernels per replay of the pair graph (launch accounting)
    // sos_solve_host: device staging of the caller's host buffers (lazy)
    float* d_hV;
    float* d_hp;
    double* d_hl;
    int64_t hl_cap;
    // sos_solve_host: the last step's update releases finished row chunks of V
    // (rowsig[c] counts tile halves stored; chunk c = row blocks [c, c+1) x sig_blocks)
    // and a copy stream ships each chunk to the host while the rest still runs
    unsigned* d_rowsig;
    int sig_blocks;
    std::vector<uint32_t> sig_expect;
    bool sig_on;
    cudaStream_t copy_st;
    cudaEvent_t sig_ev;
    int64_t launches;
    int num_sms;
    int64_t l2_bytes;      // L2 size (the split update keeps V, m, v in L2 when they fit)
    int upd_rows;          // rows per block of the split update (0: not chosen yet)
    Timing* timing;
};

// counts every kernel launch of a plan and, when timing is on, brackets it
// with CUDA events recorded on the launch stream
struct LaunchScope {
    Plan& P;
    int kind;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    LaunchScope(Plan& p, int k, cudaStream_t s) : P(p), kind(k), st(s) {
        if (P.timing && P.timing->on) {
            a = P.timing->get();
            cudaEventRecord(a, st);
        }
    }
    ~LaunchScope() {
        P.launches++;
        if (a) {
            cudaEvent_t b = P.timing->get();
            cudaEventRecord(b, st);
            P.timing->recs.push_back(TimingRec{kind, a, b});
        }
    }
};

// ---- kernels (defined in the .cu files) ----
void launch_index_build(Index& ix, cudaStream_t st);
void launch_beta_table(const Index& ix, uint8_t* beta, cudaStream_t st);
void launch_pair_lookup(const Index& ix, const int64_t* i, const int64_t* j, int64_t cnt, uint32_t* out,
                        cudaStream_t st);
// number of degree-D monomials in n variables, C(n+D-1, D)
inline int64_t rmax_level_count(int n, int D) {
    long double c = 1;
    for (int t = 1; t <= D; ++t) c = c * (n + D - t) / t;
    return (int64_t)(c + 0.5L);
}
// R row maxima through the monomial lattice (sos_index.cu); scratch holds the
// levels strictly between degree 2d and degree d
void launch_rmax_dp(const Index& ix, const float* res, float* scratch, unsigned* rrow, cudaStream_t st,
                    const Scalars* sc, const DevOpt* opt, int use_stop);

void launch_vmax(Plan& P, const float* V, cudaStream_t st, unsigned* vrow = nullptr, unsigned* vcol = nullptr);
void launch_pack_v(Plan& P, const float* V, cudaStream_t st, unsigned* vrow = nullptr,
                   unsigned* vcol = nullptr);  // maxima + VQ
void launch_pack_vtq(Plan& P, const float* V, cudaStream_t st, const unsigned* vcol = nullptr);
void launch_residual(Plan& P, const float* coef, const float* p, float* res, cudaStream_t st);
// losses_from_opt: record into the loss array set for the current sos_descend call;
// zero0 / zero1 (n0 / n1 words), zero_coef (M floats), zero_r (Np words, R row
// maxima accumulated by atomicMax): accumulators to clear for the next stage
void launch_step_begin(Plan& P, double* losses, cudaStream_t st, bool losses_from_opt = false,
                       unsigned* zero0 = nullptr, int64_t n0 = 0, unsigned* zero1 = nullptr, int64_t n1 = 0,
                       float* zero_coef = nullptr, unsigned* zero_r = nullptr);
void launch_rmax(Plan& P, const float* res, cudaStream_t st, int use_stop, bool rrow_zeroed = false);
void launch_pack_rq(Plan& P, const float* res, cudaStream_t st, int use_stop);
// maxima + RQ; rrow_zeroed: rrow already cleared on the stream (direct maxima)
void launch_pack_r(Plan& P, const float* res, cudaStream_t st, int use_stop, bool rrow_zeroed = false);
// sos_descend after its first step (long K): RQ sliced with kHeadroom x the
// previous step's exact R row maxima, this step's exact maxima into rrow_cur
// (cleared before), rows outside the window re-sliced; urow_r = scale per row
void launch_pack_r_headroom(Plan& P, const float* res, const unsigned* rrow_prev, unsigned* rrow_cur,
                            unsigned* urow_r, cudaStream_t st);
// the cost model choosing the direct R maxima pass over the lattice DP
bool rmax_direct_default(const Index& ix);
// sos_descend: maxima buffers of the current and the next step
struct DescendBufs {
    const unsigned* vrow_cur;  // exact row maxima of the current V
    const unsigned* vcol_cur;  // exact column maxima of the current V
    unsigned* vrow_next;       // exact row maxima of the updated V (atomicMax, zeroed before)
    unsigned* vcol_next;       // exact column maxima of the updated V
    const unsigned* ucol_cur;  // column scales the current VTQ was written with (backward B unscale)
    const uint8_t* tmap_vtq_cur;  // tensor map of the current VTQ buffer
    uint8_t* vtq_next;         // VTQ buffer the update writes for the next step
    const unsigned* urow_r;    // scales the RQ rows were written with (nullptr: the exact rrow)
};
// plans with fewer K-blocks (N / 64) than this use the split step (Plan::split)
constexpr int kSplitKb = 48;
// tiny plans (one cooperative kernel per sos_descend call) by default while N^2 r
// is at most this: measured crossover with the split step between N = r = 286
// (32.2K vs 31.8K steps/s) and 330 (25.8K vs 29.5K), profiles/r2_tiny_ab.log
constexpr double kTinyMaxWork = 2.0e7;
// split step, between forward and backward: residual + loss, step bookkeeping
// (t += 1, loss record: losses[0], or the sos_descend array from DevOpt with
// losses_from_opt), with colmax the exact column maxima of V (atomicMax into
// vcol, cleared by the previous k_mid -- or already exact), V^T slices, R row
// maxima (direct), coef cleared, R slices; zero_cols (rowsVT words) cleared
// for the next step's k_mid
void launch_mid(Plan& P, const float* p, const float* V, unsigned* vcol, bool colmax, unsigned* zero_cols,
                double* losses, bool losses_from_opt, cudaStream_t st);
// split step, after the backward: GD / Adam on blocks of whole rows of V (the
// gradient in P.d_grad); with vq_next also the next step's VQ against the EXACT
// new row maxima (vrow_next); a stopped descent copies the current maxima
void launch_update_rows(Plan& P, float* V, uint8_t* vq_next, const unsigned* vrow_cur, unsigned* vrow_next,
                        cudaStream_t st);
// cooperative grid of k_mid (blocks) and the R blocks each holds (tiles_per_block)
int mid_grid_for(int64_t nkbN, int64_t rowsVT, int64_t M, int num_sms, int* tiles_per_block, int* hold_v);
int tiny_grid_for(int num_sms);
int launch_tiny_descend(Plan& P, float* V, const float* p, int64_t steps, cudaStream_t st);
// slices written by the update use kHeadroom x the current row maximum
constexpr float kHeadroom = 2.f;

// pdl: launch with programmatic stream serialization (the kernel's setup overlaps
// the previous kernel's tail; used where that kernel holds no TMEM)
void launch_gemm_fwd(Plan& P, float* coef, const float* V_for_vtq, cudaStream_t st, const unsigned* urow = nullptr,
                     const unsigned* vcol = nullptr, bool zero_scal = false, bool pdl = false);
// backward storing 4RV into grad; vcol / tmap_vtq: column scales and tensor map of
// the V^T slices to read (default: the plan's VTQ and vcol)
void launch_gemm_bwd(Plan& P, float* grad, cudaStream_t st, const unsigned* vcol = nullptr,
                     const uint8_t* tmap_vtq = nullptr, bool pdl = false);
// whether the forward's aux warps can hide the V^T pack (elements per aux thread
// vs K-blocks per CTA pair over the forward's actual grid)
bool vtq_fits_aux(const Plan& P);
void launch_gemm_bwd_update(Plan& P, float* V, cudaStream_t st, const DescendBufs* db = nullptr);
// sos_descend, long K: re-slice the rows (and with vtq_next the columns) whose new
// maximum left the headroom window; one launch (sos_pointwise.cu)
void launch_descend_fixup(Plan& P, const float* V, const unsigned* vrow_cur, unsigned* vrow_next,
                          const unsigned* urow_cur, unsigned* urow_next, const unsigned* vcol_cur, unsigned* vcol_next,
                          unsigned* ucol_next, uint8_t* vtq_next, cudaStream_t st);
bool make_q_tmap(void* map, const uint8_t* base, int64_t rows_total, int64_t nkb, int box_rows);
// CTA pairs of the persistent GEMM grid (co-resident clusters)
int resident_gemm_pairs(int num_sms);

}  // namespace sos
