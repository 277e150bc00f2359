// sos_internal.cuh -- shared definitions of the CUDA path (not part of the ABI).
//
// HBM layouts:
//   * split operand tiles "S-layout": an fp32 matrix X[rows][K] is stored as
//     fp16 hi/lo pairs scaled by a power of two s (x*s = hi + lo + O(2^-22 |x*s|)),
//     in K-blocks of 32:   byte offset of row `row`, K-block kb =
//         (kb * rows_total + row) * 128
//     and inside that 128-byte row the 16-byte chunk c (c<4: hi of k=8c..8c+7,
//     c>=4: lo of k=8(c-4)..) lives at physical chunk c ^ (row & 7) -- exactly
//     the UMMA K-major SWIZZLE_128B image, so a 128-row x 32-K tile is one
//     contiguous 16 KB block copied to shared memory by one bulk copy.
//       VS  = V   as [rK/32][Np][128B]   (forward A and B operands, K = column of V)
//       VTS = V^T as [Np/32][rN][128B]   (backward B operand, K = row of V)
//       RS  = R   as [Np/32][Np][128B]   (backward A operand, K = column j of R)
//   * pair-rank table PT[jb][i][32] (uint32): PT[((j/32)*Np + i)*32 + j%32] =
//     rank(alpha_i + alpha_j), 0xFFFFFFFF for padding (i >= N or j >= N).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

namespace sos {

// kernel kinds for per-launch event timing (sos_plan_timing_read)
enum KernelKind { KK_ABSMAX_V = 0, KK_PACK_V, KK_GEMM_FWD, KK_RESIDUAL, KK_ABSMAX_R, KK_PACK_R, KK_GEMM_BWD,
                  KK_UPDATE, KK_COUNT };

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

constexpr int kBlockM = 128;   // tile rows per CTA (UMMA M = 256 per CTA pair)
constexpr int kBlockN = 256;   // tile cols  (UMMA N)
constexpr int kBlockK = 32;    // fp32-equivalent K per stage (hi+lo = 128 B rows)
constexpr int kPad = 256;      // Np = N rounded up to kPad
constexpr int kEpiWarps = 8;       // 4 TMEM lane quarters x 2 column halves
constexpr int kEpiCols = kBlockN / 2;
constexpr int kAuxWarps = 2;       // optimiser-update warps of the backward GEMM
constexpr int kGemmThreads = 64 + 32 * (kEpiWarps + kAuxWarps);  // producer, MMA, epilogue, aux
// K-blocks accumulated in TMEM before the epilogue drains them into fp32
// registers: tcgen05 fp32 accumulation truncates, so the number of in-TMEM
// adds per value is bounded.
constexpr int kSegKB = 16;
// bounded K-skew between the CTAs of a GEMM (see the producer in sos_gemm.cu)
constexpr int kSkewEpoch = 16;  // K-blocks per progress epoch
constexpr int kSkewLag = 2;     // epochs a CTA may run ahead of the slowest
constexpr int kSkewMaxSpin = 8192;  // bounded wait (x 256 ns): the skew bound is a locality hint, never a deadlock
constexpr uint32_t kInvalidRank = 0xFFFFFFFFu;
constexpr int kMaxVars = 64;       // n + 2d <= 64
constexpr int kMaxDeg2 = 64;

struct Scalars {           // device-resident per-step scalars
    unsigned int absmax_v; // float bits of max |V|
    unsigned int absmax_r; // float bits of max |res|
    float s_v;             // power-of-two scale for the V split
    float s_r;             // power-of-two scale for the R split
    double loss;           // sum res^2
    double pnorm2;         // sum p^2
};

// the device-side stopping rule of sos_step (sos_opt_set_stop), read after
// the residual kernel completed the loss and |p|^2 reductions
__device__ __forceinline__ bool descent_stopped(const Scalars* sc, double tol) {
    return tol > 0.0 && sc->loss <= tol * sc->pnorm2;
}

struct Index {
    int n, d;
    int64_t N, M, Np;
    int nb;                    // rows of the binomial table = n + 2d
    uint32_t* d_binom;         // [nb][2d+1] C(x,k), x < nb, k <= 2d   (device)
    uint8_t* d_ms;             // [N][d] sorted variable indices of alpha_i
    uint8_t* d_alpha;          // [N][n] exponents of alpha_i
    uint32_t* d_pt;            // pair-rank table PT (Np*Np)
};

struct TileCoord { int a; int b; };  // a: 256-row block (CTA pair), b: 256-col block

struct Plan {
    const Index* idx;
    int64_t r, rK, rN;
    uint8_t* d_vs;    // VS
    uint8_t* d_vts;   // VTS
    uint8_t* d_rs;    // RS
    float* d_coef;    // M
    float* d_res;     // M
    float* d_m;       // Adam moments (lazy)
    float* d_v;
    Scalars* d_scal;
    float* d_ring;    // per-CTA gradient tile ring of the fused backward + update
    unsigned long long* d_progress;  // [2] K-skew counters (fwd, bwd)
    TileCoord* d_tiles2_fwd; int ntiles2_fwd;  // CTA-pair tiles (256-row blocks)
    TileCoord* d_tiles2_bwd; int ntiles2_bwd;
    alignas(64) uint8_t tmap_vs[128];   // CUtensorMap of VS, VTS, RS (2-SM TMA loads)
    alignas(64) uint8_t tmap_vts[128];
    alignas(64) uint8_t tmap_rs[128];
    int opt_kind; float lr, b1, b2, eps; int64_t t; bool opt_ready;
    double stop_tol;  // sos_opt_set_stop: skip backward + update once loss <= stop_tol * |p|^2
    int64_t launches;
    int num_sms;
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

void launch_absmax_v(Plan& P, const float* V, cudaStream_t st);
void launch_pack_v(Plan& P, const float* V, bool with_vts, cudaStream_t st);
void launch_residual(Plan& P, const float* coef, const float* p, float* res, cudaStream_t st);
void launch_absmax_res(Plan& P, const float* res, cudaStream_t st);
void launch_pack_r(Plan& P, const float* res, cudaStream_t st, double stop_tol);
void launch_gemm2_fwd(Plan& P, float* coef, const float* V_for_vts, cudaStream_t st);
void launch_gemm2_bwd(Plan& P, float* grad, cudaStream_t st);
void launch_gemm2_bwd_update(Plan& P, float* V, cudaStream_t st);
bool make_split_tmap(void* map, const uint8_t* base, int64_t rows_total, int64_t num_kb);

}  // namespace sos
