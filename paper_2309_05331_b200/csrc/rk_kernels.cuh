// rk_kernels.cuh — device kernels of librkb200 and their host launchers.
//
// K1 pointwise fused step (exp / logistic), K2 lincomb + plane pack, K3 fused Gray–Scott
// stage kernel, K4 max-norm reductions.  See DESIGN.md §Kernels for the roofline of each.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rkb {

enum RhsKind { RHS_NONE = -1, RHS_EXP = 0, RHS_LOGISTIC = 1, RHS_GRAY_SCOTT = 2 };

// Epilogues of the fused Gray–Scott stage kernel.
enum Epilogue {
    EPI_K = 0,          // write k_i = F(Y_i)
    EPI_FINAL = 1,      // write u_new = u + sum beta_j k_j (+ beta_i k_i), k_i not stored
    EPI_FINAL_ERR = 2,  // EPI_FINAL + embedded error ratio and its max (CK54 adaptive)
    EPI_FSAL_ERR = 3    // Y_s is u_new (FSAL): write Y_s and k_s, error ratio + max (DOPRI5)
};

constexpr int kMaxSlots = 5;  // k_j arrays read by one stage (DOPRI5 stages 6/7, CK54 stage 6)

// ---------------------------------------------------------------------------------------
// K1: pointwise step of a whole RK scheme in registers (vector states).
struct PwCoef {
    double g[7][7];    // dt * a_ij
    double beta[7];    // dt * b_j
    double delta[7];   // dt * (b_j - bhat_j)
};
struct PwArgs {
    const double* u;
    double* u_out;
    int64_t count;     // fp64 values (ncomp * local elements)
    int rhs;           // RHS_EXP / RHS_LOGISTIC
    double lambda;
    int nsteps;        // >= 1 fixed steps in registers (ignored with error ratio)
    double dt, atol, rtol;
    unsigned long long* errmax;  // error-ratio max (uint64 bits), non-null => error mode
    PwCoef cf;
};
cudaError_t launch_pointwise(int scheme, const PwArgs& a, cudaStream_t st, int num_sms);

// ---------------------------------------------------------------------------------------
// K3: fused Gray–Scott stage kernel.  Grid state layout [z][c][y][x], 2 components.
struct GsStageArgs {
    const double* u;
    const double* k[kMaxSlots];  // slot arrays, increasing stage index j
    double g[kMaxSlots];         // Y coefficient per slot (0: slot not in Y, no halo load)
    double beta[kMaxSlots];      // final-combination weight per slot (0: skip)
    double delta[kMaxSlots];     // error weight per slot (0: skip)
    double beta_new, delta_new;  // weights of the k_i computed by this stage
    double* out_k;
    double* out_u;
    const double* ghost_lo;      // Y_i plane z=-1   [2][ny][nx]; null => periodic wrap in slab
    const double* ghost_hi;      // Y_i plane z=nzl  [2][ny][nx]
    unsigned long long* errmax;
    double dt, atol, rtol;
    double d1, d2, F, FK, inv_h2;
    int nx, ny, nzl;
    int z_lo, z_hi;              // output planes [z_lo, z_hi) (boundary mode: see zmode)
    int zchunk;                  // output planes per CTA
    int zmode;                   // 0: contiguous chunks; 1: chunk 0 = plane 0, chunk 1 = nzl-1
    int nslots;
};
// Launch over the planes described by a.z_lo/z_hi/zmode; epi = Epilogue.
cudaError_t launch_gs_stage(int epi, const GsStageArgs& a, cudaStream_t st, int* nlaunch);

// Pack Y_i on own planes 0 and nzl-1 into send[0 .. 2*plane) = [lo | hi].
cudaError_t launch_gs_pack(const GsStageArgs& a, double* send, cudaStream_t st);

// ---------------------------------------------------------------------------------------
// K2 / K4: algebra.
struct LincombArgs {
    double* out;
    const double* in[14];
    double coef[14];
    int k;
    int64_t count;
};
cudaError_t launch_lincomb(const LincombArgs& a, cudaStream_t st, int num_sms);
cudaError_t launch_norm_inf(const double* x, int64_t count, unsigned long long* out,
                            cudaStream_t st, int num_sms);

}  // namespace rkb
