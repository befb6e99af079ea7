// rk_kernels.cuh — device kernels of librkb200 and their host launchers.
//
// K1 pointwise fused step (exp / logistic), K2 lincomb + halo-plane pack, K3 fused
// Gray–Scott stage kernel (TMA-fed), K4 max-norm reductions.  DESIGN.md §Kernels gives the
// roofline and the algorithmic bytes of each.
#pragma once
#include <cuda.h>
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
// Grid arrays in HBM use a PADDED periodic layout: [z][c][ny+2][P] fp64 with P >= nx+2 even
// (16-byte rows for TMA); logical cell (x, y) sits at padded (x+1, y+1), and the producer
// of every array also writes the periodic copies x=-1 -> nx-1, x=nx -> 0 (and y alike) into
// the 1-cell ring, so a TMA box of (TX+2) x (TY+2) cells around any tile is exactly the
// periodic neighbourhood, with no wrap logic in the consumer.
struct GridGeom {
    int nx, ny, nzl;
    int P;          // padded row pitch (elements)
    int64_t cs;     // component stride = (ny+2)*P
    int64_t ps;     // plane stride = 2*cs
};
void gs_tile_dims(int* tx, int* ty);
// 4D tensor map (x, y, c, z) over a padded array of `nplanes` planes; box = one tile + ring.
cudaError_t encode_grid_map(CUtensorMap* m, const double* base, const GridGeom& g, int nplanes);

// K3: fused Gray–Scott stage kernel.
struct GsStageArgs {
    CUtensorMap tm_u;
    CUtensorMap tm_k[kMaxSlots];
    CUtensorMap tm_glo, tm_ghi;  // ghost planes z=-1, z=nzl (multi-GPU); else periodic wrap
    GridGeom geo;
    const double* u;             // raw pointers (pack kernel)
    const double* k[kMaxSlots];
    double g[kMaxSlots];         // Y coefficient per slot (0: slot not in Y)
    double beta[kMaxSlots];      // final-combination weight per slot (0: skip)
    double delta[kMaxSlots];     // error weight per slot (0: skip)
    double beta_new, delta_new;  // weights of the k_i computed by this stage
    double* out_k;
    double* out_u;
    unsigned long long* errmax;
    double dt, atol, rtol;
    double d1, d2, F, FK, inv_h2;
    int has_glo, has_ghi;
    int z_lo, z_hi;              // output planes [z_lo, z_hi) (zmode 0)
    int zchunk;                  // output planes per CTA
    int zmode;                   // 0: contiguous chunks; 1: chunk 0 = plane 0, chunk 1 = nzl-1
    int nslots;
};
cudaError_t launch_gs_stage(int epi, const GsStageArgs& a, cudaStream_t st, int* nlaunch);

// Y_i on own planes 0 and nzl-1 (whole padded planes) -> send = [lo plane | hi plane].
cudaError_t launch_gs_pack(const GsStageArgs& a, double* send, cudaStream_t st);
// Refresh the periodic ring of every (plane, component) slice of a padded array (after a
// user copy into the interior); nslices = planes * components.
cudaError_t launch_fill_ring(double* a, const GridGeom& g, int nslices, cudaStream_t st);

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
