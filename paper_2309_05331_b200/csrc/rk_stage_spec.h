// rk_stage_spec.h — compile-time description of every fused stage launch.
//
// One table, used by the host scheduler (which k buffers to bind, which coefficients) and
// by the device kernels (which terms exist), so zero Butcher coefficients are skipped at
// compile time on the GPU exactly where the oracle skips them (R-17).
//
// Fixed step (do_step / integrate_const): stages 0..L, L = last j with b_j != 0; stage L is
// fused with u_new = u + sum beta_j k_j (EPI_FINAL).
// Adaptive, no FSAL (CK54): stage L fused with u_new and the error ratio (EPI_FINAL_ERR).
// Adaptive, FSAL (DOPRI5, row s == b, b_s == 0): stage s-1 writes u_new and the partial
// error sum e' = sum_{j<s} delta_j k_j (EPI_FINAL_EPART, into k_{s-1}'s buffer, which no
// later stage needs); stage s reads Y_s = u_new directly (a_sj = b_j), computes
// k_s = F(u_new) (the next step's k1), e = e' + delta_s k_s and the ratio (EPI_TAIL_ERR).
// That is 31 arrays per try instead of 33.
// The adaptive flag `ad` also names the error-ratio reading: 1 = Odeint's
// r = |e|/(atol + rtol(|u| + dt|k1|)) (R-12), 2 = SPEC's r = |e|/(atol + rtol max(|u|, |u_new|))
// (R-28), which needs no k1: the FSAL tail then reads e' and u only (30 arrays).
#pragma once
#include "rk_tableau.h"

namespace rkb {

enum Epilogue {
    EPI_K = 0,            // store k_i
    EPI_FINAL = 1,        // store u_new = w + beta_i k_i
    EPI_FINAL_ERR = 2,    // EPI_FINAL + error ratio max
    EPI_FINAL_EPART = 3,  // EPI_FINAL + store e' = e + delta_i k_i
    EPI_TAIL_ERR = 4,     // Y = u_new (base); store k_i; e = e' + delta_i k_i; ratio max
    EPI_AB = 5,           // Adams–Bashforth: store f_n; u_new = u + g_0 f_n + sum_s g_s h_s
    EPI_ABM = 6,          // ABM corrector: Y = u_p (slots), u_new = u + m_0 F(u_p) + sum_s m_s h_s
    EPI_AHEAD = 7         // stage before the final one: store Y_F = u + sum a_Fj k_j (tile + ring),
                          // W = u + sum b_j k_j and (adaptive) E = sum e_j k_j, all through j = i
};

// Scheme ids of the Adams–Bashforth k-step methods (rk_b200.h RK_ADAMS_BASHFORTH1..8).
constexpr int kSchemeAB0 = 10;
__host__ __device__ constexpr bool is_ab_scheme(int S) { return S > kSchemeAB0 && S <= kSchemeAB0 + 8; }
// ... and of the Adams–Bashforth–Moulton (PECE) methods (RK_ADAMS_BASHFORTH_MOULTON1..8)
constexpr int kSchemeABM0 = 20;
__host__ __device__ constexpr bool is_abm_scheme(int S) { return S > kSchemeABM0 && S <= kSchemeABM0 + 8; }
// schemes whose slots are Adams history entries (resolved by the host's history ring)
__host__ __device__ constexpr bool is_multistep(int S) { return is_ab_scheme(S) || is_abm_scheme(S); }

constexpr int kMaxSlots = 10;  // RKF78 adaptive final stage: k1, k4..k12
constexpr int SLOT_U = -1;  // slot source: the state u itself (TAIL stage: old u)

struct StageSpec {
    int valid = 0;
    int epi = EPI_K;
    int nslots = 0;
    int src[kMaxSlots] = {};               // k index (>= 0) or SLOT_U
    bool halo[kMaxSlots] = {};             // slot enters Y (needs the periodic ring)
    bool gnz[kMaxSlots] = {}, bnz[kMaxSlots] = {}, dnz[kMaxSlots] = {};
    int j[kMaxSlots] = {};                 // stage index of the slot (coefficients)
    bool bnew = false, dnew = false;       // beta_i / delta_i nonzero
    int out_k = -1;                        // k buffer written (EPI_K, EPI_FINAL_EPART e', TAIL k_s)
    bool writes_u = false;                 // stores u_new
    bool base_unew = false;                // TAIL: array 0 (Y source) is u_new, used as is
    int den_u = SLOT_U - 1;                // TAIL: slot holding old u for the ratio (else base)
    int den_k1 = -1;                       // slot holding k1 for the ratio
    int epart = -1;                        // TAIL: slot holding e'
    // "write ahead": the stage A = F-1 before the final-combination stage F
    // stores F's stage value and the partial final / error sums instead of k_A, so stage F
    // reads one halo array and one or two own-cell arrays instead of u and every k_j.
    bool anz2[kMaxSlots] = {};             // AHEAD: a_Fj != 0 (slot enters Y_F)
    bool a2new = false;                    // AHEAD: a_FA != 0
    int out_w = -1, out_e = -1;            // AHEAD: k buffers receiving W and E
    int base_src = -1;                     // F after AHEAD: k buffer holding Y_F (the base)
    int wslot = -1, eslot = -1;            // F after AHEAD: slots holding W and E
    // AHEAD for a K8 fixed-step tail pair (ad == 5): the stage i = L-2 also stores the base of the
    // last stage's value, Z_L = u + sum_{j<=i} a_Lj k_j (tile + ring), into k buffer out_z
    bool anz3[kMaxSlots] = {};             // a_Lj != 0
    bool a3new = false;                    // a_Li != 0
    int out_z = -1;
};

__host__ __device__ constexpr bool t_anz(const Tableau& T, int i, int j) { return rat_nz(T.a[i][j]); }
__host__ __device__ constexpr bool t_bnz(const Tableau& T, int j) { return rat_nz(T.b[j]); }
__host__ __device__ constexpr bool t_enz(const Tableau& T, int j) { return rat_nz(err_weight(T, j)); }
__host__ __device__ constexpr int last_stage(const Tableau& T, bool ad);
__host__ __device__ constexpr bool is_fsal(const Tableau& T, bool ad);

__host__ __device__ constexpr int last_stage(const Tableau& T, bool ad) {
    int last = 0;
    for (int j = 0; j < T.s; ++j)
        if (t_bnz(T, j) || (ad && t_enz(T, j))) last = j;
    return last;
}

__host__ __device__ constexpr bool is_fsal(const Tableau& T, bool ad) {
    if (!ad || T.err_order == 0) return false;
    const int L = last_stage(T, true);
    if (t_bnz(T, L)) return false;
    for (int j = 0; j < L; ++j)
        if (T.a[L][j].n * T.b[j].d != T.b[j].n * T.a[L][j].d) return false;
    return true;
}

// Index of the final-combination stage (u_new): the last stage, or the one before DOPRI5's tail.
__host__ __device__ constexpr int fin_stage(const Tableau& T, bool ad) {
    return is_fsal(T, ad) ? last_stage(T, ad) - 1 : last_stage(T, ad);
}

// Whether the final stage F is fed by a write-ahead stage A = F-1: only for fixed steps and
// FSAL error control (a non-FSAL error stage needs u and k1 at F for the ratio), and only if
// it moves fewer arrays (reads + writes of stages A and F) and fits the slot limit.
__host__ __device__ constexpr bool use_ahead(const Tableau& T, int ad) {
    if (T.s == 0 || (ad && T.err_order == 0)) return false;
    const bool fsal = is_fsal(T, ad != 0);
    if (ad && !fsal) return false;
    const int F = fin_stage(T, ad != 0), A = F - 1;
    if (A < 0) return false;
    int curA = 2, curF = 1 + (ad ? 2 : 1), ahA = 1 + 2 + (ad ? 1 : 0), ahF = 1 + 1 + (ad ? 1 : 0) + (ad ? 2 : 1);
    int slotsA = 0;
    for (int j = 0; j < A; ++j) {
        if (t_anz(T, A, j)) ++curA;
        const bool needF = t_anz(T, F, j) || t_bnz(T, j) || (ad && t_enz(T, j));
        if (needF) ++curF;
        if (t_anz(T, A, j) || needF) {
            ++ahA;
            ++slotsA;
        }
    }
    if (t_anz(T, F, A) || t_bnz(T, A) || (ad && t_enz(T, A))) ++curF;  // k_A itself
    return slotsA <= kMaxSlots && ahA + ahF < curA + curF;
}

// Tile rows per thread in the stencil kernel (1 or 2).  Two-row tiles (32x16) amortise the
// per-plane overhead of the light stages (at most one k input, or Adams–Bashforth k <= 4,
// whose extra inputs are own-cell only) and halve their ring re-reads.
__host__ __device__ constexpr int stage_rows(const StageSpec& P) {
    return (P.nslots <= 1 || (P.epi == EPI_AB && P.nslots <= 3)) ? 2 : 1;
}

__host__ __device__ constexpr int num_stages(int S, bool ad) {
    return is_multistep(S) ? 1 : last_stage(tableau_of(S), ad) + 1;
}

__host__ __device__ constexpr StageSpec stage_spec(int S, int ad, int i) {
    StageSpec p{};
    if (is_ab_scheme(S)) {
        // one RHS evaluation per step: base = u_n (tile + ring), slots = f_{n-1} .. f_{n-k+1}
        // (own cells only, newest first); the host binds out_k to a free history buffer
        if (ad || i != 0) return p;
        const int k = S - kSchemeAB0;
        p.valid = 1;
        p.epi = EPI_AB;
        p.nslots = k - 1;
        for (int s = 0; s < k - 1; ++s) {
            p.src[s] = s;  // history position (newest first), resolved by the host
            p.j[s] = s + 1;
            p.bnz[s] = true;
        }
        p.bnew = true;
        p.writes_u = true;
        p.out_k = k > 1 ? 0 : -1;  // AB1 (= Euler) keeps no history: f_n is never read again
        return p;
    }
    if (is_abm_scheme(S)) {
        // PEC of one PECE step (the final E, F(u_{n+1}), is the next step's k1-type launch):
        // slot 0 = f_n (history scratch, just evaluated), slot s = f_{n-s}; all enter
        // Y = u_p = u + sum_s (dt beta_s) slot_s; the corrector adds m_0 F(u_p) first, then
        // m_{s+1} slot_s for s < k-1 (newest first, R-26).  No k is stored.
        if (ad || i != 0) return p;
        const int k = S - kSchemeABM0;
        p.valid = 1;
        p.epi = EPI_ABM;
        p.nslots = k;
        for (int s = 0; s < k; ++s) {
            p.src[s] = s == 0 ? k - 1 : s - 1;  // history ring positions (host rk_runtime.cu)
            p.j[s] = s;
            p.halo[s] = true;
            p.gnz[s] = true;
            p.bnz[s] = s < k - 1;
        }
        p.bnew = true;
        p.writes_u = true;
        return p;
    }
    const Tableau T = tableau_of(S);
    if (ad == 5) {  // fixed step whose last two stages run as one K8 pair (L-1, L): stages 0..L-3
                    // as usual, stage L-2 writes ahead Y_{L-1} (the pair's source, ring), Z_L (the
                    // pair's base, ring) and W = u + sum_{j<=L-2} b_j k_j (own cells)
        const int L5 = last_stage(T, false);
        if (T.s < 4 || L5 < 3 || i < 0 || i > L5 - 2) return p;
        if (i < L5 - 2) return stage_spec(S, 0, i);
        for (int j = 0; j < i; ++j) {
            const bool need = t_anz(T, i, j) || t_anz(T, i + 1, j) || t_anz(T, i + 2, j) || t_bnz(T, j);
            if (!need) continue;
            const int s = p.nslots++;
            if (s >= kMaxSlots) return StageSpec{};  // does not fit: not offered (fixed_tail_ok)
            p.src[s] = j;
            p.j[s] = j;
            p.halo[s] = t_anz(T, i, j);
            p.gnz[s] = t_anz(T, i, j);
            p.anz2[s] = t_anz(T, i + 1, j);
            p.anz3[s] = t_anz(T, i + 2, j);
            p.bnz[s] = t_bnz(T, j);
        }
        p.valid = 1;
        p.epi = EPI_AHEAD;
        p.a2new = t_anz(T, i + 1, i);
        p.a3new = t_anz(T, i + 2, i);
        p.bnew = t_bnz(T, i);
        p.out_k = i;      // Y_{L-1} into k_i's buffer (k_i is never stored)
        p.out_z = i + 1;  // Z_L into k_{L-1}'s buffer (never stored)
        p.out_w = i + 2;  // W into k_L's buffer (never stored)
        return p;
    }
    if (ad == 4) {  // fixed step, the last stage fed by a K8 pair that wrote ahead Y_L (k buffer 0,
                    // with its ring) and W = u + sum_{j<L} b_j k_j (k buffer 1): Y-direct, u_new = W + b_L k_L
        const int L4 = last_stage(T, false);
        if (T.s < 3 || i != L4) return p;
        p.valid = 1;
        p.epi = EPI_FINAL;
        p.base_src = 0;
        p.nslots = 1;
        p.src[0] = 1;
        p.j[0] = L4 - 1;
        p.wslot = 0;
        p.writes_u = true;
        p.bnew = t_bnz(T, L4);
        return p;
    }
    if (T.s == 0 || (ad && T.err_order == 0)) return p;
    const int L = last_stage(T, ad);
    if (i < 0 || i > L) return p;
    const bool fsal = is_fsal(T, ad);
    p.valid = 1;
    if (fsal && i == L) {  // TAIL: Y_s = u_new, slots e' (k_{L-1} buffer), u, k1 (Odeint ratio)
        p.epi = EPI_TAIL_ERR;
        p.base_unew = true;
        p.nslots = ad == 2 ? 2 : 3;
        p.src[0] = L - 1; p.j[0] = L - 1;
        p.src[1] = SLOT_U; p.j[1] = 0;
        p.src[2] = 0; p.j[2] = 0;
        p.epart = 0;
        p.den_u = 1;
        p.den_k1 = ad == 2 ? -1 : 2;
        p.dnew = t_enz(T, i);
        p.out_k = 1;  // k2's buffer: dead after the stage values (a_s2 = 0 for DOPRI5)
        return p;
    }
    const bool fin = fsal ? (i == L - 1) : (i == L);
    const bool err = ad && fin;
    const int F = fin_stage(T, ad != 0);
    if (use_ahead(T, ad) && i == F - 1) {  // AHEAD: Y_F, W (and E) at own cells
        for (int j = 0; j < i; ++j) {
            const bool need = t_anz(T, i, j) || t_anz(T, F, j) || t_bnz(T, j) || (ad && t_enz(T, j));
            if (!need) continue;
            const int s = p.nslots++;
            p.src[s] = j;
            p.j[s] = j;
            p.halo[s] = t_anz(T, i, j);
            p.gnz[s] = t_anz(T, i, j);
            p.anz2[s] = t_anz(T, F, j);
            p.bnz[s] = t_bnz(T, j);
            p.dnz[s] = ad && t_enz(T, j);
        }
        p.epi = EPI_AHEAD;
        p.a2new = t_anz(T, F, i);
        p.bnew = t_bnz(T, i);
        p.dnew = ad && t_enz(T, i);
        p.out_k = i;                        // Y_F into k_A's buffer (k_A is never stored)
        p.out_w = ad ? F + 1 : F;           // fixed: k_F's buffer (never stored)
        p.out_e = ad ? F + 2 : -1;          // FSAL: k_F's buffer receives e' at stage F
        return p;
    }
    if (use_ahead(T, ad) && i == F) {  // final stage fed by AHEAD: Y_F is the base (Y-direct)
        p.base_src = F - 1;
        p.nslots = ad ? 2 : 1;
        p.src[0] = ad ? F + 1 : F;
        p.j[0] = F - 1;
        p.wslot = 0;
        if (ad) {
            p.src[1] = F + 2;
            p.j[1] = F - 1;
            p.eslot = 1;
        }
        p.writes_u = true;
        p.bnew = t_bnz(T, i);
        if (!ad) {
            p.epi = EPI_FINAL;
        } else {
            p.epi = EPI_FINAL_EPART;
            p.dnew = t_enz(T, i);
            p.out_k = i;
        }
        return p;
    }
    for (int j = 0; j < i; ++j) {
        const bool need = t_anz(T, i, j) || (fin && t_bnz(T, j)) || (err && (t_enz(T, j) || (ad == 1 && j == 0)));
        if (!need) continue;
        const int s = p.nslots++;
        p.src[s] = j;
        p.j[s] = j;
        p.halo[s] = t_anz(T, i, j);
        p.gnz[s] = t_anz(T, i, j);
        p.bnz[s] = fin && t_bnz(T, j);
        p.dnz[s] = err && t_enz(T, j);
        if (err && ad == 1 && j == 0) p.den_k1 = s;
    }
    if (!fin) {
        p.epi = EPI_K;
        p.out_k = i;
    } else {
        p.writes_u = true;
        p.bnew = t_bnz(T, i);
        if (!ad) {
            p.epi = EPI_FINAL;
        } else if (fsal) {
            p.epi = EPI_FINAL_EPART;
            p.dnew = t_enz(T, i);
            p.out_k = i;  // e' into k_i's own buffer (k_i itself is not needed later)
        } else {
            p.epi = EPI_FINAL_ERR;
            p.dnew = t_enz(T, i);
        }
    }
    return p;
}

}  // namespace rkb
