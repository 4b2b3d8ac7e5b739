// decode_body.cuh -- K3..K7 for one signal with the whole CTA: the
// sequential part of sfft4 over the bucket vectors produced by the encode.
// Shared by decode_kernel (one signal per CTA) and fused_kernel.
//   for every iteration m (proj/src/sfft4.cpp:38-113):
//     K3  subtract the prediction of the tones already found
//         (predict_buckets + subtract, proj/src/bucketize.cpp:70-104);
//     K4  stable order of buckets by |y0| desc, budget, 0.2*kth threshold
//         (sfft4.cpp:75-91);
//     K5  multiscale location, a lane group per selected bucket, lanes = the
//         l candidate blocks (locate_frequency / locate_step,
//         proj/src/locate.cpp:63-123);
//     K6  estimate y0/G, |G| < 0.5 reject, f = sigma^-1 u, per-iteration
//         found map, accumulate (sfft4.cpp:27-36, 92-105);
//   K7  keep the K largest (stable by |c| desc over ascending f), output in
//       ascending f (sfft4.cpp:170-178).
// Compiled with --fmad=false; every decision reads FP64 values computed with
// the reference's operation order.  G comes from the window's device table.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "cta_sort.cuh"
#include "encode.hpp"
#include "plan_dev.cuh"

#ifndef DEC_TL_MARK
#define DEC_TL_MARK(m) do { } while (0)
#endif

namespace msfft_b200 {
namespace {

struct DecShared {
    int acc_n, new_n, cur;
    double thr;
    // the iteration's locate stage table and first taus, copied from the
    // (grid-constant) plan at the top of each iteration: the stage chain of
    // K5 then reads shared memory instead of missing the constant cache once
    // per stage
    double st_len[kMaxStageTable], st_blk[kMaxStageTable];
    int64_t st_tau[kMaxStageTable];
};

struct DecArgs {
    double2* y;
    const int64_t* sigma;
    const int64_t* sigma_inv;
    int64_t* out_f;
    double2* out_c;
    int64_t* out_count;
    int32_t* err;
    int64_t* tr_bucket;
    int64_t* tr_f;
    double2* tr_v;
    // fused kernel only: before iteration m, wait until gate_done[m] reaches
    // gate_need[m] (encode tasks of this signal's chunk and iteration m)
    const int32_t* gate_done;
    const int32_t* gate_need;
};

__device__ __forceinline__ int32_t load_acquire(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct Scratch {
    dptr<int64_t> acc_f[2];
    dptr<double2> acc_c[2];
    dptr<int64_t> tone_u;
    dptr<int64_t> tone_i;
    dptr<double> mag;
    dptr<int32_t> order;
    dptr<int64_t> cand_f;
    dptr<double2> cand_v;
    dptr<int32_t> cand_first;
    dptr<double2> cand_sum;
    dptr<double2> rot;      // [tone][round] e^{-2 pi i tau_r u / n}; later the staged rounds
    dptr<int32_t> bstart;   // [b + 1] per-bucket list offsets
    dptr<int32_t> blist;    // [acc] tone indices grouped by bucket
    dptr<double2> gc;       // [acc][3] G * c per tone and bucket offset
    dptr<double> phi;       // [budget][stages] phase of y0 / y_tau
    dptr<int32_t> pcode;    // [budget][stages] 0 ok, 1 y_tau == 0, 2 quotient == 0
    dptr<uint64_t> sk[2];   // large sizes: radix-sort keys (ping-pong)
    dptr<int32_t> sv[2];    //              and values
    dptr<int32_t> flag;     //              scan flags
    dptr<int64_t> nfs;      //              new found frequencies
};

__device__ __forceinline__ double ghat_at(const DevIter& it, int64_t d) {
    return it.ghat[d + it.gmax];
}

// unit_root (proj/src/bucketize.cpp:12-18): e^{-2 pi i (e mod n)/n}; the
// division by the power of two n is an exact multiplication by 1/n.
__device__ __forceinline__ double2 unit_root(int64_t n, double inv_n, int64_t e) {
    e &= (n - 1);
    const double a = -kTwoPi * static_cast<double>(e) * inv_n;
    double s, c;
    sincos(a, &s, &c);
    return make_double2(c, s);
}

// ---- the locate stage chain (locate_frequency's narrowing loop,
// proj/src/locate.cpp:63-123) for one ranked bucket, shortest form.  The
// stage count and every stage's operands are known up front: each stage
// first loads the next stage's phase code and phase (clamped index, no
// branch), and per lane the next block offsets (j + 0.5) * rblk, the u_min
// steps (j - q/2) * rblk and tau/n are formed off the chain; the argmin
// carries the winner's step.  With the group size and the blocks per lane
// fixed at compile time a stage is one basic block, so those loads and
// products overlap the chain center -> phase -> distance -> argmin -> u_min.
// Every value equals the reference's: tau/n and the 1/n scalings are exact
// powers of two, so (center * tau/n) - trunc(..) is fmod(center * tau, n) /
// n, and round(f * 2pi) equals round(round(x * 2pi) / n) (locate.cpp:19-23).
//   phi/code: the bucket's per-stage phase and phase code (stage s at [s-1]);
//   st_blk[s-1]: block width of stage s; st_tau[s]: tau of stage s.
// Lanes glane = 0..GSZ-1 of the group hold blocks glane + i*GSZ.  Returns
// the final u_min; clears `ok` on a nullopt / throwing phase and raises
// kDecErrPhaseZero in *err for the latter.
template <int GSZ, int JPL, class PhiP, class CodeP, class BlkP, class TauP>
__device__ __forceinline__ double locate_stages(double u_min, int nst, bool live, bool& ok,
                                                int glane, int64_t lcfg, double hq, double inv_n,
                                                PhiP phi, CodeP code_p, BlkP st_blk, TauP st_tau,
                                                int32_t* err) {
    double jd[JPL];
    bool jv[JPL];
#pragma unroll
    for (int i = 0; i < JPL; ++i) {
        const int64_t j = glane + static_cast<int64_t>(i) * GSZ;
        jv[i] = j < lcfg;
        jd[i] = static_cast<double>(j);
    }
    const int last = nst > 0 ? nst - 1 : 0;
    int code = live && nst > 0 ? code_p[0] : 1;
    double ph = live && nst > 0 ? phi[0] : 0.0;
    double rb = st_blk[0];
    double offc[JPL], step[JPL];
#pragma unroll
    for (int i = 0; i < JPL; ++i) {
        offc[i] = (jd[i] + 0.5) * rb;
        step[i] = (jd[i] - hq) * rb;
    }
    double step0 = (0.0 - hq) * rb;  // block 0: every distance NaN
    double ton = static_cast<double>(st_tau[1]) * inv_n;
    bool err2 = false;
    for (int stage = 1; stage <= nst; ++stage) {
        // the next stage's operands (the last stage reloads its own)
        const int sn = stage < nst ? stage : last;
        const int code_n = live ? static_cast<int>(code_p[sn]) : 1;
        const double phi_n = live ? static_cast<double>(phi[sn]) : 0.0;
        const double rb_n = st_blk[sn];
        const int64_t tau_n = st_tau[sn + 1];
        // this stage's chain
        double best_d = INFINITY, best_step = step0;
        int best_j = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < JPL; ++i) {
            const double y = (u_min + offc[i]) * ton;
            double f = y - trunc(y);
            f = f < 0 ? f + 1.0 : f;
            const double d = circular_phase_distance(f * kTwoPi, ph);
            const bool better = jv[i] && d < best_d;
            best_d = better ? d : best_d;
            best_j = better ? glane + i * GSZ : best_j;
            best_step = better ? step[i] : best_step;
        }
        // 1: locate_frequency returns nullopt; 2: phase_of throws
        err2 = err2 || (ok && code == 2);
        ok = ok && code == 0;
        // lowest block index wins ties (strict < in ascending order)
#pragma unroll
        for (int o = GSZ >> 1; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, best_d, o);
            const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
            const double os = __shfl_xor_sync(0xffffffffu, best_step, o);
            const bool take = od < best_d || (od == best_d && oj < best_j);
            best_d = take ? od : best_d;
            best_j = take ? oj : best_j;
            best_step = take ? os : best_step;
        }
        u_min = u_min + best_step;
        code = code_n;
        ph = phi_n;
#pragma unroll
        for (int i = 0; i < JPL; ++i) {
            offc[i] = (jd[i] + 0.5) * rb_n;
            step[i] = (jd[i] - hq) * rb_n;
        }
        step0 = (0.0 - hq) * rb_n;
        ton = static_cast<double>(tau_n) * inv_n;
    }
    if (err2 && glane == 0) atomicCAS(err, 0, kDecErrPhaseZero);
    return u_min;
}

// locate_stages covers group sizes 2..16 with up to 4 blocks per lane
__device__ __forceinline__ bool locate_fast_ok(int gsz, int64_t jpl) {
    return jpl <= 4 && gsz >= 2 && gsz <= 16;
}

template <class PhiP, class CodeP, class BlkP, class TauP>
__device__ __forceinline__ double locate_stages_dispatch(int gsz, int64_t jpl, double u_min,
                                                         int nst, bool live, bool& ok, int glane,
                                                         int64_t lcfg, double hq, double inv_n,
                                                         PhiP phi, CodeP code, BlkP st_blk,
                                                         TauP st_tau, int32_t* err) {
#define MSFFT_LOCATE_G(G)                                                                  \
    do {                                                                                   \
        if (jpl == 1)                                                                      \
            return locate_stages<G, 1>(u_min, nst, live, ok, glane, lcfg, hq, inv_n, phi, code, \
                                       st_blk, st_tau, err);                               \
        if (jpl == 2)                                                                      \
            return locate_stages<G, 2>(u_min, nst, live, ok, glane, lcfg, hq, inv_n, phi, code, \
                                       st_blk, st_tau, err);                               \
        return locate_stages<G, 4>(u_min, nst, live, ok, glane, lcfg, hq, inv_n, phi, code,    \
                                   st_blk, st_tau, err);                                   \
    } while (0)
    if (gsz == 16) MSFFT_LOCATE_G(16);
    if (gsz == 8) MSFFT_LOCATE_G(8);
    if (gsz == 4) MSFFT_LOCATE_G(4);
    MSFFT_LOCATE_G(2);
#undef MSFFT_LOCATE_G
}

// Barrier of a decode group: the whole CTA (bar_id 0, __syncthreads) or a
// warp-aligned group of kThreads threads on named barrier bar_id.
template <int kThreads>
__device__ __forceinline__ void group_sync(int bar_id) {
    if (bar_id == 0)
        __syncthreads();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kThreads) : "memory");
}

// Decodes signal s with the kThreads threads starting at threadIdx.x ==
// grp_base (the whole CTA, or one half of it when a fused CTA decodes two
// signals); base = this signal's scratch (shared or global memory).  The
// large-size paths (cta_radix_sort) need the whole CTA.
template <int kThreads = kDecThreads>
__device__ __forceinline__ void decode_signal(const DevPlan& plan, const DecLayout& lay,
                                           const DecArgs& A, int64_t s, unsigned char* base,
                                           DecShared& sh, int* sort_smem, int grp_base = 0,
                                           int bar_id = 0) {
    const int tid = static_cast<int>(threadIdx.x) - grp_base;
    const auto gsync = [bar_id] { group_sync<kThreads>(bar_id); };
    const int lane = tid & 31;

    Scratch S;
    const int64_t cap = lay.cap, capb = cap > lay.b_max ? cap : lay.b_max;
    const int64_t bud = lay.budget_max, rmax = lay.rounds_max;
    const auto at = [base](int64_t off) { return base + off; };
    for (int p = 0; p < 2; ++p) {
        S.acc_f[p] = make_dptr(reinterpret_cast<int64_t*>(at(lay.off_acc_f[p])), cap);
        S.acc_c[p] = make_dptr(reinterpret_cast<double2*>(at(lay.off_acc_c[p])), cap);
    }
    S.tone_u = make_dptr(reinterpret_cast<int64_t*>(at(lay.off_tone_u)), cap);
    S.tone_i = make_dptr(reinterpret_cast<int64_t*>(at(lay.off_tone_i)), capb);
    S.mag = make_dptr(reinterpret_cast<double*>(at(lay.off_mag)), capb);
    S.order = make_dptr(reinterpret_cast<int32_t*>(at(lay.off_order)), lay.b_max);
    S.cand_f = make_dptr(reinterpret_cast<int64_t*>(at(lay.off_cand_f)), bud);
    S.cand_v = make_dptr(reinterpret_cast<double2*>(at(lay.off_cand_v)), bud);
    S.cand_first = make_dptr(reinterpret_cast<int32_t*>(at(lay.off_cand_first)), bud);
    S.cand_sum = make_dptr(reinterpret_cast<double2*>(at(lay.off_cand_sum)), bud);
    S.rot = make_dptr(reinterpret_cast<double2*>(at(lay.off_rot)), (cap > bud ? cap : bud) * rmax);
    S.bstart = make_dptr(reinterpret_cast<int32_t*>(at(lay.off_bstart)), lay.b_max + 1);
    S.blist = make_dptr(reinterpret_cast<int32_t*>(at(lay.off_blist)), cap);
    S.gc = make_dptr(reinterpret_cast<double2*>(at(lay.off_gc)), cap * 3);
    S.phi = make_dptr(reinterpret_cast<double*>(at(lay.off_phi)), bud * rmax);
    S.pcode = make_dptr(reinterpret_cast<int32_t*>(at(lay.off_pcode)), bud * rmax);
    const int64_t nsort = lay.big ? lay.sort_n : 0;
    for (int p = 0; p < 2; ++p) {
        S.sk[p] = make_dptr(lay.big ? reinterpret_cast<uint64_t*>(at(lay.off_sk[p])) : nullptr, nsort);
        S.sv[p] = make_dptr(lay.big ? reinterpret_cast<int32_t*>(at(lay.off_sv[p])) : nullptr, nsort);
    }
    S.flag = make_dptr(lay.big ? reinterpret_cast<int32_t*>(at(lay.off_flag)) : nullptr,
                       lay.big ? nsort + kThreads : 0);
    S.nfs = make_dptr(lay.big ? reinterpret_cast<int64_t*>(at(lay.off_nfs)) : nullptr, nsort);
    if (!lay.big) sort_smem = nullptr;

    if (tid == 0) {
        sh.acc_n = 0;
        sh.cur = 0;
    }
    gsync();

    const int64_t n = plan.n;
    const int64_t nmask = n - 1;
    const double inv_n = plan.inv_n;
    double2* ysig = A.y + s * plan.values_per_signal;

    int64_t sel_off = 0;  // trace offset: sum of earlier budgets
#ifdef MSFFT_DECODE_PROFILE
    long long prof_t[16];
#define DEC_MARK(id) do { if (tid == 0) prof_t[id] = clock64(); } while (0)
#else
#define DEC_MARK(id) do { } while (0)
#endif
    for (int m = 0; m < plan.iters; ++m) {
        DEC_MARK(0);
        if (A.gate_done) {  // fused: iteration m's buckets must be encoded
            if (tid == 0) {
                while (load_acquire(&A.gate_done[m]) < A.gate_need[m]) __nanosleep(64);
                __threadfence();
            }
            gsync();
#ifdef MSFFT_TIMELINE
            DEC_TL_MARK(m);
#endif
        }
        const DevIter& it = plan.it[m];
        const int64_t b = it.b, L = it.l_width;
        const double Ld = static_cast<double>(L);
        const double invL = 1.0 / Ld;  // exact: L is a power of two
        const int nr = it.nrounds;
        const int64_t* taus = plan.taus + it.tau_off;
        // stage tables of up to kMaxStageTable stages in shared memory (read
        // after the next group barrier, K3 or K4); longer schedules take the
        // general locate loop
        const int nst_tab = it.nstage_tab < kMaxStageTable ? it.nstage_tab : -1;
        if (tid < kMaxStageTable) {
            if (tid <= nst_tab) sh.st_len[tid] = it.stage_len[tid];
            if (tid < nst_tab) sh.st_blk[tid] = it.stage_blk[tid];
            sh.st_tau[tid] = tid < nr ? taus[tid] : 0;
        }
        const auto tau_at = [&](int r) { return r < kMaxStageTable ? sh.st_tau[r] : taus[r]; };
        const auto Y = make_dptr(ysig + it.yoff, static_cast<int64_t>(nr) * b);
        const int64_t sg = A.sigma[s * plan.iters + m];
        const int64_t sgi = A.sigma_inv[s * plan.iters + m];
        const int acc_n = sh.acc_n;
        const int cur = sh.cur;
        const auto AF = cur ? S.acc_f[1] : S.acc_f[0];
        const auto AC = cur ? S.acc_c[1] : S.acc_c[0];

        // ---- K3: subtract the prediction of everything already known.
        // predict_buckets (bucketize.cpp:84-93) adds, per known tone in
        // ascending f, (G_{jL-u} * c) * e^{-2 pi i tau u/n} into buckets
        // j = i-1, i, i+1.  Step 1 evaluates G*c per (tone, offset) and the
        // rotation per (tone, round) once; step 2 sums, per (round, bucket),
        // the contributions (G*c) * rot in ascending tone order -- the
        // reference's order and operands.
        if (acc_n > 0) {
            for (int j = tid; j < acc_n; j += kThreads) {
                const int64_t u = (sg * AF[j]) & nmask;
                const int64_t i = static_cast<int64_t>(floor(static_cast<double>(u) * invL + 0.5));
                S.tone_u[j] = u;
                S.tone_i[j] = i;
                // G_{jL-u} * c for the three buckets: independent of the round
                const double2 c = AC[j];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double g = ghat_at(it, (i - 1 + d) * L - u);
                    S.gc[j * 3 + d] = make_double2(g * c.x, g * c.y);
                }
            }
            gsync();
            DEC_MARK(1);
            // warps 1.. evaluate the rotations while warp 0 builds the lists
            static_assert(kThreads > 32, "the rotation loop needs warps besides warp 0");
            for (int e = tid - 32; e >= 0 && e < acc_n * nr; e += kThreads - 32) {
                const int j = e / nr, r = e - j * nr;
                S.rot[e] = unit_root(n, inv_n, tau_at(r) * S.tone_u[j]);
            }
            // per-bucket tone lists (ascending tone index = ascending f),
            // built by warp 0 while the other warps evaluate contributions:
            // counts, a scan, then a stable fill; lanes of a 32-tone chunk
            // that share a bucket are ranked with __match_any_sync.
            if (tid < 32) {
                const auto cnt = S.order;  // free until K4
                for (int64_t bk = tid; bk < b; bk += 32) cnt[bk] = 0;
                __syncwarp();
                for (int j0 = 0; j0 < acc_n; j0 += 32) {
                    const int j = j0 + tid;
                    const int bk = j < acc_n ? static_cast<int>(S.tone_i[j] & (b - 1)) : -1;
                    const unsigned grp = __match_any_sync(0xffffffffu, bk);
                    if (bk >= 0 && (grp & ((1u << tid) - 1u)) == 0) cnt[bk] += __popc(grp);
                    __syncwarp();
                }
                int carry = 0;  // exclusive scan -> bstart, cnt becomes the fill cursor
                for (int64_t base0 = 0; base0 < b; base0 += 32) {
                    const int64_t idx = base0 + tid;
                    const int c0 = idx < b ? cnt[idx] : 0;
                    int v = c0;
                    for (int o = 1; o < 32; o <<= 1) {
                        const int w = __shfl_up_sync(0xffffffffu, v, o);
                        if (tid >= o) v += w;
                    }
                    if (idx < b) {
                        S.bstart[idx] = carry + v - c0;
                        cnt[idx] = carry + v - c0;
                    }
                    carry += __shfl_sync(0xffffffffu, v, 31);
                }
                if (tid == 0) S.bstart[b] = carry;
                __syncwarp();
                for (int j0 = 0; j0 < acc_n; j0 += 32) {
                    const int j = j0 + tid;
                    const int bk = j < acc_n ? static_cast<int>(S.tone_i[j] & (b - 1)) : -1;
                    const unsigned grp = __match_any_sync(0xffffffffu, bk);
                    if (bk >= 0) {
                        const int pos = cnt[bk] + __popc(grp & ((1u << tid) - 1u));
                        S.blist[pos] = j;
                    }
                    __syncwarp();
                    if (bk >= 0 && (grp & ((1u << tid) - 1u)) == 0) cnt[bk] += __popc(grp);
                    __syncwarp();
                }
            }
            gsync();
            DEC_MARK(2);
            // bucket beta collects, in ascending tone order, the tones whose
            // own bucket is beta+1 (offset jj = i-1), beta (jj = i) and
            // beta-1 (jj = i+1): a three-way merge of the sorted lists.
            const int64_t total = static_cast<int64_t>(nr) * b;
            for (int64_t e = tid; e < total; e += kThreads) {
                const int r = static_cast<int>(e / b);
                const int64_t beta = e - r * b;
                int p[3], q3[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const int64_t bk = (beta + 1 - d) & (b - 1);
                    p[d] = S.bstart[bk];
                    q3[d] = S.bstart[bk + 1];
                }
                const double2 o = Y[e];  // issued before the merge walk
                double2 pred = make_double2(0.0, 0.0);
                bool any = false;
                for (;;) {
                    int best = -1, bj = 0x7fffffff;
#pragma unroll
                    for (int d = 0; d < 3; ++d)
                        if (p[d] < q3[d] && S.blist[p[d]] < bj) {
                            bj = S.blist[p[d]];
                            best = d;
                        }
                    if (best < 0) break;
                    ++p[best];
                    // the contribution G*c * rot, evaluated here (same operands)
                    const double2 v = cmul(S.gc[bj * 3 + best], S.rot[static_cast<int64_t>(bj) * nr + r]);
                    pred.x += v.x;
                    pred.y += v.y;
                    any = true;
                }
                if (any) Y[e] = make_double2(o.x - pred.x, o.y - pred.y);
            }
            gsync();
            DEC_MARK(3);
        }

        // ---- K4: stable descending order of |y0|, budget and threshold
        for (int64_t j = tid; j < b; j += kThreads) {
            const double2 v = Y[j];
            const double mg = cabs_ref(v.x, v.y);
            S.mag[j] = mg == mg ? mg : -1.0;  // NaN (unvalidated input) ranks last
        }
        gsync();
        DEC_MARK(4);
        if (b > kSmallRank && sort_smem) {
            // stable radix sort by |y0| descending (ties: lower bucket first)
            for (int64_t j = tid; j < b; j += kThreads) {
                S.sk[0][j] = desc_key(S.mag[j]);
                S.sv[0][j] = static_cast<int32_t>(j);
            }
            gsync();
            const bool fl = cta_radix_sort<kThreads>(S.sk[0], S.sv[0], S.sk[1], S.sv[1],
                                                     static_cast<int>(b), 64, sort_smem,
                                                     sort_smem + 16 * kThreads);
            const auto V = fl ? S.sv[1] : S.sv[0];
            for (int64_t j = tid; j < b; j += kThreads) S.order[j] = V[j];
        } else {
            for (int64_t j = tid; j < b; j += kThreads) {
                const double mj = S.mag[j];
                int64_t rank = 0;
                for (int64_t i = 0; i < b; ++i) {
                    const double mi = S.mag[i];
                    rank += (mi > mj) || (mi == mj && i < j);
                }
                S.order[rank] = static_cast<int32_t>(j);
            }
        }
        gsync();
        DEC_MARK(5);
        const int64_t budget = it.budget;
        if (tid == 0) sh.thr = 0.2 * S.mag[S.order[budget - 1]];
        gsync();
        DEC_MARK(6);
        const double thr = sh.thr;
        // every ranked bucket's round values, staged in shared memory in one
        // pass (the rotation area is free after K3): the locate stages
        // then never wait on L2
        const auto yr = S.rot;  // free after K3
        for (int64_t e = tid; e < budget * nr; e += kThreads) {
            const int64_t rk = e / nr, st = e - rk * nr;
            yr[e] = Y[st * b + S.order[rk]];
        }
        gsync();
        DEC_MARK(11);
        // phase_of(y0 / y_tau) (locate.cpp:110) depends only on the bucket
        // values, not on the narrowing region, so every (rank, stage) pair is
        // evaluated at once here; the stage chain below only scans blocks.
        // pcode: 0 ok, 1 y_tau == 0 (nullopt), 2 quotient == 0 (phase_of throws)
        const int ns = nr - 1;
        for (int64_t e = tid; e < budget * ns; e += kThreads) {
            const int64_t rk = e / ns, st = e - rk * ns + 1;
            const double2 y0e = yr[rk * nr], yt = yr[rk * nr + st];
            int code = 0;
            double ph = 0.0;
            if (yt.x == 0.0 && yt.y == 0.0) {
                code = 1;
            } else {
                const double2 z = cdiv_ref(y0e.x, y0e.y, yt.x, yt.y);
                if (z.x == 0.0 && z.y == 0.0) code = 2;
                ph = atan2(z.y, z.x);
                if (ph < 0.0) ph += kTwoPi;
                ph = ph + 0.0;
            }
            S.phi[e] = ph;
            S.pcode[e] = code;
        }
        gsync();
        DEC_MARK(12);

        // ---- K5 + K6: locate and estimate.  A group of `gsz` lanes takes one
        // ranked bucket; the region length evolves identically for every
        // bucket, so all groups run the same number of stages and the
        // shuffles stay convergent.
        // stage-chain operands converted once: q/2, n and the taus as doubles
        const int64_t lcfg = plan.l;
        const double q = plan.q, hq = plan.q / 2.0, nd_r = static_cast<double>(n), inv_n_r = inv_n;
        const int nst_r = nst_tab;
        // group size: enough lanes for the l blocks, shrunk (each lane then
        // scans several blocks) until every ranked bucket fits in one pass
        int gsz = lcfg > 16 ? 32 : (lcfg > 8 ? 16 : (lcfg > 4 ? 8 : 4));
        while (gsz > 1 && kThreads / gsz < budget) gsz >>= 1;
        const int glane = lane & (gsz - 1);
        const int groups = kThreads / gsz;
        const int gid = tid / gsz;
        const int64_t rounds_up = (budget + groups - 1) / groups * groups;
        const int first_gid_of_warp = (tid & ~31) / gsz;
        for (int64_t rank = gid; rank < rounds_up; rank += groups) {
            // a warp whose groups are all past the budget has nothing to
            // locate (warp-uniform, so no shuffle loses a participant)
            if (rank - (gid - first_gid_of_warp) >= budget) continue;
            const bool live = rank < budget;
            const int64_t beta = live ? S.order[rank] : 0;
            int64_t f_out = -1;
            double2 v_out = make_double2(0.0, 0.0);
            const double2 y0 = live ? yr[rank * nr] : make_double2(0.0, 0.0);
            bool ok = live && S.mag[beta] > thr;
            if (ok && y0.x == 0.0 && y0.y == 0.0) ok = false;
            double u_min = (2.0 * static_cast<double>(beta) - 1.0) * Ld / 2.0;
            double len = Ld;
            const int nst = nst_r;  // host-precomputed stage lengths (or -1)
            const int64_t jpl = (lcfg + gsz - 1) / gsz;  // blocks per lane
            if (nst >= 0 && nst < nr && locate_fast_ok(gsz, jpl)) {
#ifdef MSFFT_DECODE_PROFILE
                const long long t_chain0 = clock64();
#endif
                const int64_t pe0 = rank * ns;
                u_min = locate_stages_dispatch(gsz, jpl, u_min, nst, live, ok, glane, lcfg, hq,
                                               inv_n_r, &S.phi[pe0], &S.pcode[pe0], sh.st_blk,
                                               sh.st_tau, A.err);
                if (nst > 0) len = sh.st_len[nst];
#ifdef MSFFT_DECODE_PROFILE
                if (tid == 0 && s < 1)
                    printf("DECPROF chain m=%d nst=%d jpl=%lld gsz=%d cycles=%lld (%.0f per stage)\n", m,
                           nst, (long long)jpl, gsz, clock64() - t_chain0,
                           nst > 0 ? (double)(clock64() - t_chain0) / nst : 0.0);
#endif
            } else if (nst >= 0 && nst < nr) {
                // the usual case: the stage count and every stage's operands
                // are known up front, so the next stage's phase code, phase,
                // tau, block width and length load while this stage runs;
                // only center -> phase -> distance -> argmin -> u_min stays
                // on the dependent chain.  Same operations as the loop below.
                const int64_t pe0 = rank * ns;
                int code_n = live && nst > 0 ? S.pcode[pe0] : 1;
                double phi_n = live && nst > 0 ? S.phi[pe0] : 0.0;
                double rblk_n = sh.st_blk[0], len_n = sh.st_len[1];
                double tau_n = static_cast<double>(tau_at(1));
                for (int stage = 1; stage <= nst; ++stage) {
                    const int code = code_n;
                    const double phi = phi_n, rblk = rblk_n, nlen = len_n;
                    const double tau = tau_n;
                    if (stage < nst) {
                        if (live) {
                            code_n = S.pcode[pe0 + stage];
                            phi_n = S.phi[pe0 + stage];
                        }
                        rblk_n = sh.st_blk[stage];
                        len_n = sh.st_len[stage + 1];
                        tau_n = static_cast<double>(tau_at(stage + 1));
                    }
                    if (ok && code != 0) {
                        // 1: locate_frequency returns nullopt; 2: phase_of throws
                        if (code == 2 && glane == 0) atomicCAS(A.err, 0, kDecErrPhaseZero);
                        ok = false;
                    }
                    double best_d = INFINITY;
                    int best_j = 0x7fffffff;
                    for (int64_t j = glane; j < lcfg; j += gsz) {
                        const double center = u_min + (static_cast<double>(j) + 0.5) * rblk;
                        const double d = circular_phase_distance(
                            position_phase_d(center, tau, nd_r, inv_n_r), phi);
                        if (d < best_d) {
                            best_d = d;
                            best_j = static_cast<int>(j);
                        }
                    }
                    for (int o = gsz >> 1; o > 0; o >>= 1) {
                        const double od = __shfl_xor_sync(0xffffffffu, best_d, o);
                        const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
                        if (od < best_d || (od == best_d && oj < best_j)) {
                            best_d = od;
                            best_j = oj;
                        }
                    }
                    if (best_j == 0x7fffffff) best_j = 0;
                    u_min = u_min + (static_cast<double>(best_j) - hq) * rblk;
                    len = nlen;
                }
            } else {
                int stage = 0;
                while (nst >= 0 ? stage < nst : len > 1.0 + 1e-9) {
                    ++stage;
                    if (stage >= nr) {  // cannot happen for sfft4's own tau plans
                        if (ok && glane == 0) atomicCAS(A.err, 0, kDecErrRounds);
                        ok = false;
                        break;  // uniform: every group sees the same stage count
                    }
                    double phi = 0.0;
                    if (ok) {
                        const int64_t pe = rank * ns + (stage - 1);
                        const int code = S.pcode[pe];
                        if (code == 1) {
                            ok = false;  // locate_frequency returns nullopt
                        } else {
                            if (code == 2) {  // phase_of throws
                                if (glane == 0) atomicCAS(A.err, 0, kDecErrPhaseZero);
                                ok = false;
                            }
                            phi = S.phi[pe];
                        }
                    }
                    const int64_t tau = tau_at(stage);
                    const double rblk =
                        nst >= 0 ? sh.st_blk[stage - 1] : len / static_cast<double>(lcfg);
                    double best_d = INFINITY;
                    int best_j = 0x7fffffff;
                    for (int64_t j = glane; j < lcfg; j += gsz) {
                        const double center = u_min + (static_cast<double>(j) + 0.5) * rblk;
                        const double d = circular_phase_distance(
                            position_phase(center, tau, n, inv_n), phi);
                        if (d < best_d) {
                            best_d = d;
                            best_j = static_cast<int>(j);
                        }
                    }
                    // lowest block index wins ties (strict < in ascending order)
                    for (int o = gsz >> 1; o > 0; o >>= 1) {
                        const double od = __shfl_xor_sync(0xffffffffu, best_d, o);
                        const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
                        if (od < best_d || (od == best_d && oj < best_j)) {
                            best_d = od;
                            best_j = oj;
                        }
                    }
                    if (best_j == 0x7fffffff) best_j = 0;  // all distances NaN: reference keeps 0
                    u_min = u_min + (static_cast<double>(best_j) - q / 2.0) * rblk;
                    len = nst >= 0 ? sh.st_len[stage] : len * (q + 1.0) / static_cast<double>(lcfg);
                }
            }
            if (ok) {
                const double lo = u_min, hi = u_min + len;
                int64_t u = static_cast<int64_t>(ceil(lo));
                if (!(static_cast<double>(u) < hi)) u = llround(0.5 * (lo + hi));
                u &= nmask;  // u mod n (n is a power of two): locate.cpp:120-121
                const int64_t i = static_cast<int64_t>(floor(static_cast<double>(u) * invL + 0.5));
                const double g = ghat_at(it, i * L - u);
                if (!(fabs(g) < 0.5)) {
                    v_out = make_double2(y0.x / g, y0.y / g);
                    f_out = (sgi * u) & nmask;
                }
            }
            if (live && glane == 0) {
                S.cand_f[rank] = f_out;
                S.cand_v[rank] = v_out;
                if (A.tr_bucket) {
                    A.tr_bucket[sel_off + rank] = beta;
                    A.tr_f[sel_off + rank] = f_out;
                    A.tr_v[sel_off + rank] = v_out;
                }
            }
        }
        gsync();
        DEC_MARK(7);

        // ---- K6 (merge): found[f] = 0 + v_r1 + v_r2 + ... in rank order
        // (std::map operator[] then +=), then acc[f] += found[f].  The first
        // accepted rank of each f carries the sum; the found set is merged
        // into the ascending acc list (ping-pong buffers).
        const int nxt = cur ^ 1;
        const auto NF = nxt ? S.acc_f[1] : S.acc_f[0];
        const auto NC = nxt ? S.acc_c[1] : S.acc_c[0];
        if (tid == 0) sh.new_n = 0;
        if (budget > kSmallBudget && sort_smem) {
            // large budgets: stable sort of the accepted ranks by f (equal f
            // keep rank order), runs summed in rank order, then a merge of
            // the new f into the ascending acc list by binary searches
            const int padded = static_cast<int>((budget + kThreads - 1) / kThreads * kThreads);
            int key_bits = 4;
            while (key_bits < 62 && (uint64_t{1} << key_bits) <= static_cast<uint64_t>(n)) key_bits += 4;
            for (int64_t r = tid; r < budget; r += kThreads) {
                const int64_t fr = S.cand_f[r];
                S.sk[0][r] = fr >= 0 ? static_cast<uint64_t>(fr) : static_cast<uint64_t>(n);
                S.sv[0][r] = static_cast<int32_t>(r);
            }
            for (int r = tid; r < padded; r += kThreads) S.flag[r] = 0;
            gsync();
            const bool fl = cta_radix_sort<kThreads>(S.sk[0], S.sv[0], S.sk[1], S.sv[1],
                                                     static_cast<int>(budget), key_bits,
                                                     sort_smem, sort_smem + 16 * kThreads);
            const auto Ks = fl ? S.sk[1] : S.sk[0];
            const auto Vs = fl ? S.sv[1] : S.sv[0];
            for (int64_t p = tid; p < budget; p += kThreads) {
                const uint64_t f = Ks[p];
                if (f >= static_cast<uint64_t>(n) || (p > 0 && Ks[p - 1] == f)) continue;
                double2 sum = make_double2(0.0, 0.0);
                for (int64_t p2 = p; p2 < budget && Ks[p2] == f; ++p2) {
                    const double2 v = S.cand_v[Vs[p2]];
                    sum.x += v.x;
                    sum.y += v.y;
                }
                S.cand_sum[Vs[p]] = sum;
                int lo = 0, hi = acc_n;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (static_cast<uint64_t>(AF[mid]) < f) lo = mid + 1; else hi = mid;
                }
                const bool present = lo < acc_n && static_cast<uint64_t>(AF[lo]) == f;
                S.flag[p] = present ? 0 : 1;
                S.nfs[p] = present ? -2 : -1;  // marks a run start (-1 new, -2 present)
            }
            gsync();
            // flag -> index among the new f; remember which positions start runs
            for (int64_t p = tid; p < budget; p += kThreads) {
                const uint64_t f = Ks[p];
                const bool start = f < static_cast<uint64_t>(n) && !(p > 0 && Ks[p - 1] == f);
                S.cand_first[p] = start ? (S.flag[p] ? 1 : 2) : 0;  // indexed by position here
            }
            gsync();
            const int nnew = cta_exclusive_scan<kThreads>(S.flag, padded, sort_smem + 16 * kThreads);
            for (int64_t p = tid; p < budget; p += kThreads)
                if (S.cand_first[p] == 1) S.nfs[S.flag[p]] = static_cast<int64_t>(Ks[p]);
            gsync();
            for (int j = tid; j < acc_n; j += kThreads) {
                const int64_t fj = AF[j];
                int lo = 0, hi = nnew;  // new f below fj
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (S.nfs[mid] < fj) lo = mid + 1; else hi = mid;
                }
                const int before = lo;
                int plo = 0, phi2 = static_cast<int>(budget);  // run of fj among the found
                while (plo < phi2) {
                    const int mid = (plo + phi2) >> 1;
                    if (Ks[mid] < static_cast<uint64_t>(fj)) plo = mid + 1; else phi2 = mid;
                }
                double2 c = AC[j];
                if (plo < budget && Ks[plo] == static_cast<uint64_t>(fj)) {
                    const double2 add = S.cand_sum[Vs[plo]];
                    c = make_double2(c.x + add.x, c.y + add.y);
                }
                NF[j + before] = fj;
                NC[j + before] = c;
            }
            for (int64_t p = tid; p < budget; p += kThreads) {
                if (S.cand_first[p] != 1) continue;
                const int64_t fr = static_cast<int64_t>(Ks[p]);
                int lo = 0, hi = acc_n;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (AF[mid] < fr) lo = mid + 1; else hi = mid;
                }
                const double2 sum = S.cand_sum[Vs[p]];
                NF[lo + S.flag[p]] = fr;
                NC[lo + S.flag[p]] = make_double2(0.0 + sum.x, 0.0 + sum.y);
            }
            if (tid == 0) sh.new_n = nnew;
        } else {
        // cand_first[r]: 0 = not the first accepted rank of its f,
        // 1 = first and f is new, 2 = first and f already accumulated.
        for (int64_t r = tid; r < budget; r += kThreads) {
            const int64_t fr = S.cand_f[r];
            int first = fr >= 0;
            for (int64_t r2 = 0; first && r2 < r; ++r2) first = S.cand_f[r2] != fr;
            if (first) {
                double2 sum = make_double2(0.0, 0.0);
                for (int64_t r2 = r; r2 < budget; ++r2)
                    if (S.cand_f[r2] == fr) {
                        sum.x += S.cand_v[r2].x;
                        sum.y += S.cand_v[r2].y;
                    }
                S.cand_sum[r] = sum;
                int lo = 0, hi = acc_n;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (AF[mid] < fr) lo = mid + 1; else hi = mid;
                }
                if (lo < acc_n && AF[lo] == fr) first = 2;
            }
            S.cand_first[r] = first;
        }
        gsync();
        DEC_MARK(8);
        // acc entries move up by the number of NEW found f below them
        for (int j = tid; j < acc_n; j += kThreads) {
            const int64_t fj = AF[j];
            int64_t before = 0;
            int64_t hit = -1;
            for (int64_t r = 0; r < budget; ++r) {
                const int cf = S.cand_first[r];
                if (!cf) continue;
                const int64_t fr = S.cand_f[r];
                if (cf == 1 && fr < fj) ++before;
                if (cf == 2 && fr == fj) hit = r;
            }
            double2 c = AC[j];
            if (hit >= 0) c = make_double2(c.x + S.cand_sum[hit].x, c.y + S.cand_sum[hit].y);
            NF[j + before] = fj;
            NC[j + before] = c;
        }
        // new f: insert at #{acc f < f} + #{new found f < f}
        for (int64_t r = tid; r < budget; r += kThreads) {
            if (S.cand_first[r] != 1) continue;
            const int64_t fr = S.cand_f[r];
            int lo = 0, hi = acc_n;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (AF[mid] < fr) lo = mid + 1; else hi = mid;
            }
            int64_t ubefore = 0;
            for (int64_t r3 = 0; r3 < budget; ++r3)
                ubefore += S.cand_first[r3] == 1 && S.cand_f[r3] < fr;
            const int64_t pos = lo + ubefore;
            const double2 sum = S.cand_sum[r];
            NF[pos] = fr;
            NC[pos] = make_double2(0.0 + sum.x, 0.0 + sum.y);
            atomicAdd(&sh.new_n, 1);
        }
        }  // small-budget merge
        gsync();
        DEC_MARK(9);
        if (tid == 0) {
            sh.acc_n = acc_n + sh.new_n;
            sh.cur = nxt;
        }
        sel_off += budget;
        gsync();
        DEC_MARK(10);
#ifdef MSFFT_DECODE_PROFILE
        if (tid == 0 && s < 2)
            printf("DECPROF s=%lld m=%d acc=%d b=%lld budget=%lld | K3 %lld %lld %lld | K4 %lld %lld %lld | K5 %lld %lld %lld | K6 %lld %lld %lld\n",
                   (long long)s, m, acc_n, (long long)b, (long long)budget,
                   acc_n ? prof_t[1] - prof_t[0] : 0LL, acc_n ? prof_t[2] - prof_t[1] : 0LL,
                   acc_n ? prof_t[3] - prof_t[2] : 0LL,
                   prof_t[4] - (acc_n ? prof_t[3] : prof_t[0]), prof_t[5] - prof_t[4],
                   prof_t[6] - prof_t[5], prof_t[11] - prof_t[6], prof_t[12] - prof_t[11], prof_t[7] - prof_t[12], prof_t[8] - prof_t[7],
                   prof_t[9] - prof_t[8], prof_t[10] - prof_t[9]);
#endif
    }

    // ---- K7: keep the K largest |c| (stable over ascending f), emit in f order
    const int acc_n = sh.acc_n;
    const int cur = sh.cur;
    const auto AF = cur ? S.acc_f[1] : S.acc_f[0];
    const auto AC = cur ? S.acc_c[1] : S.acc_c[0];
    const int64_t K = plan.k;
    for (int j = tid; j < acc_n; j += kThreads) {
        const double2 c = AC[j];
        const double mg = cabs_ref(c.x, c.y);
        S.mag[j] = mg == mg ? mg : -1.0;
    }
    gsync();
    if (acc_n > kSmallAcc && sort_smem) {
        // stable sort by |c| descending over ascending f; keep ranks < K;
        // output positions by a prefix count over f order
        const int padded = (acc_n + kThreads - 1) / kThreads * kThreads;
        for (int j = tid; j < acc_n; j += kThreads) {
            S.sk[0][j] = desc_key(S.mag[j]);
            S.sv[0][j] = j;
        }
        for (int j = tid; j < padded; j += kThreads) S.flag[j] = 0;
        gsync();
        const bool fl = cta_radix_sort<kThreads>(S.sk[0], S.sv[0], S.sk[1], S.sv[1], acc_n, 64,
                                                 sort_smem, sort_smem + 16 * kThreads);
        const auto V = fl ? S.sv[1] : S.sv[0];
        for (int r = tid; r < acc_n && r < K; r += kThreads) S.flag[V[r]] = 1;
        gsync();
        for (int j = tid; j < acc_n; j += kThreads) S.tone_i[j] = S.flag[j];
        gsync();
        cta_exclusive_scan<kThreads>(S.flag, padded, sort_smem + 16 * kThreads);
        for (int j = tid; j < acc_n; j += kThreads) {
            if (!S.tone_i[j]) continue;
            const int64_t pos = S.flag[j];
            MSFFT_DCHECK(pos >= 0 && pos < K);
            A.out_f[s * K + pos] = AF[j];
            A.out_c[s * K + pos] = AC[j];
        }
    } else {
        for (int j = tid; j < acc_n; j += kThreads) {
            const double mj = S.mag[j];
            int64_t rank = 0;
            for (int i = 0; i < acc_n; ++i) {
                const double mi = S.mag[i];
                rank += (mi > mj) || (mi == mj && i < j);
            }
            S.tone_i[j] = rank < K ? 1 : 0;
        }
        gsync();
        for (int j = tid; j < acc_n; j += kThreads) {
            if (!S.tone_i[j]) continue;
            int64_t pos = 0;
            for (int i = 0; i < j; ++i) pos += S.tone_i[i];
            MSFFT_DCHECK(pos >= 0 && pos < K);
            A.out_f[s * K + pos] = AF[j];
            A.out_c[s * K + pos] = AC[j];
        }
    }
    if (tid == 0) A.out_count[s] = acc_n < K ? acc_n : K;
}

}  // namespace
}  // namespace msfft_b200
