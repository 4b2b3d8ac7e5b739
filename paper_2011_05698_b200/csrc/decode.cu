// decode.cu -- K3..K7: one persistent CTA per signal runs the whole
// sequential part of sfft4 over the bucket vectors produced by the encode:
//   for every iteration m (proj/src/sfft4.cpp:38-113):
//     K3  subtract the prediction of the tones already found
//         (predict_buckets + subtract, proj/src/bucketize.cpp:70-104);
//     K4  stable order of buckets by |y0| desc, budget, 0.2*kth threshold
//         (sfft4.cpp:75-91);
//     K5  multiscale location, one warp per selected bucket, lanes = the l
//         candidate blocks (locate_frequency / locate_step,
//         proj/src/locate.cpp:63-123);
//     K6  estimate y0/G, |G| < 0.5 reject, f = sigma^-1 u, per-iteration
//         found map, accumulate (sfft4.cpp:27-36, 92-105);
//   K7  keep the K largest (stable by |c| desc over ascending f), output in
//       ascending f (sfft4.cpp:170-178).
// Compiled with --fmad=false; every decision reads FP64 values computed with
// the reference's operation order.  G comes from the window's device table.
#include <cuda_runtime.h>

#include "common.cuh"
#include "encode.hpp"

#ifndef MSFFT_DEC_MINB
#define MSFFT_DEC_MINB 3  // 3 CTAs per SM: <= 85 registers, no spills
#endif

namespace msfft_b200 {

namespace {

struct Scratch {
    int64_t* acc_f[2];
    double2* acc_c[2];
    int64_t* tone_u;
    int64_t* tone_i;
    double* mag;
    int32_t* order;
    int64_t* cand_f;
    double2* cand_v;
    int32_t* cand_first;
    double2* cand_sum;
    double2* contrib;  // [tone][round][3] predicted contributions
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

__global__ void __launch_bounds__(kDecThreads, MSFFT_DEC_MINB)
decode_kernel(const __grid_constant__ DevPlan plan, DecLayout lay, double2* __restrict__ y,
              const int64_t* __restrict__ sigma, const int64_t* __restrict__ sigma_inv,
              int64_t batch, unsigned char* __restrict__ work, int64_t* __restrict__ out_f,
              double2* __restrict__ out_c, int64_t* __restrict__ out_count,
              int32_t* __restrict__ err, int64_t* __restrict__ tr_bucket,
              int64_t* __restrict__ tr_f, double2* __restrict__ tr_v) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ int s_acc_n, s_new_n, s_cur;
    __shared__ double s_thr;

    const int64_t s = blockIdx.x;
    // err[1]: the validation pass found a non-finite sample; the call will
    // throw (ComplexSignal::validate) so there is nothing to decode.
    if (s >= batch || err[1] != 0) return;
    const int tid = threadIdx.x;
    const int lane = tid & 31;

    unsigned char* base = lay.in_smem ? dsm : work + s * lay.bytes;
    Scratch S;
    for (int p = 0; p < 2; ++p) {
        S.acc_f[p] = reinterpret_cast<int64_t*>(base + lay.off_acc_f[p]);
        S.acc_c[p] = reinterpret_cast<double2*>(base + lay.off_acc_c[p]);
    }
    S.tone_u = reinterpret_cast<int64_t*>(base + lay.off_tone_u);
    S.tone_i = reinterpret_cast<int64_t*>(base + lay.off_tone_i);
    S.mag = reinterpret_cast<double*>(base + lay.off_mag);
    S.order = reinterpret_cast<int32_t*>(base + lay.off_order);
    S.cand_f = reinterpret_cast<int64_t*>(base + lay.off_cand_f);
    S.cand_v = reinterpret_cast<double2*>(base + lay.off_cand_v);
    S.cand_first = reinterpret_cast<int32_t*>(base + lay.off_cand_first);
    S.cand_sum = reinterpret_cast<double2*>(base + lay.off_cand_sum);
    S.contrib = reinterpret_cast<double2*>(base + lay.off_contrib);

    if (tid == 0) {
        s_acc_n = 0;
        s_cur = 0;
    }
    __syncthreads();

    const int64_t n = plan.n;
    const int64_t nmask = n - 1;
    const double inv_n = plan.inv_n;
    double2* ysig = y + s * plan.values_per_signal;

    int64_t sel_off = 0;  // trace offset: sum of earlier budgets
    for (int m = 0; m < plan.iters; ++m) {
        const DevIter& it = plan.it[m];
        const int64_t b = it.b, L = it.l_width;
        const double Ld = static_cast<double>(L);
        const double invL = 1.0 / Ld;  // exact: L is a power of two
        const int nr = it.nrounds;
        const int64_t* taus = plan.taus + it.tau_off;
        double2* Y = ysig + it.yoff;
        const int64_t sg = sigma[s * plan.iters + m];
        const int64_t sgi = sigma_inv[s * plan.iters + m];
        const int acc_n = s_acc_n;
        const int cur = s_cur;
        const int64_t* AF = cur ? S.acc_f[1] : S.acc_f[0];
        const double2* AC = cur ? S.acc_c[1] : S.acc_c[0];

        // ---- K3: subtract the prediction of everything already known.
        // predict_buckets (bucketize.cpp:84-93) adds, per known tone in
        // ascending f, (G_{jL-u} * c) * e^{-2 pi i tau u/n} into buckets
        // j = i-1, i, i+1.  Step 1 evaluates each (tone, round) rotation and
        // its three contributions once; step 2 sums, per (round, bucket), the
        // contributions in ascending tone order -- the reference's order.
        if (acc_n > 0) {
            for (int j = tid; j < acc_n; j += kDecThreads) {
                const int64_t u = (sg * AF[j]) & nmask;
                S.tone_u[j] = u;
                S.tone_i[j] = static_cast<int64_t>(floor(static_cast<double>(u) * invL + 0.5));
            }
            __syncthreads();
            for (int e = tid; e < acc_n * nr; e += kDecThreads) {
                const int j = e / nr, r = e - j * nr;
                const int64_t u = S.tone_u[j], i = S.tone_i[j];
                const double2 rot = unit_root(n, inv_n, taus[r] * u);
                const double2 c = AC[j];
                double2* dst = S.contrib + static_cast<int64_t>(e) * 3;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double g = ghat_at(it, (i - 1 + d) * L - u);
                    dst[d] = cmul(make_double2(g * c.x, g * c.y), rot);
                }
            }
            __syncthreads();
            const int64_t total = static_cast<int64_t>(nr) * b;
            for (int64_t e = tid; e < total; e += kDecThreads) {
                const int r = static_cast<int>(e / b);
                const int64_t beta = e - r * b;
                double2 pred = make_double2(0.0, 0.0);
                bool any = false;
                for (int j = 0; j < acc_n; ++j) {
                    // which of the buckets i-1, i, i+1 (mod b) is beta?
                    const int64_t dlt = (beta - S.tone_i[j] + 1) & (b - 1);
                    if (dlt <= 2) {
                        const double2 v = S.contrib[(static_cast<int64_t>(j) * nr + r) * 3 + dlt];
                        pred.x += v.x;
                        pred.y += v.y;
                        any = true;
                    }
                }
                if (any) {
                    const double2 o = Y[e];
                    Y[e] = make_double2(o.x - pred.x, o.y - pred.y);
                }
            }
            __syncthreads();
        }

        // ---- K4: stable descending order of |y0|, budget and threshold
        for (int64_t j = tid; j < b; j += kDecThreads) {
            const double2 v = Y[j];
            const double mg = cabs_ref(v.x, v.y);
            S.mag[j] = mg == mg ? mg : -1.0;  // NaN (unvalidated input) ranks last
        }
        __syncthreads();
        for (int64_t j = tid; j < b; j += kDecThreads) {
            const double mj = S.mag[j];
            int64_t rank = 0;
            for (int64_t i = 0; i < b; ++i) {
                const double mi = S.mag[i];
                rank += (mi > mj) || (mi == mj && i < j);
            }
            S.order[rank] = static_cast<int32_t>(j);
        }
        __syncthreads();
        const int64_t budget = it.budget;
        if (tid == 0) s_thr = 0.2 * S.mag[S.order[budget - 1]];
        __syncthreads();
        const double thr = s_thr;

        // ---- K5 + K6: locate and estimate.  A group of `gsz` lanes (the l
        // candidate blocks rounded up to a power of two, at most 32) takes one
        // ranked bucket, so l = 16 runs two buckets per warp.  The region
        // length evolves identically for every bucket, so all groups run the
        // same number of stages and the shuffles stay convergent.
        const int64_t lcfg = plan.l;
        const double q = plan.q;
        // group size: enough lanes for the l blocks, shrunk (each lane then
        // scans several blocks) until every ranked bucket fits in one pass
        int gsz = lcfg > 16 ? 32 : (lcfg > 8 ? 16 : (lcfg > 4 ? 8 : 4));
        while (gsz > 1 && kDecThreads / gsz < budget) gsz >>= 1;
        const int glane = lane & (gsz - 1);
        const int groups = kDecThreads / gsz;
        const int gid = tid / gsz;
        const int64_t rounds_up = (budget + groups - 1) / groups * groups;
        for (int64_t rank = gid; rank < rounds_up; rank += groups) {
            const bool live = rank < budget;
            const int64_t beta = live ? S.order[rank] : 0;
            int64_t f_out = -1;
            double2 v_out = make_double2(0.0, 0.0);
            const double2 y0 = Y[beta];
            bool ok = live && S.mag[beta] > thr;
            if (ok && y0.x == 0.0 && y0.y == 0.0) ok = false;
            double u_min = (2.0 * static_cast<double>(beta) - 1.0) * Ld / 2.0;
            double len = Ld;
            int stage = 0;
            while (len > 1.0 + 1e-9) {
                ++stage;
                if (stage >= nr) {  // cannot happen for sfft4's own tau plans
                    if (ok && glane == 0) atomicCAS(err, 0, kDecErrRounds);
                    ok = false;
                    break;  // uniform: every group sees the same stage count
                }
                double phi = 0.0;
                if (ok) {
                    const double2 yt = Y[static_cast<int64_t>(stage) * b + beta];
                    if (yt.x == 0.0 && yt.y == 0.0) {
                        ok = false;  // locate_frequency returns nullopt
                    } else {
                        const double2 z = cdiv_ref(y0.x, y0.y, yt.x, yt.y);
                        if (z.x == 0.0 && z.y == 0.0) {  // phase_of throws
                            if (glane == 0) atomicCAS(err, 0, kDecErrPhaseZero);
                            ok = false;
                        }
                        phi = atan2(z.y, z.x);
                        if (phi < 0.0) phi += kTwoPi;
                        phi = phi + 0.0;
                    }
                }
                const int64_t tau = taus[stage];
                const double rblk = len / static_cast<double>(lcfg);
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
                len = len * (q + 1.0) / static_cast<double>(lcfg);
            }
            if (ok) {
                const double lo = u_min, hi = u_min + len;
                int64_t u = static_cast<int64_t>(ceil(lo));
                if (!(static_cast<double>(u) < hi)) u = llround(0.5 * (lo + hi));
                u %= n;
                if (u < 0) u += n;
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
                if (tr_bucket) {
                    tr_bucket[sel_off + rank] = beta;
                    tr_f[sel_off + rank] = f_out;
                    tr_v[sel_off + rank] = v_out;
                }
            }
        }
        __syncthreads();

        // ---- K6 (merge): found[f] = 0 + v_r1 + v_r2 + ... in rank order
        // (std::map operator[] then +=), then acc[f] += found[f].  The first
        // accepted rank of each f carries the sum; the found set is merged
        // into the ascending acc list (ping-pong buffers).
        const int nxt = cur ^ 1;
        int64_t* NF = nxt ? S.acc_f[1] : S.acc_f[0];
        double2* NC = nxt ? S.acc_c[1] : S.acc_c[0];
        if (tid == 0) s_new_n = 0;
        // cand_first[r]: 0 = not the first accepted rank of its f,
        // 1 = first and f is new, 2 = first and f already accumulated.
        for (int64_t r = tid; r < budget; r += kDecThreads) {
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
        __syncthreads();
        // acc entries move up by the number of NEW found f below them
        for (int j = tid; j < acc_n; j += kDecThreads) {
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
        for (int64_t r = tid; r < budget; r += kDecThreads) {
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
            atomicAdd(&s_new_n, 1);
        }
        __syncthreads();
        if (tid == 0) {
            s_acc_n = acc_n + s_new_n;
            s_cur = nxt;
        }
        sel_off += budget;
        __syncthreads();
    }

    // ---- K7: keep the K largest |c| (stable over ascending f), emit in f order
    const int acc_n = s_acc_n;
    const int cur = s_cur;
    const int64_t* AF = cur ? S.acc_f[1] : S.acc_f[0];
    const double2* AC = cur ? S.acc_c[1] : S.acc_c[0];
    const int64_t K = plan.k;
    for (int j = tid; j < acc_n; j += kDecThreads) {
        const double2 c = AC[j];
        const double mg = cabs_ref(c.x, c.y);
        S.mag[j] = mg == mg ? mg : -1.0;
    }
    __syncthreads();
    for (int j = tid; j < acc_n; j += kDecThreads) {
        const double mj = S.mag[j];
        int64_t rank = 0;
        for (int i = 0; i < acc_n; ++i) {
            const double mi = S.mag[i];
            rank += (mi > mj) || (mi == mj && i < j);
        }
        S.tone_i[j] = rank < K ? 1 : 0;
    }
    __syncthreads();
    for (int j = tid; j < acc_n; j += kDecThreads) {
        if (!S.tone_i[j]) continue;
        int64_t pos = 0;
        for (int i = 0; i < j; ++i) pos += S.tone_i[i];
        out_f[s * K + pos] = AF[j];
        out_c[s * K + pos] = AC[j];
    }
    if (tid == 0) out_count[s] = acc_n < K ? acc_n : K;
}

}  // namespace

DecLayout make_dec_layout(int64_t acc_cap, int64_t b_max, int64_t budget_max,
                          int64_t rounds_max) {
    DecLayout L{};
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        const int64_t o = off;
        off += (bytes + 15) & ~int64_t{15};
        return o;
    };
    const int64_t cap = std::max<int64_t>(acc_cap, 1);
    for (int p = 0; p < 2; ++p) {
        L.off_acc_f[p] = take(cap * 8);
        L.off_acc_c[p] = take(cap * 16);
    }
    L.off_tone_u = take(cap * 8);
    L.off_tone_i = take(std::max(cap, b_max) * 8);
    L.off_mag = take(std::max(cap, b_max) * 8);
    L.off_order = take(b_max * 4);
    L.off_cand_f = take(budget_max * 8);
    L.off_cand_v = take(budget_max * 16);
    L.off_cand_first = take(budget_max * 4);
    L.off_cand_sum = take(budget_max * 16);
    L.off_contrib = take(cap * rounds_max * 3 * 16);
    L.bytes = off;
    L.in_smem = off <= 96 * 1024 ? 1 : 0;
    return L;
}

void launch_decode(const DevPlan& plan, const DecLayout& lay, double2* d_y,
                   const int64_t* d_sigma, const int64_t* d_sigma_inv, int64_t batch,
                   unsigned char* d_work, int64_t* d_out_f, double2* d_out_c,
                   int64_t* d_out_count, int32_t* d_err, cudaStream_t stream,
                   int64_t* tr_bucket, int64_t* tr_f, double2* tr_v) {
    if (batch <= 0) return;
    const size_t smem = lay.in_smem ? static_cast<size_t>(lay.bytes) : 0;
    MSFFT_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    decode_kernel<<<static_cast<unsigned>(batch), kDecThreads, smem, stream>>>(
        plan, lay, d_y, d_sigma, d_sigma_inv, batch, d_work, d_out_f, d_out_c, d_out_count,
        d_err, tr_bucket, tr_f, tr_v);
    MSFFT_LAUNCH_CHECK("decode_kernel");
}

}  // namespace msfft_b200
