// fused.cu -- one persistent launch that runs the encode (K1+K2) and the
// decode (K3..K7) of a whole batch, so the HBM-bound gather and the
// issue-bound decode share every SM instead of running back to back.
//
// CTAs pull work items from a global ticket counter.  The item list is
// E(c0) E(c1) D(c0) E(c2) D(c1) ... D(c_last): E = the encode tasks of a
// chunk of signals, D = one decode per signal of a chunk.  A decode item waits
// until its chunk's encode-completion counter reaches the chunk's task count.
// Every encode item with a smaller ticket is already held by a running CTA
// and never waits, so the spin always terminates (no deadlock), and the
// encode->decode hand-off follows the threadfence-reduction pattern
// (producer: stores, __syncthreads, __threadfence, atomicAdd; consumer: spin
// on the counter, __threadfence, __syncthreads).  Compiled with --fmad=false.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "decode_body.cuh"
#include "encode_body.cuh"
#include "fused.hpp"

#ifndef MSFFT_FUSED_MINB
#define MSFFT_FUSED_MINB 2
#endif

#ifdef MSFFT_TIMELINE
// diagnostic build only: per item {start ns, end ns, smid << 48 | m << 40 | code}
__device__ unsigned long long g_timeline[1 << 16][3];
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
extern "C" int msfft_debug_timeline(void* dst, long long n_items) {
    if (n_items > (1 << 16)) n_items = 1 << 16;
    return static_cast<int>(cudaMemcpyFromSymbol(dst, g_timeline, n_items * 24));
}
#endif

namespace msfft_b200 {

namespace {

template <class T>
__global__ void __launch_bounds__(kEncThreads, MSFFT_FUSED_MINB)
fused_kernel(const __grid_constant__ DevPlan plan, DecLayout lay, DecArgs args,
             const EncTask* __restrict__ tasks, const int32_t* __restrict__ items,
             int32_t n_items, int64_t chunk, const int32_t* __restrict__ need,
             int32_t* __restrict__ done, int32_t* __restrict__ ticket, const T* __restrict__ x,
             int64_t x_stride, int64_t batch, unsigned char* __restrict__ work,
             int64_t n_counters) {
    int32_t* exit_count = ticket + n_counters - 1;  // the last counter slot
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ DecShared sh;
    __shared__ int s_item;
    static_assert(kEncThreads == kDecThreads, "fused CTA runs both bodies");
    // programmatic dependent launch: this grid reads the σ plan of the
    // kernel before it (wait), and the next launch may be scheduled as soon
    // as SM slots free up (launch_dependents); it uses other buffers
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    encode_barrier_init(&bar);
    uint32_t phase = 0;
    const bool bad_input = args.err[1] != 0;  // set by the validation pass
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(ticket, 1);
        __syncthreads();
        const int item = s_item;
        if (item >= n_items) break;
        const int32_t code = items[item];
#ifdef MSFFT_TIMELINE
        const unsigned long long tl_start = tl_now();
#endif
        if (code >= 0) {
            const EncTask& t = tasks[code];
            encode_task(plan, t, x, x_stride, batch, args.sigma, args.y, smem, &bar, phase);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                // done = counters + 1; the last counter is the exit count
                MSFFT_DCHECK((t.sig0 / chunk) * plan.iters + t.m + 2 < n_counters);
                atomicAdd(&done[(t.sig0 / chunk) * plan.iters + t.m], 1);
            }
        } else if (!bad_input) {
            // the decode waits per iteration (DecArgs::gate_*), so it can run
            // while the later iterations of its chunk are still being encoded
            const int64_t s0 = -static_cast<int64_t>(code) - 1;
            const int64_t c = s0 / chunk;
            MSFFT_DCHECK(s0 < batch && (c + 1) * plan.iters + 2 <= n_counters);
            DecArgs a = args;
            a.gate_done = done + c * plan.iters;
            a.gate_need = need + c * plan.iters;
            decode_signal<kDecThreads>(plan, lay, a, s0, lay.in_smem ? smem : work + s0 * lay.bytes,
                                       sh, nullptr);
        }
        __syncthreads();
#ifdef MSFFT_TIMELINE
        if (threadIdx.x == 0 && item < (1 << 16)) {
            unsigned smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            g_timeline[item][0] = tl_start;
            g_timeline[item][1] = tl_now();
            const unsigned m = code >= 0 ? static_cast<unsigned>(tasks[code].m) : 0xffu;
            g_timeline[item][2] = (static_cast<unsigned long long>(smid) << 48) |
                                  (static_cast<unsigned long long>(m) << 40) |
                                  static_cast<unsigned>(code);
        }
#endif
    }
    // the last CTA out resets this launch's counters (ticket, done, exit)
    // for the next launch that uses them, so no memset sits between launches
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(exit_count, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (s_last) {
        for (int64_t i = threadIdx.x; i < n_counters; i += blockDim.x) ticket[i] = 0;
        __threadfence();
    }
}

template <class T>
void launch_t(const DevPlan& plan, const DecLayout& lay, const FusedWork& fw, const T* x,
              int64_t x_stride, int64_t batch, const int64_t* d_sigma,
              const int64_t* d_sigma_inv, double2* d_y, unsigned char* d_work, int64_t* d_out_f,
              double2* d_out_c, int64_t* d_out_count, int32_t* d_err, size_t smem,
              cudaStream_t stream, bool programmatic) {
    auto k = fused_kernel<T>;
    smem_attr(k, smem);
    const int sms = sm_count();
    int per_sm = 0;
    {
        // occupancy per (device, kernel, shared memory), queried once
        static std::mutex mu;
        static std::map<std::tuple<int, const void*, size_t>, int> occ;
        int dev = 0;
        MSFFT_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lock(mu);
        const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(k), smem);
        auto it = occ.find(key);
        if (it == occ.end()) {
            MSFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kEncThreads, smem));
            occ[key] = per_sm;
        } else {
            per_sm = it->second;
        }
    }
    if (per_sm < 1) throw CudaError("fused_kernel: does not fit on an SM");
    const int64_t grid = std::min<int64_t>(static_cast<int64_t>(sms) * per_sm, fw.n_items);
    // counters are zero: from creation, then reset by the previous launch's
    // last CTA (a memset here would also serialise programmatic launches)
    DecArgs args{d_y, d_sigma, d_sigma_inv, d_out_f, d_out_c, d_out_count, d_err,
                 nullptr, nullptr, nullptr};
    if (programmatic) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(kEncThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MSFFT_CUDA(cudaLaunchKernelEx(&cfg, k, plan, lay, args, fw.tasks, fw.items, fw.n_items,
                                      fw.chunk, fw.need, fw.counters + 1, fw.counters, x, x_stride,
                                      batch, d_work, fw.n_counters));
    } else {
        k<<<static_cast<unsigned>(grid), kEncThreads, smem, stream>>>(
            plan, lay, args, fw.tasks, fw.items, fw.n_items, fw.chunk, fw.need, fw.counters + 1,
            fw.counters, x, x_stride, batch, d_work, fw.n_counters);
    }
    MSFFT_LAUNCH_CHECK("fused_kernel");
}

// ---------------------------------------------------------------------------
// Validating fused kernel.  The reference validates every sample on entry
// (ComplexSignal::validate, proj/src/signal.cpp:22-25, called from
// sfft4.cpp:133), so a validating call must read all of x once.  Run as a
// separate scan followed by the encode, the encode's random 8-B reads then
// fetch whole 128-B lines from HBM a second time (every random read fills a
// line: 4x the sectors it needs).  Here both read the same lines while they
// are in L2: the item list is V(c) E(c) D(c - lag) per chunk c of signals
// (a chunk's rows fit well inside the 126-MB L2), so each line of x comes
// from HBM once and the step is bound by the validation stream.
//   V: a slice of one row streamed through a TMA bulk-copy ring in the CTA's
//      dynamic shared memory (16-KB copies on mbarriers), integer
//      exponent tests, a non-finite sample sets err[1];
//   E: a packed encode item (encode_pack: iterations of one signal side by
//      side), loads that allocate in L2 normally;
//   D: the decode of one signal, gated per iteration on its chunk's encode
//      items and, before it starts, on its chunk's validation items (a
//      signal batch with a non-finite sample is not decoded: the call throws).
// Deadlock freedom as in fused_kernel: V and E items never wait, D items wait
// only on items with smaller tickets.
constexpr int kVChunk = 16384;
constexpr int kVRing = 8;

__device__ __forceinline__ uint32_t vnon_finite4(uint4 v, bool c128) {
    if (c128)
        return ((v.y & 0x7ff00000u) == 0x7ff00000u) | ((v.w & 0x7ff00000u) == 0x7ff00000u);
    return ((v.x & 0x7f800000u) == 0x7f800000u) | ((v.y & 0x7f800000u) == 0x7f800000u) |
           ((v.z & 0x7f800000u) == 0x7f800000u) | ((v.w & 0x7f800000u) == 0x7f800000u);
}

// Streams [src, src + len) (16-B multiple) through `slots` ring slots.
// Every copy issued here is consumed here, so each slot's mbarrier is idle
// between items; `vpar` carries the slots' parities from item to item.
template <bool C128>
__device__ __forceinline__ uint32_t validate_slice(const unsigned char* __restrict__ src,
                                                   int64_t len, unsigned char* ring,
                                                   uint64_t* vbar, uint32_t& vpar, int slots,
                                                   int policy_mode) {
    // L2 eviction class of the streamed lines (ValWork::policy & 3): 0 the
    // copy's default, 1 evict_normal, 2 evict_last, 3 evict_first
    uint64_t pol = 0;
    if (policy_mode == 1)
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else if (policy_mode == 2)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else if (policy_mode == 3)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int64_t nch = (len + kVChunk - 1) / kVChunk;
    auto issue = [&](int64_t i, int slot) {
        const int64_t off = i * kVChunk;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kVChunk), len - off));
        const uint32_t bb = smem_u32(&vbar[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes)
                     : "memory");
        if (policy_mode)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
                "[%0], [%1], %2, [%3], %4;"
                ::"r"(smem_u32(ring + slot * kVChunk)), "l"(src + off), "r"(bytes), "r"(bb),
                "l"(pol)
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                ::"r"(smem_u32(ring + slot * kVChunk)), "l"(src + off), "r"(bytes), "r"(bb)
                : "memory");
    };
    if (threadIdx.x == 0) {
        // earlier generic-proxy use of the ring (taps, arrays, decode scratch)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int i = 0; i < slots && i < nch; ++i) issue(i, i);
    }
    uint32_t acc = 0;
    int slot = 0;
    for (int64_t i = 0; i < nch; ++i) {
        const uint32_t par = (vpar >> slot) & 1u;
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&vbar[slot])),
            "r"(par)
            : "memory");
        vpar ^= 1u << slot;
        const uint4* v = reinterpret_cast<const uint4*>(ring + slot * kVChunk);
        const int64_t rem = len - i * kVChunk;
        if (rem >= kVChunk) {
#pragma unroll
            for (int e = 0; e < kVChunk / 16 / kEncThreads; ++e)
                acc |= vnon_finite4(v[threadIdx.x + e * kEncThreads], C128);
        } else {
            const int nv = static_cast<int>(rem / 16);
            for (int e = threadIdx.x; e < nv; e += kEncThreads) acc |= vnon_finite4(v[e], C128);
        }
        __syncthreads();  // the slot is consumed before it is refilled
        if (threadIdx.x == 0 && i + slots < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(i + slots, slot);
        }
        slot = slot + 1 == slots ? 0 : slot + 1;
    }
    return acc;
}

template <class T>
__global__ void __launch_bounds__(kEncThreads, MSFFT_FUSED_MINB)
fused_val_kernel(const __grid_constant__ DevPlan plan, DecLayout lay, DecArgs args,
                 const __grid_constant__ ValWork vw, const T* __restrict__ x, int64_t x_stride,
                 int64_t batch, unsigned char* __restrict__ work, int slots) {
    const FusedWork& fw = vw.fw;
    const int policy_mode = vw.policy & 3;
    // the gather's loads: evict_last (policy bit 2) or evict_normal
    uint64_t gpol;
    if (vw.policy & 4)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(gpol));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(gpol));
    int32_t* ticket = fw.counters;
    int32_t* done = ticket + 1;
    int32_t* vdone = done + fw.n_chunks * plan.iters;
    int32_t* exit_count = ticket + fw.n_counters - 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t vbar[kVRing];
    __shared__ DecShared sh;
    __shared__ int s_item, s_skip;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kVRing; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&vbar[i])));
    }
    encode_barrier_init(&bar);  // fences the inits and syncs
    uint32_t phase = 0, vpar = 0;
    constexpr bool kC128 = sizeof(T) == 16;
    const unsigned char* xb = reinterpret_cast<const unsigned char*>(x);
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(ticket, 1);
        __syncthreads();
        const int item = s_item;
        if (item >= fw.n_items) break;
        const int32_t code = fw.items[item];
        if (code >= kValItemBase) {
            const int64_t v = code - kValItemBase;
            const int64_t row = v / vw.items_per_row;
            const int64_t off = (v - row * vw.items_per_row) * vw.item_bytes;
            const int64_t len = min(vw.item_bytes, vw.row_bytes - off);
            const uint32_t bad = validate_slice<kC128>(xb + row * vw.stride_bytes + off, len, smem,
                                                       vbar, vpar, slots, policy_mode);
            if (__any_sync(0xffffffffu, bad != 0) && (threadIdx.x & 31) == 0)
                atomicExch(args.err + 1, 1);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(&vdone[row / fw.chunk], 1);
            }
        } else if (code >= 0) {
            const int2 pk = vw.packs[code];
            const EncTask* sub = fw.tasks + pk.x;
            encode_pack(plan, sub, pk.y, x, x_stride, args.sigma, args.y, smem, &bar, phase, gpol);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                for (int j = 0; j < pk.y; ++j)
                    atomicAdd(&done[(sub[j].sig0 / fw.chunk) * plan.iters + sub[j].m], 1);
            }
        } else {
            const int64_t s0 = -static_cast<int64_t>(code) - 1;
            const int64_t c = s0 / fw.chunk;
            if (threadIdx.x == 0) {
                while (load_acquire(&vdone[c]) < vw.vneed[c]) __nanosleep(128);
                s_skip = load_acquire(args.err + 1) != 0;
            }
            __syncthreads();
            if (!s_skip) {
                DecArgs a = args;
                a.gate_done = done + c * plan.iters;
                a.gate_need = fw.need + c * plan.iters;
                decode_signal<kDecThreads>(plan, lay, a, s0,
                                           lay.in_smem ? smem : work + s0 * lay.bytes, sh, nullptr);
            }
        }
        __syncthreads();
    }
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(exit_count, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (s_last) {
        for (int64_t i = threadIdx.x; i < fw.n_counters; i += blockDim.x) ticket[i] = 0;
        __threadfence();
    }
}

template <class T>
void launch_val_t(const DevPlan& plan, const DecLayout& lay, const ValWork& vw, const T* x,
                  int64_t x_stride, int64_t batch, const int64_t* d_sigma,
                  const int64_t* d_sigma_inv, double2* d_y, unsigned char* d_work,
                  int64_t* d_out_f, double2* d_out_c, int64_t* d_out_count, int32_t* d_err,
                  size_t smem, cudaStream_t stream) {
    auto k = fused_val_kernel<T>;
    smem_attr(k, smem);
    int per_sm = 0;
    MSFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kEncThreads, smem));
    if (per_sm < 1) throw CudaError("fused_val_kernel: does not fit on an SM");
    const int64_t grid = std::min<int64_t>(static_cast<int64_t>(sm_count()) * per_sm,
                                           vw.fw.n_items);
    const int slots = static_cast<int>(std::min<size_t>(kVRing, smem / kVChunk));
    if (slots < 1) throw std::invalid_argument("fused_val_kernel: shared memory below one slot");
    DecArgs args{d_y, d_sigma, d_sigma_inv, d_out_f, d_out_c, d_out_count, d_err,
                 nullptr, nullptr, nullptr};
    k<<<static_cast<unsigned>(grid), kEncThreads, smem, stream>>>(plan, lay, args, vw, x, x_stride,
                                                                  batch, d_work, slots);
    MSFFT_LAUNCH_CHECK("fused_val_kernel");
}

}  // namespace

void launch_fused_validating(const DevPlan& plan, const DecLayout& lay, const ValWork& vw,
                             const void* x, bool x_c128, int64_t x_stride, int64_t batch,
                             const int64_t* d_sigma, const int64_t* d_sigma_inv, double2* d_y,
                             unsigned char* d_work, int64_t* d_out_f, double2* d_out_c,
                             int64_t* d_out_count, int32_t* d_err, size_t smem_bytes,
                             cudaStream_t stream) {
    if (vw.fw.n_items <= 0) return;
    if (x_c128)
        launch_val_t(plan, lay, vw, static_cast<const double2*>(x), x_stride, batch, d_sigma,
                     d_sigma_inv, d_y, d_work, d_out_f, d_out_c, d_out_count, d_err, smem_bytes,
                     stream);
    else
        launch_val_t(plan, lay, vw, static_cast<const float2*>(x), x_stride, batch, d_sigma,
                     d_sigma_inv, d_y, d_work, d_out_f, d_out_c, d_out_count, d_err, smem_bytes,
                     stream);
}

int64_t fused_slots(bool x_c128, size_t smem_bytes) {
    int dev = 0, sms = 0, per_sm = 0;
    MSFFT_CUDA(cudaGetDevice(&dev));
    MSFFT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (x_c128) {
        MSFFT_CUDA(cudaFuncSetAttribute(fused_kernel<double2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem_bytes)));
        MSFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<double2>,
                                                                 kEncThreads, smem_bytes));
    } else {
        MSFFT_CUDA(cudaFuncSetAttribute(fused_kernel<float2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem_bytes)));
        MSFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<float2>,
                                                                 kEncThreads, smem_bytes));
    }
    return static_cast<int64_t>(sms) * per_sm;
}

void launch_fused(const DevPlan& plan, const DecLayout& lay, const FusedWork& fw, const void* x,
                  bool x_c128, int64_t x_stride, int64_t batch, const int64_t* d_sigma,
                  const int64_t* d_sigma_inv, double2* d_y, unsigned char* d_work,
                  int64_t* d_out_f, double2* d_out_c, int64_t* d_out_count, int32_t* d_err,
                  size_t smem_bytes, cudaStream_t stream, bool programmatic) {
    if (fw.n_items <= 0) return;
    if (x_c128)
        launch_t(plan, lay, fw, static_cast<const double2*>(x), x_stride, batch, d_sigma,
                 d_sigma_inv, d_y, d_work, d_out_f, d_out_c, d_out_count, d_err, smem_bytes,
                 stream, programmatic);
    else
        launch_t(plan, lay, fw, static_cast<const float2*>(x), x_stride, batch, d_sigma,
                 d_sigma_inv, d_y, d_work, d_out_f, d_out_c, d_out_count, d_err, smem_bytes,
                 stream, programmatic);
}

}  // namespace msfft_b200
