// fused.hpp -- persistent encode+decode launch (see fused.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "encode.hpp"
#include "plan_dev.cuh"

namespace msfft_b200 {

// Device-side work description for one batch size.
struct FusedWork {
    const EncTask* tasks = nullptr;  // encode tasks, absolute signal indices
    const int32_t* items = nullptr;  // >= 0: encode task index; < 0: -(signal+1)
    int32_t n_items = 0;
    int64_t chunk = 0;               // signals per chunk
    const int32_t* need = nullptr;   // [chunk][iteration] encode tasks
    // [0] ticket, [1 + c*iters + m] tasks done, [n_counters - 1] CTAs exited;
    // zero between launches (the last CTA of each launch resets them)
    int32_t* counters = nullptr;
    int64_t n_chunks = 0;
    int64_t n_counters = 0;
};

// The validating variant (one persistent launch = ComplexSignal::validate's
// scan + encode + decode, fused.cu): items >= kValItemBase are 128-KB style
// slices of the validation stream, 0 <= items < kValItemBase packed encode
// items (packs[i] = {first sub-task, count}), < 0 decodes.
constexpr int32_t kValItemBase = 1 << 30;
struct ValWork {
    FusedWork fw;                    // tasks = sub-tasks; need/counters as above,
                                     // plus vdone[chunk] before the exit count
    const int2* packs = nullptr;
    const int32_t* vneed = nullptr;  // [chunk] validation items
    int64_t row_bytes = 0, stride_bytes = 0, item_bytes = 0, items_per_row = 0;
    int32_t policy = 0;              // L2 eviction hint of the stream (fused.cu)
};

void launch_fused_validating(const DevPlan& plan, const DecLayout& lay, const ValWork& vw,
                             const void* x, bool x_c128, int64_t x_stride, int64_t batch,
                             const int64_t* d_sigma, const int64_t* d_sigma_inv, double2* d_y,
                             unsigned char* d_work, int64_t* d_out_f, double2* d_out_c,
                             int64_t* d_out_count, int32_t* d_err, size_t smem_bytes,
                             cudaStream_t stream);

// CTA slots of the fused kernel on the current device (its persistent grid).
int64_t fused_slots(bool x_c128, size_t smem_bytes);

void launch_fused(const DevPlan& plan, const DecLayout& lay, const FusedWork& fw, const void* x,
                  bool x_c128, int64_t x_stride, int64_t batch, const int64_t* d_sigma,
                  const int64_t* d_sigma_inv, double2* d_y, unsigned char* d_work,
                  int64_t* d_out_f, double2* d_out_c, int64_t* d_out_count, int32_t* d_err,
                  size_t smem_bytes, cudaStream_t stream, bool programmatic = false);

}  // namespace msfft_b200
