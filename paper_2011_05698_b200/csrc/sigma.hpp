// sigma.hpp -- device sigma plan (see sigma.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "plan_dev.cuh"

namespace msfft_b200 {

constexpr int kMaxSigmaIters = kMaxIters;

// sigma[s*iters + m], sigma_inv[s*iters + m] for s < batch from seeds[s].
// programmatic: launched with programmatic stream serialization, so it may
// start while the previous kernel on the stream is finishing (the caller
// guarantees that kernel does not use d_sigma / d_sigma_inv).
void launch_sigma(const uint64_t* d_seeds, int64_t batch, int iters, int64_t n, int64_t* d_sigma,
                  int64_t* d_sigma_inv, cudaStream_t stream, bool programmatic = false);

}  // namespace msfft_b200
