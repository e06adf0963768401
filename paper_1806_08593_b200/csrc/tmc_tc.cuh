// Tensor-core (tcgen05) path of the TMC message pass.  Stub until the sm_100a kernels land:
// tc_supported() returns false so every edge runs on the SIMT kernels.
#pragma once
#include <cstddef>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/tmc.h"
#include "tmc_internal.h"

namespace tmc {

struct TcLatentBuf { bool ok = false; };

inline bool tc_supported(const std::vector<int>&, const std::vector<int>&, const std::vector<int>&) { return false; }
inline void tc_plan(const std::vector<int>&, const std::vector<int>&, const std::vector<int>&, const std::vector<int>&,
                    int, int, size_t&, std::vector<TcLatentBuf>& bufs) { bufs.clear(); }
inline bool tc_edge_ok(const TcLatentBuf& b) { return b.ok; }
inline tmc_status tc_forward(const std::vector<int>&, const std::vector<int>&, const std::vector<int>&,
                             const std::vector<int>&, int, int, const tmc_latent_in*, void*,
                             const std::vector<TcLatentBuf>&, cudaStream_t) { return TMC_OK; }
inline void tc_pass_forward(const PassArgs&, const TcLatentBuf&, void*, bool, cudaStream_t) {}
inline void tc_pass_backward(const PassArgs&, const TcLatentBuf&, void*, bool, int, cudaStream_t) {}
inline bool tc_factors_ok(int, int, int) { return false; }
inline tmc_status tc_factors(const tmc_latent_in*, float*, int, int, int, int, cudaStream_t) { return TMC_OK; }

}  // namespace tmc
