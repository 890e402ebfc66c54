// jit.h -- NVRTC specialisation of the step kernels (internal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "qmpm_device.cuh"

namespace qmpm {

struct JitModule {
  CUmodule module;
  CUfunction bin_count, p2g, g2p, append;
  int regs_p2g, regs_g2p;
  unsigned smem_warp_p2g, smem_warp_g2p;  // shared memory per warp
  std::string log;
};

// the generated preamble + #include of step_kernels.cuh for one layout; xk = log2(dx / Delta_x)
// when the next-step key can come from the integer x codes (0: from the decoded floats)
std::string spec_source(int dim, int material, const LayoutDev& L, int p2g_warps, int g2p_warps, int p2g_minb,
                        int g2p_minb, int xk, bool slab);
// xk of spec_source for a layout and a cell size (api.cu)
int integer_key_shift(int dim, const LayoutDev& L, float inv_dx);
cudaError_t jit_get(const std::string& src, JitModule& out, std::string& err);

// the standalone codec specialised on one layout (codec_kernels.cuh)
struct CodecJit {
  CUfunction encode, decode, matmul3;
};
// wv / vv: vector widths (4, 2, 1) usable for the records / the vals rows
std::string codec_spec_source(const CodecDev& C, bool dither, bool counters, int wv, int vv);
cudaError_t jit_codec(const std::string& src, CodecJit& out, std::string& err);

// the quantized smoke step (smoke_kernels.cuh) on a velocity and a pressure layout
struct SmokeJit {
  CUfunction advect_u, advect_refl, div, jacobi, jacobi2, project, advect_rho;
};
std::string smoke_spec_source(const CodecDev& U, const CodecDev& P, int wvu, int wvp);
cudaError_t jit_smoke(const std::string& src, SmokeJit& out, std::string& err);
cudaError_t jit_set_smem(CUfunction f, size_t bytes);
int jit_occupancy(CUfunction f, int threads, size_t smem);
cudaError_t jit_launch(CUfunction f, unsigned grid, unsigned block, size_t smem, cudaStream_t st, void** args);
cudaError_t jit_launch3(CUfunction f, dim3 grid, dim3 block, size_t smem, cudaStream_t st, void** args);

}  // namespace qmpm
