// libdiomp_b200: single translation unit (device globals live in common.cuh).
// Build: see paper_2506_02486_b200/build.py (nvcc -gencode arch=compute_100a,code=sm_100a).
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "core.cuh"
#include "rma.cuh"
#include "heap.cuh"
#include "stencil.cuh"
#include "collectives.cuh"
#include "gemm.cuh"
#ifdef DIOMP_EXPERIMENTS
// NVSwitch multicast allreduce: measured slower than the exact P2P kernel on
// this box, experiments build only
#include "nvls.cuh"
#endif
