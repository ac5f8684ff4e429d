// kernels.cuh -- all device code of libtsqr (sm_100a).
#pragma once
#include "common.cuh"
#include "small_kernels.cuh"
#include "stream_kernels.cuh"
#include "fused_allreduce.cuh"
#include "cluster_small.cuh"
