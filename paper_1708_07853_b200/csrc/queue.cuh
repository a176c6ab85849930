// queue.cuh -- the self-resetting global tile queue shared by the level
// kernels (dwt2.cu keeps its own copy inside the TMA producer loop).
//
// Warps take tile indices from an atomic counter (dynamic load balancing:
// under full HBM load some SMs run up to 1.5x slower than others, so static
// tile assignments wait for the slowest).  counter[0] hands out tiles;
// a warp that draws past the end increments counter[1], and the last warp
// of the grid to do so zeroes both for the next launch (which cannot start
// its own fetches before this grid completes: stream order and
// griddepcontrol.wait).
#pragma once

__device__ __forceinline__ long long dwt2_queue_fetch(unsigned int *counter, long long ntiles, int nwarps, int lane)
{
    long long t = 0;
    if (lane == 0) {
        t = (long long)atomicAdd(counter, 1u);
        if (t >= ntiles && atomicAdd(counter + 1, 1u) == unsigned(nwarps - 1)) {
            atomicExch(counter, 0u);
            atomicExch(counter + 1, 0u);
        }
    }
    return __shfl_sync(0xffffffffu, t, 0);
}
