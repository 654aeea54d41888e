// Device-side checks of the CHECKED build (librbf_checked.so, build.py
// --checked; compiled with -DRBF_CHECKED).  The product build compiles both
// macros to nothing.
//  RBF_DCHECK(cond): bounds / invariant assertion; on failure prints the site
//    and traps (the launch fails with an error the caller sees, never a hang).
//  RBF_JITTER(): a lane-dependent, time-varying __nanosleep (0..~250 ns) at the
//    points where warp-synchronous code hands shared memory between lanes (ring
//    stores before a flush, flush reads after a store batch, block barriers):
//    it scrambles the relative progress of the lanes and warps, so a missing
//    __syncwarp / __syncthreads / mbarrier wait shows up as a changed result.
//    tools/race_probe.py runs every kernel family under it and compares the
//    results bit for bit with the product build (compute-sanitizer is closed on
//    the GPU pool this was developed on, profiles/r02/race_probe.md).
#pragma once
#ifdef RBF_CHECKED
#include <cstdio>
#define RBF_DCHECK(cond)                                                                           \
  do {                                                                                             \
    if (!(cond)) {                                                                                 \
      printf("RBF_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                   \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
#define RBF_JITTER()                                                                               \
  do {                                                                                             \
    const unsigned _h = ((unsigned)clock() ^ (threadIdx.x * 0x9E3779B9u)) * 0x85EBCA6Bu;          \
    __nanosleep((_h >> 24) & 0xFFu);                                                               \
  } while (0)
#else
#define RBF_DCHECK(cond) ((void)0)
#define RBF_JITTER() ((void)0)
#endif
