// k1_kernels.cu -- the K1 builds (see k_sweep.cu for the design and the
// launch logic).  Compiled once per build with -DNALAR_K1_PART=k, so the
// nine ~500 KB kernels compile in parallel; without a part: all of them.
#include "k1_body.cuh"

namespace nalar {

template <bool kOut, bool kProf, bool kIn, bool kNext>
__device__ __forceinline__ void k1_entry(const SweepParams& p, uint8_t* smem) {
    // an invalid table (K0's verdict, complete before the zero kernel ran)
    // is never swept: nalar_step queues this kernel before the host has seen it
    // this CTA's block record and the verdict: independent loads, one round trip
    const uint4* rec = reinterpret_cast<const uint4*>(p.blk_order) + 2 * (size_t)blockIdx.x;
    const uint4 ca = rec[0], cb = rec[1];
    if (!p.stream_in && *p.verdict) return;
    if (cb.w) k1_body<true, kOut, kProf, kIn, kNext>(p, smem, ca, cb);
    else k1_body<false, kOut, kProf, kIn, kNext>(p, smem, ca, cb);
}

// K1 builds.  Code compiled into the sweep costs the plain epoch even when a
// runtime flag skips it (measured: streamed-output stores in P3 +1.2 us at C4,
// the NALAR_F_PROFILE stamps +1.1 us at C4 and +7.5 us at C5), so each mode
// has its own build: <outputs to host, profile stamps, streamed staging,
// NEXT-1/4 marks> x {one CTA per SM (a one-wave table, C4), two (several
// waves, C5: 64 registers)}.

#define NALAR_K1_KERNEL(NAME, MINB, OUT, PROF, IN, NEXT)                        \
    __global__ void __launch_bounds__(kK1Threads, MINB) NAME(SweepParams p) {    \
        extern __shared__ __align__(128) uint8_t smem[];                         \
        k1_entry<OUT, PROF, IN, NEXT>(p, smem);                                  \
    }
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 0
NALAR_K1_KERNEL(k1_sweep, 1, false, false, false, false)          // the plain epoch
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 1
NALAR_K1_KERNEL(k1_sweep_x2, 2, false, false, false, false)
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 2
NALAR_K1_KERNEL(k1_sweep_step, 1, true, false, true, false)       // nalar_step (streamed in / out)
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 3
NALAR_K1_KERNEL(k1_sweep_step_x2, 2, false, false, true, false)
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 4
NALAR_K1_KERNEL(k1_sweep_next, 1, false, false, false, true)      // HoL migration / batching on
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 5
NALAR_K1_KERNEL(k1_sweep_next_x2, 2, false, false, false, true)
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 6
NALAR_K1_KERNEL(k1_sweep_prof, 1, false, true, false, false)      // NALAR_F_PROFILE: the plain build + stamps
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 7
NALAR_K1_KERNEL(k1_sweep_x2_prof, 2, false, true, false, false)   //   (what bench.py's spans time)
#endif
#if !defined(NALAR_K1_PART) || NALAR_K1_PART == 8
NALAR_K1_KERNEL(k1_sweep_prof_all, 1, true, true, true, true)     // NALAR_F_PROFILE, any other mode
#endif
#undef NALAR_K1_KERNEL

}  // namespace nalar
