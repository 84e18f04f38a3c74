// Launcher of cellmap_kernel<M, SCH>; instantiated per order in kern_m*.cu so
// the eight orders compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

#include "cellmap.cuh"

namespace hw {

// Counters of the dynamic tile schedule (cellmap_kernel): kSchedSlots pairs
// per device, zeroed once; each launch takes the next pair round robin and
// its last CTA zeroes it again.  Launches in flight at the same time (other
// streams, the next step under programmatic dependent launch) use different
// pairs unless kSchedSlots launches are in flight together.
constexpr int kSchedSlots = 256;
inline cudaError_t sched_slot(int dev, int** out) {
  constexpr int kDevs = 64;
  static std::atomic<int*> base[kDevs];
  static std::atomic<unsigned> seq[kDevs];
  if (dev >= kDevs) {
    *out = nullptr;  // static schedule
    return cudaSuccess;
  }
  int* p = base[dev].load(std::memory_order_acquire);
  if (p == nullptr) {
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    p = base[dev].load(std::memory_order_acquire);
    if (p == nullptr) {
      cudaError_t e;
      if ((e = cudaMalloc(&p, 2 * kSchedSlots * sizeof(int))) != cudaSuccess) return e;
      if ((e = cudaMemset(p, 0, 2 * kSchedSlots * sizeof(int))) != cudaSuccess) return e;
      if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
      base[dev].store(p, std::memory_order_release);
    }
  }
  *out = p + 2 * (seq[dev].fetch_add(1, std::memory_order_relaxed) % kSchedSlots);
  return cudaSuccess;
}

// Persistent grid: one wave of CTAs (SM count x resident CTAs per SM).
template <int M, int SCH>
cudaError_t launch_cellmap(const CellMapArgs& a, cudaStream_t st) {
  using C = CMCfg<M, SCH>;
  static_assert(C::SMEM <= 227 * 1024, "stage ring exceeds the 227 KB shared-memory limit");
  static_assert(C::NK <= 64, "per-lane parity bit masks hold at most 64 k-steps");
  static_assert(C::TJ % 8 == 0 && C::NW % (C::TJ / 8) == 0,
                "a warp's stacked M-tiles need whole rows of TJ / 8 M-tiles per warp group");
  static_assert(C::NW % 4 == 0 && (C::NPW == 4 || C::NPW == 8) &&
                    (C::NW / 4) * C::CREGS + (C::NPW / 4) * C::PREGS <=
                        65536 / C::NTHREADS / 8 * 8 * ((C::NW + C::NPW) / 4),
                "setmaxnreg split must fit the launch register allocation of each SM sub-partition");
  auto kern = cellmap_kernel<M, SCH>;
  // the attribute, SM count and occupancy are per device and never change:
  // set / query them once per device (saves ~10 us of host time per launch)
  constexpr int kDevs = 64;
  static std::atomic<int> grid_cache[kDevs];  // SM count x resident CTAs per SM + 1 (0 = unset)
  cudaError_t e;
  int dev = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  int cached = dev < kDevs ? grid_cache[dev].load(std::memory_order_acquire) : 0;
  if (cached == 0) {
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM)) != cudaSuccess)
      return e;
    int nsm = 0, per_sm = 0;
    if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NTHREADS, C::SMEM)) != cudaSuccess)
      return e;
    cached = nsm * (per_sm > 0 ? per_sm : 1) + 1;
    if (dev < kDevs) grid_cache[dev].store(cached, std::memory_order_release);
  }
  const int64_t ntiles = ((a.nty + C::TJ - 1) / C::TJ) * ((a.ntrows + C::TR - 1) / C::TR);
  if (ntiles >= (int64_t(1) << 24)) return cudaErrorInvalidValue;  // the kernel decodes tile ids in float
  int64_t nblk = cached - 1;
  if (nblk > ntiles) nblk = ntiles;
  if (nblk <= 0) return cudaSuccess;
  CellMapArgs args = a;
  args.sched = nullptr;  // static round-robin tile schedule
  if (cm_dyn(SCH, M) && (e = sched_slot(dev, &args.sched)) != cudaSuccess) return e;
#if HW_CM_PDL
  // Programmatic stream serialisation: this grid may be scheduled before the
  // previous kernel in the stream has finished; the kernel's
  // griddepcontrol.wait holds every access to step data until it has.
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)nblk);
  lc.blockDim = dim3(C::NTHREADS);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kern, args);
#else
  kern<<<(unsigned)nblk, C::NTHREADS, C::SMEM, st>>>(args);
  return cudaGetLastError();
#endif
}

#define HW_INSTANTIATE_CELLMAP(M)                                                   \
  template cudaError_t launch_cellmap<M, kDiss>(const CellMapArgs&, cudaStream_t); \
  template cudaError_t launch_cellmap<M, kCons>(const CellMapArgs&, cudaStream_t); \
  template cudaError_t launch_cellmap<M, kBoot>(const CellMapArgs&, cudaStream_t);

}  // namespace hw
