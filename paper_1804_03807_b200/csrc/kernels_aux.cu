// Explicit instantiation of the auxiliary tracker kernel (double-double
// tracking and the per-step trace hook, csrc/track_aux.cuh) for one
// n = NID_N; its own translation unit so it compiles beside kernels_inst.cu.
#include "launch.h"
#include "track_aux.cuh"

#ifndef NID_N
#error "NID_N must be defined"
#endif

namespace nid {

// Grid of a tracker launch: as many blocks as stay resident (cap), at least one
// per 32 paths -- and a launch smaller than the machine is dealt round the SMs
// (one block per path up to the SM count) instead of being packed 32 to a block.
static int track_grid(long long P, int cap, int max_blocks, int* is_static) {
  int dev = 0, sms = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long need = (P + rows::SLOTS - 1) / rows::SLOTS;
  long long spread = P < sms ? P : sms;
  long long blocks = need > spread ? need : spread;
  if (blocks > cap) blocks = cap;
  if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  *is_static = blocks * rows::SLOTS >= P ? 1 : 0;
  return (int)blocks;
}

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)

int CAT(launch_track_aux_, NID_N)(const TrackArgs& a, int max_blocks, cudaStream_t s) {
  const void* fn = (const void*)track_aux_kernel<NID_N>;
  const int threads = 32 * rows::groups<NID_N>();
  const int smem = (int)ctl::Lay<NID_N>::bytes();
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
  TrackArgs b = a;
  const int blocks = track_grid(a.P, sms * (per < 1 ? 1 : per), max_blocks, &b.static_claim);
  track_aux_kernel<NID_N><<<blocks, threads, smem, s>>>(b);
  return blocks;
}

}  // namespace nid
