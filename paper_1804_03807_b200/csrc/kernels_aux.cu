// Explicit instantiation of the auxiliary tracker kernel (double-double
// tracking and the per-step trace hook, csrc/track_aux.cuh) for one
// n = NID_N; its own translation unit so it compiles beside kernels_inst.cu.
#include "launch.h"
#include "track_aux.cuh"

#ifndef NID_N
#error "NID_N must be defined"
#endif

namespace nid {

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
  int blocks = sms * (per < 1 ? 1 : per);
  long long need = (a.P + rows::SLOTS - 1) / rows::SLOTS;
  if (need < blocks) blocks = (int)need;
  if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  TrackArgs b = a;
  b.static_claim = need <= blocks ? 1 : 0;
  track_aux_kernel<NID_N><<<blocks, threads, smem, s>>>(b);
  return blocks;
}

}  // namespace nid
