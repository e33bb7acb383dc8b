// Explicit instantiation of every per-size kernel for one n = NID_N.
// The build compiles this file once per n in 1..16 (in parallel), so each
// size gets fully unrolled register-resident code.
#include "endpoint.cuh"
#include "launch.h"
#include "track_common.cuh"
#include "track_ctl.cuh"

#ifndef NID_N
#error "NID_N must be defined"
#endif

namespace nid {

static int blocks_for(const void* fn, int threads, int smem = 0) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
  if (per < 1) per = 1;
  return sms * per;
}

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

// row-split thread-per-path tracker: 32 path slots per block, G warps
int CAT(launch_track_, NID_N)(const TrackArgs& a, int max_blocks, cudaStream_t s) {
  const void* fn = (const void*)track_ctl_kernel<NID_N>;
  const int threads = 32 * rows::groups<NID_N>();
  const int smem = (int)ctl::smem_bytes<NID_N>();
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  TrackArgs b = a;
  const int blocks = track_grid(a.P, blocks_for(fn, threads, smem), max_blocks, &b.static_claim);
  track_ctl_kernel<NID_N><<<blocks, threads, smem, s>>>(b);
  return blocks;
}

// the same tracker with the term table in the launch's parameter bank
int CAT(launch_track_pt_, NID_N)(const TrackArgsPT& a, int max_blocks, cudaStream_t s) {
  // a per-cell polyhedral homotopy (t-weighted coefficients) runs its own
  // instantiation: the linear-homotopy kernel carries none of its code
  const void* fn = a.t.poly ? (const void*)track_pt_kernel<NID_N, true> : (const void*)track_pt_kernel<NID_N, false>;
  const int threads = 32 * rows::groups<NID_N>();
  const int smem = (int)ctl::Lay<NID_N>::bytes();
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  TrackArgsPT* b = new TrackArgsPT(a);  // ~22 KB: off the stack
  const int blocks = track_grid(a.a.P, blocks_for(fn, threads, smem), max_blocks, &b->a.static_claim);
  if (a.t.poly)
    track_pt_kernel<NID_N, true><<<blocks, threads, smem, s>>>(*b);
  else
    track_pt_kernel<NID_N, false><<<blocks, threads, smem, s>>>(*b);
  delete b;
  return blocks;
}

int CAT(launch_endpoint_, NID_N)(const EndpointArgs& a, int blocks, cudaStream_t s) {
  endpoint_kernel<NID_N><<<blocks, 128, 0, s>>>(a);
  return blocks;
}

int CAT(launch_refine_, NID_N)(const RefineArgs& a, int blocks, cudaStream_t s) {
  refine_kernel<NID_N><<<blocks, 128, 0, s>>>(a);
  return blocks;
}

int CAT(launch_ddrefine_, NID_N)(const DDRefineArgs& a, int blocks, cudaStream_t s) {
  ddrefine_kernel<NID_N><<<blocks, 128, 0, s>>>(a);
  return blocks;
}

int CAT(launch_eval_, NID_N)(const EvalArgs& a, int blocks, cudaStream_t s) {
  eval_kernel<NID_N><<<blocks, 128, 0, s>>>(a);
  return blocks;
}

int CAT(launch_newton_, NID_N)(const NewtonArgs& a, int blocks, cudaStream_t s) {
  newton_kernel<NID_N><<<blocks, 128, 0, s>>>(a);
  return blocks;
}

int CAT(track_regs_, NID_N)() {
  cudaFuncAttributes at;
  if (cudaFuncGetAttributes(&at, (const void*)track_ctl_kernel<NID_N>) != cudaSuccess) return -1;
  return at.numRegs;
}

int CAT(track_pt_regs_, NID_N)() {
  cudaFuncAttributes at;
  if (cudaFuncGetAttributes(&at, (const void*)track_pt_kernel<NID_N, false>) != cudaSuccess) return -1;
  return at.numRegs;
}

int CAT(track_threads_, NID_N)() { return rows::SLOTS; }  // path slots per block

int CAT(track_smem_, NID_N)() { return (int)ctl::smem_bytes<NID_N>(); }

}  // namespace nid
