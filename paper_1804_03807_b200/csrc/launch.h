// Per-size launchers (defined in kernels_inst.cu, one translation unit per n).
#pragma once
#include <cuda_runtime.h>

struct TrackArgs;
struct TrackArgsPT;
struct EndpointArgs;
struct RefineArgs;
struct DDRefineArgs;
struct EvalArgs;
struct NewtonArgs;

namespace nid {
#define NID_DECL(n)                                                        \
  int launch_track_##n(const TrackArgs&, int, cudaStream_t);               \
  int launch_track_pt_##n(const TrackArgsPT&, int, cudaStream_t);          \
  int launch_track_aux_##n(const TrackArgs&, int, cudaStream_t);           \
  int track_pt_regs_##n();                                                  \
  int launch_endpoint_##n(const EndpointArgs&, int, cudaStream_t);         \
  int launch_refine_##n(const RefineArgs&, int, cudaStream_t);             \
  int launch_ddrefine_##n(const DDRefineArgs&, int, cudaStream_t);         \
  int launch_eval_##n(const EvalArgs&, int, cudaStream_t);                 \
  int launch_newton_##n(const NewtonArgs&, int, cudaStream_t);             \
  int track_regs_##n();                                                     \
  int track_threads_##n();                                                  \
  int track_smem_##n();
NID_DECL(1) NID_DECL(2) NID_DECL(3) NID_DECL(4) NID_DECL(5) NID_DECL(6) NID_DECL(7) NID_DECL(8)
NID_DECL(9) NID_DECL(10) NID_DECL(11) NID_DECL(12) NID_DECL(13) NID_DECL(14) NID_DECL(15) NID_DECL(16)
#undef NID_DECL
}  // namespace nid
