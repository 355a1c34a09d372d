// gm_comm.cuh -- the register exchange of an element-sharded sketch over
// NCCL (NVLink / NVSwitch), configs 4-5 at N > 1 GPUs.
//
// "Sketch per site, merge centrally": every rank sketches
// a contiguous shard of the element set; the k registers (16 B each) are then
// combined register by register.  Two exchanges, both in place on (y, s):
//   * all-reduce-min: ncclAllReduce(y, MIN) -> y_min; ids of the ranks that
//     hold y_min (UINT64_MAX elsewhere, mask_min_ids_kernel);
//     ncclAllReduce(ids, MIN) -- the register-wise lexicographic (y, id)
//     minimum, i.e. sketch_naive's smaller-id tie rule (sketch.py:196-205);
//   * all-gather + merge: ncclAllGather of every rank's registers and the
//     device merge in rank order -- merge([sketch_rank0, ...]) exactly,
//     earlier rank wins exact ties (estimate.py:103-125).
// Both equal the whole set's sketch (partition law, test_estimate.py:174-199)
// unless two ranks hold different elements with identical y bits.
//
// NCCL is opened at run time (dlopen "libnccl.so.2": the copy the process
// already has -- torch's -- or the system one), so the library loads, and
// every other entry point works, on hosts without NCCL.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

namespace gmk {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  bool ok = false;
  char why[256] = "";
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(api.why, sizeof(api.why), "libnccl.so.2 not loadable: %s", dlerror());
      return;
    }
#define GM_NCCL_SYM(field, name)                                                  \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));              \
  if (!api.field) {                                                               \
    snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks %s", name);            \
    return;                                                                       \
  }
    GM_NCCL_SYM(get_unique_id, "ncclGetUniqueId")
    GM_NCCL_SYM(comm_init_rank, "ncclCommInitRank")
    GM_NCCL_SYM(comm_destroy, "ncclCommDestroy")
    GM_NCCL_SYM(all_reduce, "ncclAllReduce")
    GM_NCCL_SYM(all_gather, "ncclAllGather")
    GM_NCCL_SYM(group_start, "ncclGroupStart")
    GM_NCCL_SYM(group_end, "ncclGroupEnd")
    GM_NCCL_SYM(error_string, "ncclGetErrorString")
    GM_NCCL_SYM(get_version, "ncclGetVersion")
#undef GM_NCCL_SYM
    api.ok = true;
  });
  return api;
}

// one communicator per rank (its device fixed at init) + exchange scratch
struct GmComm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
  double* ybuf = nullptr;  // all-reduce: y_min [k]; all-gather: [nranks, k]
  u64* sbuf = nullptr;     // masked ids [k] / gathered ids [nranks, k]
  size_t cap = 0;          // registers of scratch per buffer
};

// ids of the registers this rank holds at the minimum; UINT64_MAX elsewhere
__global__ void mask_min_ids_kernel(const double* __restrict__ y_local, const double* __restrict__ y_min,
                                    const u64* __restrict__ s, u64* __restrict__ s_masked, u32 k) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    s_masked[j] = __double_as_longlong(y_local[j]) == __double_as_longlong(y_min[j]) ? s[j] : ~0ull;
}

}  // namespace gmk
