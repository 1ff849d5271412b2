// Kernel launch wrapper with a recording mode: every kernel of a planning
// cycle is launched through tmpcb::launch(), which either launches it on the
// stream or -- while ctx.cu records a cycle -- appends (function, grid,
// block, a copy of the arguments) to a list.  ctx.cu builds one CUDA graph
// per GPU from that list and, on the following cycles, only rewrites the
// kernel nodes' arguments (cudaGraphExecKernelNodeSetParams: new s0, seed,
// shard) before replaying it (the cycle as a graph per GPU).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

namespace tmpcb {

struct LaunchRec {
  const void* func = nullptr;
  dim3 grid, block;
  std::shared_ptr<void> holder;  // owns the argument copies
  std::vector<void*> args;       // pointers into *holder, kernel parameter order
};

// Non-null while ctx.cu records a cycle (thread-local: contexts on other host
// threads keep launching directly).
std::vector<LaunchRec>*& launch_recorder();

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t stream,
                          Args&&... args) {
  static_assert(sizeof...(KArgs) == sizeof...(Args), "kernel argument count");
  if (std::vector<LaunchRec>* rec = launch_recorder()) {
    using Tup = std::tuple<std::decay_t<KArgs>...>;
    auto t = std::make_shared<Tup>(std::forward<Args>(args)...);
    LaunchRec r;
    r.func = reinterpret_cast<const void*>(kern);
    r.grid = grid;
    r.block = block;
    std::apply([&](auto&... a) { (r.args.push_back(static_cast<void*>(&a)), ...); }, *t);
    r.holder = std::move(t);
    rec->push_back(std::move(r));
    return cudaSuccess;
  }
  kern<<<grid, block, 0, stream>>>(std::forward<Args>(args)...);
  return cudaGetLastError();
}

}  // namespace tmpcb
