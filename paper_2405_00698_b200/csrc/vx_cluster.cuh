// vx_cluster.cuh — thread-block-cluster primitives shared by the cluster
// integrator (integrator_cluster.cu) and the clustered streaming integrator
// (integrator_stream.cu): DSMEM addressing, remote stores, the cluster barrier.
#pragma once

#include <cstdint>

namespace vx {
namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// generic address of the same shared-memory object in CTA `rank` of the
// cluster: stores through it are plain (predicable, schedulable) generic
// stores with the 64-bit base computed once, instead of a shared::cluster
// store that ptxas rebuilds from the shared window every time
template <typename T>
__device__ __forceinline__ T* map_generic(T* p, uint32_t rank) {
    uint64_t r;
    asm("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
    return reinterpret_cast<T*>(r);
}
__device__ __forceinline__ void st_remote(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v));
}
// predicated DSMEM store (no branch around the asm, so the chunk stays straight-line code)
__device__ __forceinline__ void st_remote_if(bool p, uint32_t addr, double v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared::cluster.f64 [%0], %1;\n\t}" ::"r"(addr),
        "d"(v), "r"(static_cast<int>(p)));
}
__device__ __forceinline__ void st_remote_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the two halves of cluster_barrier(), for split-phase synchronisation
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

}  // namespace
}  // namespace vx
