// Peer-memory exchange of the sharded apply over NVLink /
// NVSwitch: each rank's exchange buffers (its depth slab's spectrum and the
// full-depth spectrum of its quadrant-mode shard) are plain cudaMalloc
// allocations shared through CUDA IPC handles, so a rank's column moves
// (shard.cu, move_planes) store straight into the destination rank's buffer
// -- the transpose is one pass of peer stores, no pack / NCCL all-to-all /
// unpack. Completion is a flag per (destination, source) pair in the
// destination's memory: the source's signal kernel release-stores the
// exchange epoch there (system scope) after its move kernels in stream
// order; the destination's wait kernel acquire-loads its G flags before the
// next stage reads the buffer (bounded spin: a peer that never arrives sets a
// sticky timeout flag, which emie_cu_peer_status reports, and the waits
// return instead of hanging the GPU; the context stays usable).
#include "operator.cuh"

namespace emie_cu {

namespace {

constexpr int kMaxPeers = 64;
struct PeerFlags {
  int* p[kMaxPeers];
};

__device__ int g_peer_timeout = 0;  // sticky: a wait gave up on a peer

__global__ void peer_signal_kernel(PeerFlags f, int G, int me, int epoch) {
  // the earlier kernels' remote NVLink stores (moves, fused transposes) are
  // ordered before the flag by the kernel boundary; the system-scope fence
  // makes that ordering explicit for the peers that acquire the flag
  asm volatile("fence.sc.sys;" ::: "memory");
  const int g = threadIdx.x;
  if (g < G) {
    int* a = f.p[g] + me;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(a), "r"(epoch) : "memory");
  }
}

__global__ void peer_wait_kernel(const int* flags, int G, int epoch) {
  const int g = threadIdx.x;
  if (g < G) {
    long long spins = 0;
    int v;
    while (true) {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + g) : "memory");
      if (v - epoch >= 0) break;  // epochs only grow (wrap-safe difference)
      if (*reinterpret_cast<volatile int*>(&g_peer_timeout)) break;  // an earlier wait already gave up
      __nanosleep(200);
      if (++spins > (1LL << 27)) {  // ~30 s: a peer is gone; report it, never hang
        atomicExch(&g_peer_timeout, 1);
        break;
      }
    }
  }
  __syncthreads();
  // the next stage reads the buffer with TMA (async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

}  // namespace

// reads and clears the sticky timeout flag (synchronises the device)
int peer_status() {
  int v = 0;
  EMIE_CUDA(cudaDeviceSynchronize());
  EMIE_CUDA(cudaMemcpyFromSymbol(&v, g_peer_timeout, sizeof(int)));
  if (v) {
    const int z = 0;
    EMIE_CUDA(cudaMemcpyToSymbol(g_peer_timeout, &z, sizeof(int)));
  }
  return v;
}

void peer_signal(int* const* flag_ptrs, int G, int me, int epoch, cudaStream_t st) {
  if (!flag_ptrs || G < 1 || G > kMaxPeers || me < 0 || me >= G)
    fail(EMIE_CU_INVALID_ARGUMENT, "peer_signal: bad arguments");
  PeerFlags f{};
  for (int g = 0; g < G; ++g) {
    if (!flag_ptrs[g]) fail(EMIE_CU_INVALID_ARGUMENT, "peer_signal: null flag pointer");
    f.p[g] = flag_ptrs[g];
  }
  peer_signal_kernel<<<1, 64, 0, st>>>(f, G, me, epoch);
  check_launch("peer_signal_kernel");
}

void peer_wait(const int* flags, int G, int epoch, cudaStream_t st) {
  if (!flags || G < 1 || G > kMaxPeers) fail(EMIE_CU_INVALID_ARGUMENT, "peer_wait: bad arguments");
  peer_wait_kernel<<<1, 64, 0, st>>>(flags, G, epoch);
  check_launch("peer_wait_kernel");
}

}  // namespace emie_cu
