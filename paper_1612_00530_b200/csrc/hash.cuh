// Counter-based hashing shared by the device vector fill and the config-4
// perturbation (DESIGN.md "unpinned choices" 2 and 4): splitmix64 finaliser.
#pragma once
#include <cstdint>

namespace spmvb {

__host__ __device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t h2(uint64_t seed, uint64_t a) { return sm64(sm64(seed) ^ a); }
__host__ __device__ __forceinline__ uint64_t h3(uint64_t seed, uint64_t a, uint64_t b) {
    return sm64(h2(seed, a) ^ (b * 0xD6E8FEB86659FD93ULL));
}
// 53-bit mantissa -> [0,1): exact in fp64
__host__ __device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

}  // namespace spmvb
