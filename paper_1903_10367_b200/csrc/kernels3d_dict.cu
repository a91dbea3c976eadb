// Row dictionaries of the BoxMG transfer weights (P of level ltop-1 and its
// cube-owned copy Pc).
//
// P is the one per-cycle stream that is not per-fine-vertex state: 124 fp64
// weights per coarse vertex (36.7 B per fine DoF, 14.5 GB at config 5), read
// twice per cycle (restriction, prolongation).  Its rows are a function of the
// fine operator around the coarse vertex only (the 8 coarse cells adjacent to
// it), so wherever the coefficient is piecewise constant on blocks of coarse
// cells -- the jump-coefficient problems BoxMG exists for; BASELINE config 5 has
// 27^3-cell blocks -- most rows are bitwise repeats of a few distinct rows.
// This file stores such an array losslessly as
//
//   dict[id * kDictW + q]  (row-major, the D distinct rows, rows padded to 128 doubles = 1 KB)
//   idx[ioff(r)] = id   (uint32 per row, rows of the vertex / cube grid padded)
//
// Rows are compared by their exact bit patterns: a 64-bit hash sorts them
// (cub radix sort, stable, so every class is led by its smallest row index),
// then every row is compared word by word against its class leader; any
// mismatch (a hash collision) abandons the dictionary and the caller keeps the
// dense array.  Ids are assigned in order of first occurrence.  Rows are
// row-major so a kernel's weight q is one load at an immediate offset from its
// row base; the few distinct rows a warp meets stay in L1, and the streamed
// per-vertex data is loaded evict-first so the dictionary stays in L2.  The
// kernels read the same doubles they would read from P, in the same order, so
// the iterate is bitwise unchanged.
#include <cub/cub.cuh>

namespace t3 {

// row r, term q of a plane-major array whose rows are enumerated with `inner`
// rows per pitch-padded line: element = base[q * plane + (r / inner) * pitch + r % inner]
// (idx is laid out with `iinner` rows per `ipitch`-padded line, so its rows are 16-byte multiples
// for the kernels' TMA boxes)
struct RowsView {
  const double* base;
  size_t inner, pitch, plane;
  int W;
  size_t iinner, ipitch;
  __device__ __forceinline__ size_t off(size_t r) const { return (r / inner) * pitch + r % inner; }
  __device__ __forceinline__ size_t ioff(size_t r) const { return (r / iinner) * ipitch + r % iinner; }
  __device__ __forceinline__ double at(size_t r, int q) const { return base[(size_t)q * plane + off(r)]; }
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

__global__ void kd_hash(RowsView v, size_t R, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (size_t)gridDim.x * blockDim.x) {
    uint64_t h = 0x9e3779b97f4a7c15ULL;
    for (int q = 0; q < v.W; ++q) h = mix64(h ^ (uint64_t)__double_as_longlong(v.at(r, q)) ^ (uint64_t)q << 56);
    keys[r] = h;
    vals[r] = (uint32_t)r;
  }
}

// runstart input: i at the head of a run of equal keys, 0 elsewhere (max-scanned afterwards)
__global__ void kd_heads(const uint64_t* __restrict__ keys, size_t R, uint32_t* __restrict__ hs) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += (size_t)gridDim.x * blockDim.x)
    hs[i] = (i == 0 || keys[i] != keys[i - 1]) ? (uint32_t)i : 0u;
}

__global__ void kd_leader(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ runstart, size_t R,
                          uint32_t* __restrict__ leader) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += (size_t)gridDim.x * blockDim.x)
    leader[vals[i]] = vals[runstart[i]];
}

// every row equals its leader bit for bit (else a hash collision: *bad = 1); first[r] = r leads
__global__ void kd_verify(RowsView v, const uint32_t* __restrict__ leader, size_t R, uint32_t* __restrict__ first,
                          int* bad) {
  for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (size_t)gridDim.x * blockDim.x) {
    const size_t h = leader[r];
    first[r] = h == r ? 1u : 0u;
    if (h == r) continue;
    bool eq = true;
    for (int q = 0; q < v.W && eq; ++q)
      eq = __double_as_longlong(v.at(r, q)) == __double_as_longlong(v.at(h, q));
    if (!eq) atomicOr(bad, 1);
  }
}

__global__ void kd_fill(RowsView v, const uint32_t* __restrict__ leader, const uint32_t* __restrict__ newid,
                        size_t R, uint32_t* __restrict__ idx, double* __restrict__ dict) {
  for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (size_t)gridDim.x * blockDim.x) {
    const uint32_t h = leader[r], id = newid[h];
    idx[v.ioff(r)] = id;
    if (h == r)
      for (int q = 0; q < v.W; ++q) dict[(size_t)id * kDictW + q] = v.at(r, q);
  }
}

struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

}  // namespace t3
