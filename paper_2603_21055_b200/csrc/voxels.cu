// Voxel occupancy of the global geometry set (tracker.py:81-122,
// GlobalGeomSet.insert): at most one member per voxel cell
// floor(center / voxel_size); a batch row is inserted iff its cell is not yet
// occupied and no earlier row of the same batch claimed it (first come, first
// served in row order).  The reference keeps a Python set of cell tuples and
// loops over the rows; here the cells live in a device hash table (open
// addressing, linear probing) and a batch is gated in three passes:
//   1. every row claims its cell's slot (atomicCAS on the key) and, unless
//      the cell is already occupied, lowers the slot's owner to its row index
//      (atomicMin): the smallest row index of the batch wins;
//   2. a row is kept iff it owns its slot;
//   3. the kept rows' cells become occupied.
// Cell coordinates are packed 21 bits per axis (|cell| < 2^20).

#include "common.cuh"

namespace sgad {

constexpr unsigned long long VX_EMPTY = ~0ull;
constexpr uint32_t VX_OCCUPIED = 0xFFFFFFFFu;  // a member of an earlier batch
constexpr uint32_t VX_FREE = 0xFFFFFFFEu;      // owner not yet claimed in this batch
constexpr long long VX_LIM = 1ll << 20;

__device__ __forceinline__ unsigned long long vx_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// returns the slot holding key k, inserting it if absent
__device__ __forceinline__ uint32_t vx_claim(unsigned long long* keys, uint32_t mask,
                                             unsigned long long k) {
  uint32_t s = (uint32_t)vx_hash(k) & mask;
  while (true) {
    const unsigned long long cur = keys[s];
    if (cur == k) return s;
    if (cur == VX_EMPTY) {
      const unsigned long long prev = atomicCAS(keys + s, VX_EMPTY, k);
      if (prev == VX_EMPTY || prev == k) return s;
    }
    s = (s + 1) & mask;
  }
}

__global__ void k_vx_claim(const double* __restrict__ centers, int64_t n, double voxel,
                           unsigned long long* __restrict__ keys, uint32_t* __restrict__ owner,
                           uint32_t mask, uint32_t* __restrict__ slot_of,
                           uint32_t* __restrict__ bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) c[a] = (long long)floor(centers[3 * i + a] / voxel);
  if (c[0] < -VX_LIM || c[0] >= VX_LIM || c[1] < -VX_LIM || c[1] >= VX_LIM || c[2] < -VX_LIM ||
      c[2] >= VX_LIM) {
    atomicExch(bad, 1u);
    slot_of[i] = 0xFFFFFFFFu;
    return;
  }
  const unsigned long long k = ((unsigned long long)(c[0] + VX_LIM) << 42) |
                               ((unsigned long long)(c[1] + VX_LIM) << 21) |
                               (unsigned long long)(c[2] + VX_LIM);
  const uint32_t s = vx_claim(keys, mask, k);
  slot_of[i] = s;
  if (owner[s] != VX_OCCUPIED) atomicMin(owner + s, (uint32_t)i);
}

__global__ void k_vx_keep(int64_t n, const uint32_t* __restrict__ owner,
                          const uint32_t* __restrict__ slot_of, uint8_t* __restrict__ keep,
                          uint32_t* __restrict__ n_keep) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool k = false;
  if (i < n) {
    const uint32_t s = slot_of[i];
    k = s != 0xFFFFFFFFu && owner[s] == (uint32_t)i;
    keep[i] = k ? 1 : 0;
  }
  const uint32_t c = (uint32_t)__syncthreads_count(k);
  if (threadIdx.x == 0 && c) atomicAdd(n_keep, c);
}

// commit the kept rows' cells; if any row was out of range the whole batch
// is abandoned and the cells it claimed are released
__global__ void k_vx_commit(int64_t n, const uint8_t* __restrict__ keep,
                            const uint32_t* __restrict__ slot_of, uint32_t* __restrict__ owner,
                            const uint32_t* __restrict__ bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || slot_of[i] == 0xFFFFFFFFu) return;
  if (*bad) owner[slot_of[i]] = VX_FREE;
  else if (keep[i]) owner[slot_of[i]] = VX_OCCUPIED;
}

__global__ void k_vx_init(unsigned long long* __restrict__ keys, uint32_t* __restrict__ owner,
                          uint32_t cap) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cap) {
    keys[i] = VX_EMPTY;
    owner[i] = VX_FREE;
  }
}

// move the occupied cells of an old table into a fresh (larger) one
__global__ void k_vx_rehash(const unsigned long long* __restrict__ okeys,
                            const uint32_t* __restrict__ oowner, uint32_t ocap,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ owner,
                            uint32_t mask) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ocap || okeys[i] == VX_EMPTY || oowner[i] != VX_OCCUPIED) return;
  owner[vx_claim(keys, mask, okeys[i])] = VX_OCCUPIED;
}

}  // namespace sgad

struct sgad_voxels {
  sgad::DevBuf keys, owner, slot_of, counters;
  uint32_t cap = 0;
  int64_t occupied = 0;
  uint32_t* pinned = nullptr;
};

using namespace sgad;

static inline unsigned vblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

static int vx_reserve(sgad_voxels* v, int64_t need, cudaStream_t st) {
  uint64_t want = 1024;
  while (want < 2 * (uint64_t)need) want <<= 1;
  SGAD_REQUIRE(want <= (1ull << 31), "voxel table too large (%lld cells)", (long long)need);
  if (want <= v->cap) return SGAD_OK;
  DevBuf nk, no;
  SGAD_CHECK_CUDA(nk.ensure(sizeof(unsigned long long) * want));
  SGAD_CHECK_CUDA(no.ensure(sizeof(uint32_t) * want));
  k_vx_init<<<vblk(want, 256), 256, 0, st>>>(nk.as<unsigned long long>(), no.as<uint32_t>(),
                                             (uint32_t)want);
  SGAD_LAUNCH_CHECK();
  if (v->cap) {
    k_vx_rehash<<<vblk(v->cap, 256), 256, 0, st>>>(
        v->keys.as<unsigned long long>(), v->owner.as<uint32_t>(), v->cap,
        nk.as<unsigned long long>(), no.as<uint32_t>(), (uint32_t)want - 1);
    SGAD_LAUNCH_CHECK();
    SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  v->keys.release();
  v->owner.release();
  v->keys = nk;
  v->owner = no;
  nk.p = no.p = nullptr;  // ownership moved
  v->cap = (uint32_t)want;
  return SGAD_OK;
}

extern "C" {

int sgad_voxels_create(sgad_voxels** out) {
  SGAD_REQUIRE(out != nullptr, "sgad_voxels_create: null out");
  sgad_voxels* v = new sgad_voxels();
  if (cudaMallocHost(&v->pinned, 4 * sizeof(uint32_t)) != cudaSuccess) {
    delete v;
    set_error("cudaMallocHost failed");
    return SGAD_E_CUDA;
  }
  *out = v;
  return SGAD_OK;
}

int sgad_voxels_destroy(sgad_voxels* v) {
  if (!v) return SGAD_OK;
  v->keys.release();
  v->owner.release();
  v->slot_of.release();
  v->counters.release();
  if (v->pinned) cudaFreeHost(v->pinned);
  delete v;
  return SGAD_OK;
}

int sgad_voxels_gate(sgad_voxels* v, const double* centers, int64_t n, double voxel_size,
                     uint8_t* keep, int64_t* n_keep, void* stream_) {
  SGAD_REQUIRE(v && n >= 0 && n_keep && voxel_size > 0.0 && (n == 0 || (centers && keep)),
               "sgad_voxels_gate: bad arguments");
  SGAD_REQUIRE(n < (1ll << 31) - 2, "sgad_voxels_gate: batch too large");
  cudaStream_t st = (cudaStream_t)stream_;
  *n_keep = 0;
  if (n == 0) return SGAD_OK;
  if (int rc = vx_reserve(v, v->occupied + n, st)) return rc;
  SGAD_CHECK_CUDA(v->slot_of.ensure(sizeof(uint32_t) * n));
  SGAD_CHECK_CUDA(v->counters.ensure(sizeof(uint32_t) * 2));
  SGAD_CHECK_CUDA(cudaMemsetAsync(v->counters.p, 0, sizeof(uint32_t) * 2, st));
  uint32_t* cnt = v->counters.as<uint32_t>();
  k_vx_claim<<<vblk(n, 256), 256, 0, st>>>(centers, n, voxel_size, v->keys.as<unsigned long long>(),
                                           v->owner.as<uint32_t>(), v->cap - 1,
                                           v->slot_of.as<uint32_t>(), cnt + 1);
  SGAD_LAUNCH_CHECK();
  k_vx_keep<<<vblk(n, 256), 256, 0, st>>>(n, v->owner.as<uint32_t>(), v->slot_of.as<uint32_t>(),
                                          keep, cnt);
  SGAD_LAUNCH_CHECK();
  k_vx_commit<<<vblk(n, 256), 256, 0, st>>>(n, keep, v->slot_of.as<uint32_t>(),
                                            v->owner.as<uint32_t>(), cnt + 1);
  SGAD_LAUNCH_CHECK();
  SGAD_CHECK_CUDA(cudaMemcpyAsync(v->pinned, cnt, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  SGAD_CHECK_CUDA(cudaStreamSynchronize(st));
  SGAD_REQUIRE(v->pinned[1] == 0,
               "voxel cell index beyond +-2^20 (voxel_size too small for the scene)");
  *n_keep = v->pinned[0];
  v->occupied += v->pinned[0];
  return SGAD_OK;
}

}  // extern "C"
