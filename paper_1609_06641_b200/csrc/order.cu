// order.cu — output orderings other than dyadic.
//
// NATURAL  (Sylvester order, fwht_natural, transforms.hpp:147-172):
//   y_nat[i] = y_dy[rev_m(i)]           (natural_to_dyadic, orderings.hpp:70-78)
// SEQUENCY (rows sorted by sign changes, orderings.hpp:82-90 + :92-102):
//   y_seq[s] = y_dy[s ^ (s >> 1)]
// Both are applied as one gather pass over the dyadic result, coalesced on both
// sides:
//   * bit reversal, m >= 10: view i = (a, b, c) with a = top 5 bits, c = low 5
//     bits; rev(i) = (rev c, rev b, rev a), so a 32 x 32 tile (all a, c for one
//     b) reads 32 contiguous runs of 32 and writes 32 contiguous runs of 32
//     through a padded shared-memory tile;
//   * bit reversal, m < 10 and the Gray-code permutation: whole rows, or
//     1024-element blocks (gray(s) keeps s's block up to a block permutation),
//     gathered through shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "launch.cuh"

namespace chwb {
namespace {

__device__ __forceinline__ uint32_t brev_m(uint32_t x, int m) { return m == 0 ? 0u : (__brev(x) >> (32 - m)); }

// m >= 10: tile (a, c) for fixed middle bits b; E = element storage type.
template <class E>
__global__ void rev_tiled_kernel(const E* __restrict__ src, E* __restrict__ dst, int m, uint64_t rows) {
  __shared__ E tile[32][33];
  const int mb = m - 10;  // middle bits
  const uint64_t n = 1ull << m;
  const uint64_t tiles_per_row = 1ull << mb;
  const uint64_t t = blockIdx.x;
  const uint64_t row = t >> mb;
  if (row >= rows) return;
  const uint32_t b = (uint32_t)(t & (tiles_per_row - 1));
  const uint32_t rb = brev_m(b, mb);
  const E* s = src + row * n;
  E* d = dst + row * n;
  const uint32_t tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // read: in[rev c][rev b][rev a] for all a (contiguous: low 5 bits = rev a)
  for (uint32_t rc = ty; rc < 32; rc += 8) {
    const uint64_t off = ((uint64_t)rc << (m - 5)) | ((uint64_t)rb << 5) | tx;  // tx = rev a
    tile[rc][tx] = s[off];
  }
  __syncthreads();
  // write: out[a][b][c] for all c (contiguous), value = in[rev c][rev b][rev a]
  for (uint32_t a = ty; a < 32; a += 8) {
    const uint32_t ra = brev_m(a, 5);
    const uint32_t c = tx;
    const uint32_t rc = brev_m(c, 5);
    const uint64_t off = ((uint64_t)a << (m - 5)) | ((uint64_t)b << 5) | c;
    d[off] = tile[rc][ra];
  }
}

// Whole rows (n <= 1024) or 1024-element blocks through shared memory.
// GRAY: out[s] = in[gray(s)]; else out[i] = in[rev_m(i)] (m <= 10 only).
template <class E, bool GRAY>
__global__ void block_gather_kernel(const E* __restrict__ src, E* __restrict__ dst, int m, uint64_t rows) {
  __shared__ E buf[1024];
  const uint32_t bl = m < 10 ? (uint32_t)m : 10u;  // log2 block length
  const uint32_t blen = 1u << bl;
  const uint64_t n = 1ull << m;
  const uint64_t blocks_per_row = n >> bl;
  const uint32_t per_cta = 1024u >> bl;  // blocks (rows when m < 10) per CTA
  for (uint32_t k = 0; k < per_cta; ++k) {
    const uint64_t g = (uint64_t)blockIdx.x * per_cta + k;
    const uint64_t row = g / blocks_per_row;
    if (row >= rows) break;
    const uint64_t B = g - row * blocks_per_row;  // output block
    uint64_t Bs = B;                              // source block
    uint32_t flip = 0;
    if (GRAY) {
      Bs = B ^ (B >> 1);
      flip = (bl < (uint32_t)m) ? (uint32_t)(B & 1) << (bl - 1) : 0u;
    }
    const E* s = src + row * n + (Bs << bl);
    E* d = dst + row * n + (B << bl);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < blen; i += blockDim.x) buf[i] = s[i];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < blen; i += blockDim.x) {
      const uint32_t j = GRAY ? ((i ^ (i >> 1)) ^ flip) : brev_m(i, (int)bl);
      d[i] = buf[j];
    }
  }
}

template <class E>
chw_status permute_typed(const void* src, void* dst, chw_order order, int64_t batch, int m, cudaStream_t st) {
  const E* s = static_cast<const E*>(src);
  E* d = static_cast<E*>(dst);
  const uint64_t rows = (uint64_t)batch;
  if (order == CHW_ORDER_NATURAL && m >= 10) {
    const uint64_t tiles = rows << (m - 10);
    // Grid splits advance by a whole number of rows (tiles are row-major).
    const uint64_t step = (0x7fffffffull >> (m - 10)) << (m - 10);
    for (uint64_t t0 = 0; t0 < tiles; t0 += step) {
      const unsigned g = (unsigned)std::min<uint64_t>(tiles - t0, step);
      // Offset by whole rows only: tiles are row-major, so t0 is row-aligned here.
      const uint64_t row0 = t0 >> (m - 10);
      rev_tiled_kernel<E><<<g, dim3(32, 8), 0, st>>>(s + (row0 << m), d + (row0 << m), m, rows - row0);
      if (chw_status r = check_launch("rev_tiled_kernel")) return r;
    }
    return CHW_OK;
  }
  const uint32_t bl = m < 10 ? (uint32_t)m : 10u;
  const uint64_t blocks = rows << (m - (int)bl);
  const uint32_t per_cta = 1024u >> bl;
  const uint64_t ctas = (blocks + per_cta - 1) / per_cta;
  if (ctas > 0x7fffffffull) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: batch too large to reorder");
  const unsigned threads = std::min<uint32_t>(256u, std::max<uint32_t>(32u, 1u << bl));
  if (order == CHW_ORDER_SEQUENCY)
    block_gather_kernel<E, true><<<(unsigned)ctas, threads, 0, st>>>(s, d, m, rows);
  else
    block_gather_kernel<E, false><<<(unsigned)ctas, threads, 0, st>>>(s, d, m, rows);
  return check_launch("block_gather_kernel");
}

}  // namespace

// dst[r][i] = src[r][p(i)] for the requested order (src != dst).
chw_status permute_order(const void* src, void* dst, size_t elem_bytes, chw_order order, int64_t batch, int m,
                         cudaStream_t st) {
  if (batch == 0) return CHW_OK;
  switch (elem_bytes) {
    case 2:
      return permute_typed<uint16_t>(src, dst, order, batch, m, st);
    case 4:
      return permute_typed<uint32_t>(src, dst, order, batch, m, st);
    case 8:
      return permute_typed<unsigned long long>(src, dst, order, batch, m, st);
  }
  return fail(CHW_ERR_UNSUPPORTED, "chw_forward: element size");
}

}  // namespace chwb
