// page_layout.cuh -- where element (token t, column c) of one cache page lives in HBM.
//
// The reference keeps each cache as a contiguous row-major GrowMat (proj/include/lorakv/kvcache.hpp:
// 161-206); pages are this library's layout and are chosen for the kernels that read them:
//
//   fp32 pages: row-major [P tokens][width]; when the width is a multiple of 4 elements the 16-byte chunks of a
//       row are XOR-swizzled with the token index -- chunk' = chunk ^ (t & swz), swz + 1 = the largest power of two
//       <= 8 that divides the chunks per row -- so that a contiguous bulk copy of 8 tokens lands in shared memory
//       as a tile whose TF32 MMA fragments (fla_decode_f32.cu) load without bank conflicts
//   bf16 pages whose row width is not a multiple of 8 elements: row-major [P tokens][width]
//   bf16 pages (the hot path):
//       [width / bw column blocks][P tokens][bw elements], bw = 64 when width % 64 == 0, the width
//       itself when it is 8, 16 or 32, and 8 otherwise.  Inside a block every token owns one row of
//       2*bw bytes and the 16-byte chunks of a row are XOR-swizzled with the address bits above
//       bit 7 -- chunk' = chunk ^ ((byte_offset >> 7) & (chunks_per_row - 1)).  For 128/64/32-byte
//       rows this is exactly the SWIZZLE_128B / 64B / 32B pattern of TMA and of the tcgen05
//       shared-memory descriptors, so a plain contiguous bulk copy (cp.async.bulk) of any 8-token
//       aligned run of a block lands in shared memory as a canonical swizzled operand tile:
//       bank-conflict-free for ldmatrix and directly consumable by tcgen05.mma, with no tensor map.
#pragma once

#include <cstdint>

namespace lk {

struct PageLayout {
  int P;        // tokens per page
  int width;    // elements per token row (d_head, or the padded rank)
  int bw;       // column-block width in elements; == width for row-major pages
  int swz;      // chunks_per_row - 1 when swizzled, 0 otherwise
  int eb;       // bytes per element
};

__host__ __device__ inline PageLayout make_page_layout(int P, int width, int elem_bytes) {
  PageLayout l;
  l.P = P; l.width = width; l.bw = width; l.swz = 0; l.eb = elem_bytes;
  if (elem_bytes == 4 && width > 0 && width % 4 == 0) {
    const int chunks = width / 4;
    int s = 1;
    while (s < 8 && chunks % (2 * s) == 0) s *= 2;
    l.swz = s - 1;
  }
  if (elem_bytes == 2 && width > 0 && width % 8 == 0) {
    if (width % 64 == 0) l.bw = 64;
    else if (width == 8 || width == 16 || width == 32) l.bw = width;
    else l.bw = 8;
    l.swz = l.bw / 8 - 1;
  }
  return l;
}

// element offset of (token t, column c) from the start of the page
__host__ __device__ inline int64_t page_offset(const PageLayout& l, int t, int c) {
  if (l.eb == 4) return (int64_t)t * l.width + ((((c >> 2) ^ (t & l.swz)) << 2) | (c & 3));
  if (l.bw == l.width && l.swz == 0) return (int64_t)t * l.width + c;
  const int blk = c / l.bw, cc = c % l.bw;
  uint32_t byte = (uint32_t)t * (uint32_t)(2 * l.bw) + (uint32_t)(cc >> 3) * 16u;
  byte ^= ((byte >> 7) & (uint32_t)l.swz) << 4;
  return (int64_t)blk * l.P * l.bw + (byte >> 1) + (cc & 7);
}

}  // namespace lk
