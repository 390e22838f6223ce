// Canonical reduction tiling shared by host and device code.
#pragma once
#include <cuda_runtime.h>

namespace ep {

constexpr int kTileRows = 16;
constexpr int kBlockTiles = 16;  // tiles per canonical block

// Canonical tile map: rows are cut into segments of seg_rows, each segment into
// tiles of kTileRows aligned at the segment start, and the tiles into blocks of
// kBlockTiles.
__host__ __device__ inline int imin(int a, int b) { return a < b ? a : b; }

struct TileMap {
  int rows;
  int seg_rows;
  int tiles_per_seg;
  int num_segs;
  __host__ __device__ int num_tiles() const { return num_segs * tiles_per_seg; }
  // first row and row count of tile b (count <= 0: tile does not exist)
  __host__ __device__ void tile(int b, int& r0, int& nr) const {
    const int seg = b / tiles_per_seg;
    const int t = b - seg * tiles_per_seg;
    r0 = seg * seg_rows + t * kTileRows;
    const int seg_end = imin(seg * seg_rows + seg_rows, rows);
    nr = imin(kTileRows, seg_end - r0);
  }
  __host__ __device__ int tiles_in_seg(int seg) const {
    const int r0 = seg * seg_rows;
    const int r1 = imin(r0 + seg_rows, rows);
    return (r1 - r0 + kTileRows - 1) / kTileRows;
  }
};

inline TileMap make_tile_map(int rows, int seg_rows) {
  TileMap m;
  m.rows = rows;
  m.seg_rows = seg_rows;
  m.tiles_per_seg = (seg_rows + kTileRows - 1) / kTileRows;
  m.num_segs = rows > 0 ? (rows + seg_rows - 1) / seg_rows : 0;
  return m;
}

}  // namespace ep
