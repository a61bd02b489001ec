// K2-K4 hand-written radix sorts (sort.cu): shared constants and launchers.
#pragma once
#include "common.cuh"

namespace gsb {

constexpr int kRadix = 256;
constexpr int kSortThreads = 256;
#ifndef GSB_SORT_ITEMS
#define GSB_SORT_ITEMS 8
#endif
constexpr int kSortItems = GSB_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;

// Per-render sort state, zeroed once per render: digit histograms (depth passes 0-2, tile
// passes 3-4) and the tile tickets of each persistent pass (depth 0-2, pack 3, tile 4-5).
struct SortBlock {
    uint32_t hist[5][kRadix];
    uint32_t ticket[8];
};

// 64-bit look-back status words a sort over max_elems elements needs (never cleared: every pass
// carries a fresh epoch in [1, 2^30))
size_t sort_status_words(int64_t max_elems);

// (depth, map index) order of the visible set: 3 passes over the 24-bit keys (K1's append
// order in keys_a / vis_gid), then exact tie order; result in keys_b / gid_sorted. Uses epochs
// epoch .. epoch + 2. Count: cnt[kCntVisible] (<= max_n).
void launch_depth_sort(uint32_t* keys_a, uint32_t* keys_b, int32_t* vis_gid, int32_t* gid_tmp, int32_t* gid_sorted,
                       const unsigned long long* depth_by_gid, unsigned long long* cnt, int max_n, SortBlock* sb,
                       unsigned long long* status, uint32_t epoch, cudaStream_t st);

// rank-ordered records + exclusive scan of their tile counts (emit_off[0 .. n_vis])
void launch_pack_scan(const int32_t* gid_sorted, const Splat* rec_by_gid, const unsigned long long* depth_by_gid,
                      const unsigned long long* cnt, int max_n, Splat* rec_sorted, unsigned long long* depth_sorted,
                      int32_t* rank_of /* [map size]: depth rank of each visible map index */,
                      uint32_t* emit_off, SortBlock* sb, unsigned long long* status, uint32_t epoch, cudaStream_t st);

// emission of the (tile, rank) pairs + stable sort by tile + ranges; the sorted ranks land in
// vals_b (keys in keys_b: uint16 while tiles <= 0xffff, else uint32). Uses epochs epoch,
// epoch + 1. Returns the number of kernel launches.
// zero the tile ranges [tiles], the device counters and (if non-null) the sort block
void launch_frame_init(uint2* ranges, int tiles, unsigned long long* counters, SortBlock* sb, cudaStream_t st);
int launch_tile_sort(const uint32_t* emit_off, const Splat* rec, unsigned long long* cnt, int max_n, uint32_t cap,
                     int tiles_x, int tiles, void* keys_a, void* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                     uint2* ranges, SortBlock* sb, unsigned long long* status, uint32_t epoch, cudaStream_t st);

}  // namespace gsb
