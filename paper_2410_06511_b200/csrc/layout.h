// Host-side Shard(0) layout and tile-table construction (component N1).
// Pure host code, deterministic, no CUDA calls.
#pragma once
#include <cstdint>
#include <vector>

#include "fsdp_b200.h"
#include "kernels.h"

namespace fsdpl {

inline int64_t round_up(int64_t n, int64_t a) { return ((n + a - 1) / a) * a; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int64_t kAlignElems = 16;   // flat-segment alignment in elements (R2)
constexpr int64_t kAlignBytes = 16;   // mixed fp8/bf16 slot alignment in bytes (R2)
constexpr int64_t kArenaAlign = 256;  // unsharded tensors are 256-byte aligned

struct Layout {
  int W = 1, rank = 0;
  std::vector<fsdp_param_meta_t> metas;
  std::vector<int64_t> numel;     // d0 * rest
  std::vector<uint8_t> fp8;       // eligibility
  int64_t S = 0;                  // elements per rank
  int64_t S_bytes_fp8 = 0;        // bytes per rank of the mixed fp8 slot
  uint64_t hash = 0;
  // unsharded arena offsets (bytes) for the bf16 and the fp8 unshard
  std::vector<int64_t> uoff_bf16, uoff_fp8;
  int64_t arena_bf16 = 0, arena_fp8 = 0;
};

// Returns FSDP_OK or an error status with *msg set.
fsdp_status_t compute_layout(int n, const fsdp_param_desc_t* descs, int W, int rank, Layout* out,
                             const char** msg);

// K3: per param, fp8 (e4m3) or bf16 segments of n_p elements.
std::vector<fsdpk::Tile> tiles_copy_in_fp8(const Layout& L);
// K4: per (param, rank) byte copies from the [W][slot] buffer to output tensor param.
// fp8 == false: the bf16 unshard.  Tiles are param-major; first_tile[p] marks ranges.
std::vector<fsdpk::Tile> tiles_copy_out(const Layout& L, bool fp8, std::vector<int>* first_tile);
// K5: per (param, rank) grad chunk copies + zero fill of padding / alignment gaps.
std::vector<fsdpk::Tile> tiles_rs_copy_in(const Layout& L, std::vector<int>* first_tile);
// K1: amax tiles of the eligible params of a layer; src = absolute address.
void append_tiles_amax(const Layout& L, const float* shard_dev, int reg_base,
                       std::vector<fsdpk::Tile>* out);

// ---- P2P path (p2p.h)
// Full-grad staging layout: param p at element offset stg_off[p] (128-element aligned).
std::vector<int64_t> staging_offsets(const Layout& L, int64_t* total_elems);
// Push: this rank's real rows of param p: src = shard element offset, dst = byte offset of
// those rows inside the unsharded arena (bf16 or fp8 arena), kind TK_BF16 / TK_FP8.
std::vector<fsdpk::Tile> tiles_push(const Layout& L, bool fp8);
// Pull: this rank's rows of param p: src = element offset into every rank's staging,
// dst = element offset into the fp32 grad.
std::vector<fsdpk::Tile> tiles_pull(const Layout& L, const std::vector<int64_t>& stg_off);
// Staging gather: src = byte offset in grads[param], dst = byte offset in the staging.
std::vector<fsdpk::Tile> tiles_stage(const Layout& L, const std::vector<int64_t>& stg_off, int64_t gsize);
// Store-based reduce-scatter, sender side: for every destination rank r (rotated from
// rank + 1), this rank's full-grad rows of r's Shard(0) chunk of each param go into r's
// receive buffer [W][S] at slot `rank`: src = byte offset into grads[param], dst = byte
// offset (rank * S + off_p) * gsize + j, pad = r.  include_self = false leaves out the
// tiles of this rank's own chunk (the receiver then reads them from its own grads).
std::vector<fsdpk::Tile> tiles_scatter(const Layout& L, int64_t gsize, bool include_self = true);
// Store-based reduce-scatter, receiver side: this rank's rows, src = dst = element offset
// off_p + j (the same in every slot of the receive buffer and in the fp32 grad).
std::vector<fsdpk::Tile> tiles_recv_reduce(const Layout& L);
// Receiver side reading this rank's own rows from its full grads (no own-slot copy):
// dst = off_p + j (receive slots and fp32 grad), src = row_begin * rest + j (element
// offset into grads[param]).
std::vector<fsdpk::Tile> tiles_recv_reduce_own(const Layout& L);
// True when every own-row source offset row_begin * rest * gsize is a multiple of 16 bytes
// (with 16-byte aligned grad bases the own-row reduce needs no realignment).
bool own_rows_aligned(const Layout& L, int64_t gsize);

// HSDP two-phase reduce-scatter (one NVSwitch domain): the shard's flat range [0, S) is cut
// into R pieces of P = round_up(ceil(S / R), 16) elements (piece q = [q P, min((q+1) P, S)),
// *piece = P); replica q computes piece q of its shard rank's world sum.  Returns the pull
// tiles cut at piece boundaries with tile.pad = piece index.  Cuts fall on multiples of 16
// elements of dst, and every pull tile's dst is 16-element aligned, so src moves by a
// multiple of 16 elements too: each part keeps its tile's alignment phase.
std::vector<fsdpk::Tile> split_pieces(const std::vector<fsdpk::Tile>& pull, int64_t S, int R, int64_t* piece);

}  // namespace fsdpl
