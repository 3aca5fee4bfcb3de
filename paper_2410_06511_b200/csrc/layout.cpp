// Shard(0) layout of one FSDP unit ("parameters are now represented as
// DTensors sharded on the tensor dimension 0") and the tile tables of the segmented
// kernels.  Readings: R1 ceiling division with trailing empty shards and
// zero padding; R2 16-element segment alignment (16-byte for the mixed float8 slot);
// R3 caller order.
#include "layout.h"

#include <algorithm>

namespace fsdpl {

namespace {
uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}
}  // namespace

fsdp_status_t compute_layout(int n, const fsdp_param_desc_t* descs, int W, int rank, Layout* out,
                             const char** msg) {
  if (n < 0 || (n > 0 && descs == nullptr)) { *msg = "descs is NULL"; return FSDP_ERR_INVALID_ARGUMENT; }
  if (W < 1 || rank < 0 || rank >= W) { *msg = "invalid world_size/rank"; return FSDP_ERR_INVALID_ARGUMENT; }
  Layout L;
  L.W = W;
  L.rank = rank;
  uint64_t h = 1469598103934665603ull;
  h = fnv1a(h, &W, sizeof(W));
  h = fnv1a(h, &n, sizeof(n));
  int64_t off = 0, boff = 0, u16 = 0, u8 = 0;
  for (int p = 0; p < n; ++p) {
    const fsdp_param_desc_t& d = descs[p];
    if (d.ndim < 1 || d.ndim > FSDP_MAX_NDIM) { *msg = "param ndim must be in [1, 8] (0-dim params cannot be Shard(0))"; return FSDP_ERR_SHAPE; }
    int64_t rest = 1;
    for (int i = 1; i < d.ndim; ++i) {
      if (d.shape[i] < 0) { *msg = "negative extent"; return FSDP_ERR_SHAPE; }
      rest *= d.shape[i];
    }
    const int64_t d0 = d.shape[0];
    if (d0 < 0) { *msg = "negative extent"; return FSDP_ERR_SHAPE; }
    const int64_t c = ceil_div(d0, W);
    const int64_t b = std::min<int64_t>((int64_t)rank * c, d0);
    const int64_t e = std::min<int64_t>((int64_t)(rank + 1) * c, d0);
    const int64_t np = c * rest;
    const bool f8 = d.fp8_eligible != 0;
    fsdp_param_meta_t m;
    m.dim0 = d0; m.rest = rest; m.chunk_rows = c; m.row_begin = b; m.row_count = e - b;
    m.padded_numel = np; m.elem_offset = off; m.fp8_byte_offset = boff;
    L.metas.push_back(m);
    L.numel.push_back(d0 * rest);
    L.fp8.push_back(f8 ? 1 : 0);
    off += round_up(np, kAlignElems);
    boff += round_up(np * (f8 ? 1 : 2), kAlignBytes);
    L.uoff_bf16.push_back(u16);
    L.uoff_fp8.push_back(u8);
    u16 += round_up(d0 * rest * 2, kArenaAlign);
    u8 += round_up(d0 * rest * (f8 ? 1 : 2), kArenaAlign);
    const int32_t f8i = f8 ? 1 : 0;
    h = fnv1a(h, &d.ndim, sizeof(d.ndim));
    h = fnv1a(h, d.shape, sizeof(int64_t) * d.ndim);
    h = fnv1a(h, &f8i, sizeof(f8i));
  }
  L.S = off;
  L.S_bytes_fp8 = boff;
  L.arena_bf16 = u16;
  L.arena_fp8 = u8;
  L.hash = h;
  *out = std::move(L);
  return FSDP_OK;
}

std::vector<fsdpk::Tile> tiles_copy_in_fp8(const Layout& L) {
  std::vector<fsdpk::Tile> t;
  for (size_t p = 0; p < L.metas.size(); ++p) {
    const auto& m = L.metas[p];
    const int64_t es = L.fp8[p] ? 1 : 2;
    // cover the whole 16-byte aligned slot segment: the shard is zero beyond n_p up to
    // round_up(n_p, 16) >= round_up(n_p * es, 16) / es, so the gap bytes become 0 too
    const int64_t cover = round_up(m.padded_numel * es, kAlignBytes) / es;
    for (int64_t j = 0; j < cover; j += fsdpk::kTileElems) {
      fsdpk::Tile x{};
      x.src = (uint64_t)(m.elem_offset + j);
      x.dst = (uint64_t)(m.fp8_byte_offset + j * es);
      x.n = (uint32_t)std::min<int64_t>(fsdpk::kTileElems, cover - j);
      x.param = (uint32_t)p;
      x.kind = L.fp8[p] ? fsdpk::TK_FP8 : fsdpk::TK_BF16;
      t.push_back(x);
    }
  }
  return t;
}

std::vector<fsdpk::Tile> tiles_copy_out(const Layout& L, bool fp8, std::vector<int>* first_tile) {
  std::vector<fsdpk::Tile> t;
  first_tile->assign(L.metas.size() + 1, 0);
  const int64_t slot_bytes = fp8 ? L.S_bytes_fp8 : 2 * L.S;
  for (size_t p = 0; p < L.metas.size(); ++p) {
    (*first_tile)[p] = (int)t.size();
    const auto& m = L.metas[p];
    const int64_t es = (fp8 && L.fp8[p]) ? 1 : 2;
    const int64_t boff = fp8 ? m.fp8_byte_offset : 2 * m.elem_offset;
    for (int r = 0; r < L.W; ++r) {
      // rank r's padded chunk holds elements [r*n_p, (r+1)*n_p) of the padded full tensor;
      // only those below numel are real (padding stripped, tail of the tensor).
      const int64_t first = (int64_t)r * m.padded_numel;
      const int64_t cnt = std::max<int64_t>(0, std::min<int64_t>(m.padded_numel, L.numel[p] - first));
      const int64_t bytes = cnt * es;
      for (int64_t j = 0; j < bytes; j += fsdpk::kTileBytes) {
        fsdpk::Tile x{};
        x.src = (uint64_t)(r * slot_bytes + boff + j);
        x.dst = (uint64_t)(first * es + j);
        x.n = (uint32_t)std::min<int64_t>(fsdpk::kTileBytes, bytes - j);
        x.param = (uint32_t)p;
        x.kind = fsdpk::TK_COPY;
        t.push_back(x);
      }
    }
  }
  (*first_tile)[L.metas.size()] = (int)t.size();
  return t;
}

std::vector<fsdpk::Tile> tiles_rs_copy_in(const Layout& L, std::vector<int>* first_tile) {
  std::vector<fsdpk::Tile> t;
  first_tile->assign(L.metas.size() + 1, 0);
  for (size_t p = 0; p < L.metas.size(); ++p) {
    (*first_tile)[p] = (int)t.size();
    const auto& m = L.metas[p];
    const int64_t seg = round_up(m.padded_numel, kAlignElems);
    for (int r = 0; r < L.W; ++r) {
      const int64_t c = m.chunk_rows;
      const int64_t b = std::min<int64_t>((int64_t)r * c, m.dim0);
      const int64_t e = std::min<int64_t>((int64_t)(r + 1) * c, m.dim0);
      const int64_t cnt = (e - b) * m.rest;        // real elements of rank r's chunk
      const int64_t dst0 = (int64_t)r * L.S + m.elem_offset;
      // one tile writes [j, j+n) of the aligned segment: elements below cnt come from the
      // grad, the rest (padding rows + alignment gap) are zero
      for (int64_t j = 0; j < seg; j += fsdpk::kTileElems) {
        fsdpk::Tile x{};
        x.src = (uint64_t)(b * m.rest + j);
        x.dst = (uint64_t)(dst0 + j);
        x.n = (uint32_t)std::min<int64_t>(fsdpk::kTileElems, seg - j);
        x.param = (uint32_t)p;
        x.kind = fsdpk::TK_COPY;
        x.pad = (uint32_t)std::max<int64_t>(0, std::min<int64_t>(x.n, cnt - j));  // valid source elements
        t.push_back(x);
      }
    }
  }
  (*first_tile)[L.metas.size()] = (int)t.size();
  return t;
}

void append_tiles_amax(const Layout& L, const float* shard_dev, int reg_base, std::vector<fsdpk::Tile>* out) {
  for (size_t p = 0; p < L.metas.size(); ++p) {
    if (!L.fp8[p]) continue;
    const auto& m = L.metas[p];
    for (int64_t j = 0; j < m.padded_numel; j += fsdpk::kTileElems) {
      fsdpk::Tile x{};
      x.src = (uint64_t)(uintptr_t)(shard_dev + m.elem_offset + j);
      x.dst = 0;
      x.n = (uint32_t)std::min<int64_t>(fsdpk::kTileElems, m.padded_numel - j);
      x.param = (uint32_t)(reg_base + (int)p);
      x.kind = fsdpk::TK_COPY;
      out->push_back(x);
    }
  }
}

}  // namespace fsdpl

namespace fsdpl {

std::vector<int64_t> staging_offsets(const Layout& L, int64_t* total) {
  std::vector<int64_t> off(L.metas.size());
  int64_t o = 0;
  for (size_t p = 0; p < L.metas.size(); ++p) {
    off[p] = o;
    o += round_up(L.numel[p], 128);
  }
  *total = o;
  return off;
}

// Tile size for a table covering `total` units (elements or bytes): the maximum for large
// units; for small ones about 4 tiles per SM, so a small unit spreads over the whole GPU
// instead of a few dozen SMs (the per-op latency of latency-bound units); never below
// `min_tile`, a multiple of `quantum` (keeps tile boundaries 16-byte aligned).
static int64_t tile_size_for(int64_t total, int64_t max_tile, int64_t min_tile, int64_t quantum) {
  constexpr int64_t kSmsHint = 148;
  const int64_t want = round_up(ceil_div(std::max<int64_t>(total, 1), 4 * kSmsHint), quantum);
  return std::max(min_tile, std::min(max_tile, want));
}

static int64_t own_elems(const Layout& L) {
  int64_t t = 0;
  for (const auto& m : L.metas) t += m.row_count * m.rest;
  return t;
}

std::vector<fsdpk::Tile> tiles_push(const Layout& L, bool fp8) {
  std::vector<fsdpk::Tile> t;
  const int64_t te = tile_size_for(own_elems(L), fsdpk::kTileElems, 1024, 256);
  for (size_t p = 0; p < L.metas.size(); ++p) {
    const auto& m = L.metas[p];
    const bool f8 = fp8 && L.fp8[p];
    const int64_t es = f8 ? 1 : 2;
    const int64_t base = (fp8 ? L.uoff_fp8[p] : L.uoff_bf16[p]) + m.row_begin * m.rest * es;
    const int64_t cnt = m.row_count * m.rest;
    for (int64_t j = 0; j < cnt; j += te) {
      fsdpk::Tile x{};
      x.src = (uint64_t)(m.elem_offset + j);
      x.dst = (uint64_t)(base + j * es);
      x.n = (uint32_t)std::min<int64_t>(te, cnt - j);
      x.param = (uint32_t)p;
      x.kind = f8 ? fsdpk::TK_FP8 : fsdpk::TK_BF16;
      t.push_back(x);
    }
  }
  return t;
}

std::vector<fsdpk::Tile> tiles_pull(const Layout& L, const std::vector<int64_t>& stg_off) {
  std::vector<fsdpk::Tile> t;
  const int64_t te = tile_size_for(own_elems(L), fsdpk::kTileElems, 1024, 256);
  for (size_t p = 0; p < L.metas.size(); ++p) {
    const auto& m = L.metas[p];
    const int64_t cnt = m.row_count * m.rest;
    for (int64_t j = 0; j < cnt; j += te) {
      fsdpk::Tile x{};
      x.src = (uint64_t)(stg_off[p] + m.row_begin * m.rest + j);
      x.dst = (uint64_t)(m.elem_offset + j);
      x.n = (uint32_t)std::min<int64_t>(te, cnt - j);
      x.param = (uint32_t)p;
      x.kind = fsdpk::TK_COPY;
      t.push_back(x);
    }
  }
  return t;
}

std::vector<fsdpk::Tile> tiles_scatter(const Layout& L, int64_t gsize, bool include_self) {
  // per-destination lists, then merged round robin: a persistent grid walks the table in
  // order, so every destination (and this rank's own slot, a local copy) is in flight at
  // once instead of one destination after another
  std::vector<std::vector<fsdpk::Tile>> per(L.W);
  int64_t total = 0;
  for (size_t p = 0; p < L.metas.size(); ++p) total += L.numel[p] * gsize;
  const int64_t tb = tile_size_for(total, fsdpk::kTileBytes, 2048, 512);
  for (int i = 0; i < L.W; ++i) {
    const int r = (L.rank + 1 + i) % L.W;   // destination rank, rotated per sender
    if (r == L.rank && !include_self) continue;
    for (size_t p = 0; p < L.metas.size(); ++p) {
      const auto& m = L.metas[p];
      const int64_t b = std::min<int64_t>((int64_t)r * m.chunk_rows, m.dim0);
      const int64_t e = std::min<int64_t>((int64_t)(r + 1) * m.chunk_rows, m.dim0);
      const int64_t bytes = (e - b) * m.rest * gsize;
      for (int64_t j = 0; j < bytes; j += tb) {
        fsdpk::Tile x{};
        x.src = (uint64_t)(b * m.rest * gsize + j);
        x.dst = (uint64_t)(((int64_t)L.rank * L.S + m.elem_offset) * gsize + j);
        x.n = (uint32_t)std::min<int64_t>(tb, bytes - j);
        x.param = (uint32_t)p;
        x.kind = fsdpk::TK_COPY;
        x.pad = (uint32_t)r;
        per[i].push_back(x);
      }
    }
  }
  std::vector<fsdpk::Tile> t;
  size_t longest = 0;
  for (const auto& v : per) longest = std::max(longest, v.size());
  for (size_t k = 0; k < longest; ++k)
    for (const auto& v : per)
      if (k < v.size()) t.push_back(v[k]);
  return t;
}

std::vector<fsdpk::Tile> tiles_recv_reduce(const Layout& L) {
  std::vector<fsdpk::Tile> t;
  const int64_t te = tile_size_for(own_elems(L), fsdpk::kTileElems, 1024, 256);
  for (size_t p = 0; p < L.metas.size(); ++p) {
    const auto& m = L.metas[p];
    const int64_t cnt = m.row_count * m.rest;
    for (int64_t j = 0; j < cnt; j += te) {
      fsdpk::Tile x{};
      x.src = (uint64_t)(m.elem_offset + j);
      x.dst = (uint64_t)(m.elem_offset + j);
      x.n = (uint32_t)std::min<int64_t>(te, cnt - j);
      x.param = (uint32_t)p;
      x.kind = fsdpk::TK_COPY;
      t.push_back(x);
    }
  }
  return t;
}

std::vector<fsdpk::Tile> tiles_recv_reduce_own(const Layout& L) {
  std::vector<fsdpk::Tile> t = tiles_recv_reduce(L);
  for (auto& x : t) {
    const auto& m = L.metas[x.param];
    x.src = (uint64_t)(m.row_begin * m.rest) + (x.dst - (uint64_t)m.elem_offset);
  }
  return t;
}

bool own_rows_aligned(const Layout& L, int64_t gsize) {
  for (const auto& m : L.metas)
    if (m.row_count > 0 && (m.row_begin * m.rest * gsize) % 16 != 0) return false;
  return true;
}

std::vector<fsdpk::Tile> tiles_stage(const Layout& L, const std::vector<int64_t>& stg_off, int64_t gsize) {
  std::vector<fsdpk::Tile> t;
  int64_t total = 0;
  for (size_t p = 0; p < L.metas.size(); ++p) total += L.numel[p] * gsize;
  const int64_t tb = tile_size_for(total, fsdpk::kTileBytes, 2048, 512);
  for (size_t p = 0; p < L.metas.size(); ++p) {
    const int64_t bytes = L.numel[p] * gsize;
    for (int64_t j = 0; j < bytes; j += tb) {
      fsdpk::Tile x{};
      x.src = (uint64_t)j;
      x.dst = (uint64_t)(stg_off[p] * gsize + j);
      x.n = (uint32_t)std::min<int64_t>(tb, bytes - j);
      x.param = (uint32_t)p;
      x.kind = fsdpk::TK_COPY;
      t.push_back(x);
    }
  }
  return t;
}

std::vector<fsdpk::Tile> split_pieces(const std::vector<fsdpk::Tile>& pull, int64_t S, int R, int64_t* piece) {
  const int64_t P = round_up(ceil_div(std::max<int64_t>(S, 1), R), kAlignElems);
  if (piece) *piece = P;
  std::vector<fsdpk::Tile> out;
  for (const fsdpk::Tile& t : pull) {
    int64_t d = (int64_t)t.dst, e = d + t.n;
    while (d < e) {
      const int64_t q = d / P;
      const int64_t cut = std::min<int64_t>(e, (q + 1) * P);
      fsdpk::Tile x = t;
      x.src = t.src + (uint64_t)(d - (int64_t)t.dst);
      x.dst = (uint64_t)d;
      x.n = (uint32_t)(cut - d);
      x.pad = (uint32_t)q;
      out.push_back(x);
      d = cut;
    }
  }
  return out;
}

}  // namespace fsdpl
