// plan.cpp — host-side plan: domain topology, tile geometry, per-rank protocol constants and the
// algorithmic per-rank byte counts. Pure C++, no CUDA; the kernels in
// kernels.cu execute exactly this partition (the boundary formulas are restated there on the device).
//
// Partition of one AR tile of `len` elements:
//   L = lcm(d_0..d_{D-1}) elementary segments on the grid of a FULL tile T (a multiple of L*D*V,
//   V = 16-byte vector width), clipped to len: b(s) = min(len, s*T/L). Member j of domain k (size
//   d) owns segments [j*L/d, (j+1)*L/d), so every segment has exactly one owner per domain (SURVEY
//   §8(a) a0). Piece p of segment s (reduced by domain p's owner in the cross stage):
//   c(s,p) = min(b(s+1), b(s) + p*T/(L*D)). Clipping (rather than rescaling to len) keeps every
//   piece of a ragged last tile within its scratch slot and every boundary V-aligned.
#include <algorithm>
#include <cstring>

#include "hetccl_internal.h"

namespace hetccl {

static int gcd_(int a, int b) { return b ? gcd_(b, a % b) : a; }

int build_topo(int n, const int* map, Topo* t) {
  if (n < 1 || n > kMaxRanks || !map) return -1;
  std::memset(t, 0, sizeof(*t));
  int D = 0;
  for (int r = 0; r < n; r++) {
    if (map[r] < 0 || map[r] >= n) return -1;
    D = std::max(D, map[r] + 1);
  }
  int pos = 0;
  for (int k = 0; k < D; k++) {
    t->dom_first[k] = pos;
    for (int r = 0; r < n; r++)
      if (map[r] == k) {
        t->rank_dom[r] = k;
        t->rank_idx[r] = pos - t->dom_first[k];
        t->members[pos++] = r;
      }
    t->dom_size[k] = pos - t->dom_first[k];
    if (t->dom_size[k] == 0) return -1;  // ids must be dense (reading R4)
  }
  int L = 1, dmin = n;
  for (int k = 0; k < D; k++) {
    L = L / gcd_(L, t->dom_size[k]) * t->dom_size[k];
    dmin = std::min(dmin, t->dom_size[k]);
  }
  t->n = n;
  t->D = D;
  t->L = L;
  t->dmin = dmin;
  return 0;
}

static size_t floor_to(size_t x, size_t q) { return x / q * q; }
static size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

// quantum (elements) a full tile must be a multiple of, so every boundary is V-aligned
static size_t quantum(const Topo& t, int op, int V) {
  // HETCCL_ALIGN_B: byte alignment of every piece boundary (default 256: 64-byte aligned pieces of
  // non-power-of-two tiles cost 7-9%, q20/q21)
  const char* e = getenv("HETCCL_ALIGN_B");
  const size_t mult = std::max<size_t>(1, (e ? (size_t)atol(e) : 256) / 16);
  if (op == OP_ALLREDUCE || op == OP_REDUCE) return (size_t)t.L * t.D * V * mult;
  if (op == OP_ALL_TO_ALL) return (size_t)V * mult;
  return (size_t)t.L * V * mult;
}

size_t slot_mult_num(const Topo& t, int op, size_t tile) {
  // the largest per-rank slot layout over the domains (kernels.cu; s1/s3 hold domain PEERS only)
  const size_t n = (size_t)t.n, D = (size_t)t.D;
  size_t need = 0;
  for (int k = 0; k < t.D; k++) {
    const size_t d = (size_t)t.dom_size[k], Rk = tile / d, RG = tile + (n - d) * Rk;
    size_t v = 0;
    switch (op) {
      case OP_ALLREDUCE:  // s1[d-1][Rk] | s2[D][Rk] | ag[Rk] | s3[d-1][Rk]
        v = (2 * (d - 1) + D + 1) * Rk;
        break;
      case OP_REDUCE_SCATTER:  // s1[d-1][RG] | s2[D][T]
        v = (d - 1) * RG + D * tile;
        break;
      case OP_ALL_GATHER:  // s_in[d-1][RG] | xin[n-d][T/d]
        v = (d - 1) * RG + (n - d) * Rk;
        break;
      case OP_BROADCAST:  // reg[Rk] | s3[d-1][Rk]
        v = d * Rk;
        break;
      case OP_REDUCE:  // s1[d-1][Rk] | s2[D][Rk] | fin[T] (fin used on the root)
        v = (d - 1 + D) * Rk + tile;
        break;
      case OP_ALL_TO_ALL:  // in[n-1][T] (T per block)
        v = (n - 1) * tile;
        break;
    }
    need = std::max(need, v);
  }
  return need;
}

// default scratch slot (bytes) for a topology: fits the default tile of every op
size_t default_slot_bytes(const Topo& t, size_t tile_bytes) {
  size_t need = 0;
  for (int op = OP_ALLREDUCE; op <= OP_ALL_TO_ALL; op++) {
    size_t tb = tile_bytes;
    if (op == OP_REDUCE_SCATTER || op == OP_ALL_GATHER || op == OP_ALL_TO_ALL)
      tb = std::max<size_t>(tile_bytes / (size_t)t.n, 4096);
    need = std::max(need, slot_mult_num(t, op, tb));
  }
  return (need + 4095) / 4096 * 4096 + 65536;  // room for the quantum rounding of the tile
}

size_t default_tile_bytes(int op, int n, size_t base) {
  const char* e = getenv("HETCCL_TILE_KB");
  size_t b = e ? (size_t)atol(e) * 1024 : (base ? base : (size_t)256 * 1024);
  if (op == OP_REDUCE_SCATTER || op == OP_ALL_GATHER || op == OP_ALL_TO_ALL) b /= (size_t)n;  // per shard / block
  return std::max<size_t>(b, 4096);
}

Geometry make_geometry(const Topo& t, int op, size_t count, int es, int nch_max, size_t slot_elems, size_t tile_base) {
  Geometry g{0, 0, 0};
  if (count == 0) return g;
  const int V = 16 / es;
  const size_t q = quantum(t, op, V);
  // largest tile that fits a slot
  size_t cap = q;
  {
    size_t lo = q, hi = std::max(q, slot_elems);
    hi = floor_to(hi, q);
    while (lo < hi) {  // binary search on multiples of q
      size_t mid = floor_to(lo + (hi - lo) / 2 + q, q);
      if (mid > hi) mid = hi;
      if (slot_mult_num(t, op, mid) <= slot_elems) {
        cap = mid;
        if (mid == lo) break;
        lo = mid;
      } else {
        hi = mid - q;
      }
    }
    if (slot_mult_num(t, op, lo) <= slot_elems) cap = std::max(cap, lo);
  }
  size_t target = std::max(q, floor_to(default_tile_bytes(op, t.n, tile_base) / es, q));
  size_t tile = std::min(cap, target);
  // mid-size messages: shrink the tile (down to a floor) so every channel still gets a few tiles to
  // pipeline, instead of one tile walking all stages serially (HETCCL_MIN_TILES, HETCCL_TILE_FLOOR_KB)
  const char* e1 = getenv("HETCCL_MIN_TILES");
  const char* e2 = getenv("HETCCL_TILE_FLOOR_KB");
  const size_t min_tiles = std::max(1L, e1 ? atol(e1) : 1L);  // measured: 4 or 8 lose 15-35% at 16-128 MiB
  size_t floor_el = std::max(q, floor_to((e2 ? (size_t)atol(e2) * 1024 : (size_t)32768) / es, q));
  if (op == OP_REDUCE_SCATTER || op == OP_ALL_GATHER || op == OP_ALL_TO_ALL)
    floor_el = std::max(q, floor_to(floor_el / (size_t)t.n, q));
  size_t per_ch = ceil_div(count, (size_t)nch_max * min_tiles);
  if (per_ch < tile) tile = std::min(tile, std::max(floor_el, ceil_div(per_ch, q) * q));
  per_ch = ceil_div(count, (size_t)nch_max);
  if (per_ch < tile) tile = std::max(q, ceil_div(per_ch, q) * q);
  // balance: shrink the tile so every channel runs the same number of tiles instead of some channels
  // running one extra round while the others idle (with 256-byte aligned pieces: 1+1 +5%, 2+2 +1%, mux
  // neutral, q21/q22; HETCCL_BALANCE=0 keeps the target tile)
  const char* e3 = getenv("HETCCL_BALANCE");
  if (!(e3 && *e3 == '0')) {
    const size_t nt = ceil_div(count, tile);
    if (nt > (size_t)nch_max) {
      const size_t k = ceil_div(nt, (size_t)nch_max);
      tile = std::max(q, ceil_div(ceil_div(count, (size_t)nch_max * k), q) * q);
    }
  }
  g.tile = tile;
  g.ntiles = ceil_div(count, tile);
  g.nch = (int)std::min<size_t>((size_t)nch_max, g.ntiles);
  return g;
}

int bcast_relay(const Topo& t, int root) {  // -1 if the root is alone in its domain
  const int kr = t.rank_dom[root], d = t.dom_size[kr];
  if (d < 2) return -1;
  return t.members[t.dom_first[kr] + (t.rank_idx[root] + 1) % d];
}

static int owner_of(const Topo& t, int q, int s) {  // domain q's owner of elementary segment s
  int dq = t.dom_size[q];
  return t.members[t.dom_first[q] + s / (t.L / dq)];
}

// Logical stages of each op, in dataflow order (a producer stage always precedes its consumer):
//   AR : A intra push (a1) | B intra fold + cross push (a1/a2) | C cross fold + cross AG (a2) |
//        D intra AG push (a3) | E intra copy-out (a3)
//   RS : A intra push | B domain fold + cross push | C cross fold                       (a6)
//   AG : A cross push | B intra push + copy-out of cross pieces | C intra copy-out     (a7)
//   BC : A root scatter | B cross push | C intra push + copy-out | D intra copy-out     (a8)
// A logical stage is ACTIVE when any rank has work in it (a function of the map and root only, so
// every rank drops the same stages); active stages are packed into pipeline positions 0..P-1.
namespace {
struct StageSpec {
  bool active;
  int wait_ctr;
  uint32_t wait_mask;
  int sig_ctr;
  uint32_t sig_mask;
};
}  // namespace

static int op_spec(const Topo& t, int op, int rank, int root, StageSpec st[kMaxStages]) {
  std::memset(st, 0, sizeof(StageSpec) * kMaxStages);
  for (int s = 0; s < kMaxStages; s++) st[s].wait_ctr = st[s].sig_ctr = C_NONE;
  const int k = t.rank_dom[rank], j = t.rank_idx[rank], d = t.dom_size[k], D = t.D, L = t.L, n = t.n;
  const bool any_intra = D < n, any_cross = D > 1;
  uint32_t dpeers = 0, others = 0;
  for (int r = 0; r < n; r++) {
    if (r == rank) continue;
    if (t.rank_dom[r] == k) dpeers |= 1u << r;
    else others |= 1u << r;
  }
  const int spj = L / d;
  switch (op) {
    case OP_ALLREDUCE: {
      uint32_t cross = 0;  // owners of my segments in the other domains (symmetric relation)
      for (int s = j * spj; s < (j + 1) * spj; s++)
        for (int q = 0; q < D; q++)
          if (q != k) cross |= 1u << owner_of(t, q, s);
      st[0] = {any_intra, C_NONE, 0, C_S1, dpeers};
      st[1] = {true, C_S1, dpeers, C_S2, cross};
      st[2] = {any_cross, C_S2, cross, C_AG, cross};
      st[3] = {true, C_AG, cross, C_S3, dpeers};
      st[4] = {any_intra, C_S3, dpeers, C_NONE, 0};
      return 5;
    }
    case OP_REDUCE_SCATTER:
      st[0] = {any_intra, C_NONE, 0, C_S1, dpeers};
      st[1] = {true, C_S1, dpeers, C_S2, others};
      st[2] = {any_cross, C_S2, others, C_NONE, 0};
      return 3;
    case OP_ALL_GATHER:
      st[0] = {any_cross, C_NONE, 0, C_S2, others};
      st[1] = {true, C_S2, others, C_S1, dpeers};
      st[2] = {any_intra, C_S1, dpeers, C_NONE, 0};
      return 3;
    case OP_BROADCAST: {
      // The root's port is the bound, so with a domain peer available the root only scatters (its own
      // region goes to the RELAY, the next member of its domain, who then does the root's share of the
      // cross push and of the intra all-gather): root egress T per tile instead of up to 2T.
      const int kr = t.rank_dom[root];
      const bool in_root_dom = (k == kr), is_root = (rank == root);
      const int relay = bcast_relay(t, root);
      uint32_t bcross = 0;
      auto cross_of = [&](int s) {  // other domains' owners of root-domain segment s
        for (int q = 0; q < D; q++)
          if (q != kr) bcross |= 1u << owner_of(t, q, s);
      };
      if (in_root_dom && !is_root) {
        for (int s = j * spj; s < (j + 1) * spj; s++) cross_of(s);
        if (rank == relay) {
          const int rj = t.rank_idx[root];
          for (int s = rj * spj; s < (rj + 1) * spj; s++) cross_of(s);
        }
      } else if (in_root_dom && relay < 0) {  // the root is alone in its domain: it pushes cross itself
        for (int s = j * spj; s < (j + 1) * spj; s++) cross_of(s);
      } else if (!in_root_dom) {
        for (int s = j * spj; s < (j + 1) * spj; s++) {
          const int o = owner_of(t, kr, s);
          bcross |= 1u << (o == root && relay >= 0 ? relay : o);
        }
      }
      const uint32_t root_bit = 1u << root;
      st[0] = {t.dom_size[kr] > 1, C_NONE, 0, C_S1, is_root ? dpeers : 0u};
      st[1] = {any_cross || t.dom_size[kr] > 1, C_S1, (in_root_dom && !is_root) ? root_bit : 0u, C_S2, in_root_dom ? bcross : 0u};
      st[2] = {true, C_S2, in_root_dom ? 0u : bcross, C_S3, is_root ? 0u : (dpeers & ~root_bit)};
      st[3] = {any_intra, C_S3, is_root ? 0u : (dpeers & ~root_bit), C_NONE, 0};
      return 4;
    }
    case OP_REDUCE: {
      // A intra push | B fold other domains' pieces -> their owners (D > 1) or my region -> root (D == 1) |
      // C fold my pieces + cross partials -> root | D root: everyone's final pieces -> y
      uint32_t cross = 0;
      for (int s = j * spj; s < (j + 1) * spj; s++)
        for (int q = 0; q < D; q++)
          if (q != k) cross |= 1u << owner_of(t, q, s);
      const uint32_t to_root = rank == root ? 0u : 1u << root;
      uint32_t from_all = 0;
      if (rank == root)
        for (int r = 0; r < n; r++)
          if (r != rank) from_all |= 1u << r;
      st[0] = {any_intra, C_NONE, 0, C_S1, dpeers};
      st[1] = {true, C_S1, dpeers, any_cross ? C_S2 : C_S3, any_cross ? cross : to_root};
      st[2] = {any_cross, C_S2, cross, C_S3, to_root};
      st[3] = {true, C_S3, from_all, C_NONE, 0};
      return 4;
    }
    case OP_ALL_TO_ALL: {
      uint32_t all = 0;
      for (int r = 0; r < n; r++)
        if (r != rank) all |= 1u << r;
      st[0] = {true, C_NONE, 0, C_S1, all};
      st[1] = {true, C_S1, all, C_NONE, 0};
      return 2;
    }
    default:
      return 0;
  }
}

int op_stages(int op) {
  switch (op) {
    case OP_ALLREDUCE: return 5;
    case OP_BROADCAST: return 4;
    case OP_REDUCE: return 4;
    case OP_ALL_TO_ALL: return 2;
    case OP_REDUCE_SCATTER:
    case OP_ALL_GATHER: return 3;
  }
  return 0;
}

// Packs the active logical stages into positions; the kernel maps position -> logical stage with
// the same rule (active flags are identical on every rank). Returns the number of positions.
void make_rank_plan(const Topo& t, int op, int rank, int root, RankPlan* rp) {
  std::memset(rp, 0, sizeof(*rp));
  StageSpec st[kMaxStages];
  const int nl = op_spec(t, op, rank, root, st);
  for (int s = 0; s < kMaxStages; s++) rp->wait_ctr[s] = rp->sig_ctr[s] = C_NONE;
  for (int s = 0; s < nl; s++) {
    // positions are indexed by LOGICAL stage; inactive stages get no waits/signals and are skipped
    if (!st[s].active) continue;
    rp->wait_ctr[s] = (uint8_t)(st[s].wait_mask ? st[s].wait_ctr : C_NONE);
    rp->wait_mask[s] = (uint16_t)st[s].wait_mask;
    rp->sig_ctr[s] = (uint8_t)(st[s].sig_mask ? st[s].sig_ctr : C_NONE);
    rp->sig_mask[s] = (uint16_t)st[s].sig_mask;
    rp->writes |= (uint16_t)st[s].sig_mask;
  }
}

// Bitmask of the logical stages of op that are active for this map/root (same on every rank).
uint32_t active_stages(const Topo& t, int op, int root) {
  StageSpec st[kMaxStages];
  const int nl = op_spec(t, op, 0, root, st);
  uint32_t m = 0;
  for (int s = 0; s < nl; s++)
    if (st[s].active) m |= 1u << s;
  return m;
}

// Algorithmic bytes sent/received over the peer fabric by `rank` for one op, by walking the same
// per-tile partition the kernels execute.
void plan_bytes(const Topo& t, int op, int rank, int root, size_t count, int es, size_t tile, size_t* sent,
                size_t* recv) {
  *sent = *recv = 0;
  if (count == 0 || t.n == 1 || tile == 0) return;
  const int V = 16 / es;
  const int k = t.rank_dom[rank], j = t.rank_idx[rank], d = t.dom_size[k], D = t.D, L = t.L, n = t.n;
  Geometry g{tile, (count + tile - 1) / tile, 0};
  size_t S = 0, R = 0;
  for (size_t ti = 0; ti < g.ntiles; ti++) {
    size_t len = std::min(g.tile, count - ti * g.tile);
    // full-tile grid clipped to len (kernels.cu Geo / sub_lo)
    auto seg = [&](int s) -> size_t { return std::min(len, (size_t)s * (tile / L)); };
    auto piece = [&](int s, int p) -> size_t { return std::min(seg(s + 1), seg(s) + (size_t)p * (tile / L / D)); };
    auto region = [&](int q, int m) -> size_t {  // region length of member m of domain q
      int sp = L / t.dom_size[q];
      return seg((m + 1) * sp) - seg(m * sp);
    };
    auto sub = [&](size_t l, int dd, int i) -> size_t {  // piece i of dd of a shard tile of length l
      return std::min(l, (size_t)(i + 1) * (tile / dd)) - std::min(l, (size_t)i * (tile / dd));
    };
    if (op == OP_ALLREDUCE) {
      const int spj = L / d;
      for (int i = 0; i < d; i++)
        if (i != j) {
          S += region(k, i);  // S1 out
          R += region(k, j);  // S1 in
          S += region(k, j);  // S3 out
          R += region(k, i);  // S3 in
        }
      for (int s = j * spj; s < (j + 1) * spj; s++)
        for (int q = 0; q < D; q++)
          if (q != k) {
            S += piece(s, q + 1) - piece(s, q);  // partial piece out (S2)
            R += piece(s, k + 1) - piece(s, k);  // partial in from domain q
            S += piece(s, k + 1) - piece(s, k);  // reduced piece out to domain q (AG)
            R += piece(s, q + 1) - piece(s, q);  // reduced piece in
          }
    } else if (op == OP_REDUCE_SCATTER || op == OP_ALL_GATHER) {
      size_t reg = len;  // own shard + my piece of every other-domain shard
      for (int r = 0; r < n; r++)
        if (t.rank_dom[r] != k) reg += sub(len, d, j);
      size_t intra_out = 0, intra_in = 0, cross_out = 0, cross_in = 0;
      for (int i = 0; i < d; i++)
        if (i != j) {
          size_t regi = len;
          for (int r = 0; r < n; r++)
            if (t.rank_dom[r] != k) regi += sub(len, d, i);
          intra_out += regi;  // RS: my data for peer i's region
          intra_in += reg;    // RS: peer's data for my region
        }
      for (int r = 0; r < n; r++)
        if (t.rank_dom[r] != k) {
          cross_out += sub(len, d, j);  // RS: my partial piece of shard r to r
        }
      for (int q = 0; q < D; q++)
        if (q != k)
          for (int i = 0; i < t.dom_size[q]; i++) cross_in += sub(len, t.dom_size[q], i);  // = len per domain
      if (op == OP_REDUCE_SCATTER) {
        S += intra_out + cross_out;
        R += intra_in + cross_in;
      } else {  // AG is the mirror image
        S += intra_in + cross_in;
        R += intra_out + cross_out;
      }
    } else if (op == OP_REDUCE) {
      const int spj = L / d;
      for (int i = 0; i < d; i++)
        if (i != j) {
          S += region(k, i);  // intra RS out
          R += region(k, j);  // intra RS in
        }
      for (int s = j * spj; s < (j + 1) * spj; s++)
        for (int q = 0; q < D; q++)
          if (q != k) {
            S += piece(s, q + 1) - piece(s, q);  // partial piece out
            R += piece(s, k + 1) - piece(s, k);  // partial in from domain q
          }
      size_t mine = 0;  // final pieces I own
      for (int s = j * spj; s < (j + 1) * spj; s++) mine += piece(s, k + 1) - piece(s, k);
      if (D == 1) mine = region(k, j);
      if (rank != root) S += mine;
      else R += len - mine;
    } else if (op == OP_ALL_TO_ALL) {
      S += len * (size_t)(n - 1);
      R += len * (size_t)(n - 1);
    } else if (op == OP_BROADCAST) {
      const int kr = t.rank_dom[root], spj = L / d, relay = bcast_relay(t, root), rj = t.rank_idx[root];
      const bool in_root_dom = (k == kr), is_root = (rank == root);
      // A: the root scatters every region of its domain (its own to the relay)
      if (is_root)
        for (int i = 0; i < d; i++)
          if (i != j) S += region(k, i) + (t.members[t.dom_first[k] + i] == relay ? region(k, j) : 0);
      if (in_root_dom && !is_root) R += region(k, j) + (rank == relay ? region(k, rj) : 0);
      // B: each root-domain segment crosses once to every other domain (the root's segments via the relay)
      if (D > 1) {
        const bool pushes = in_root_dom && (!is_root || relay < 0);
        for (int s = 0; s < L; s++) {
          const size_t sl = seg(s + 1) - seg(s);
          const int o = owner_of(t, kr, s);
          const int sender = (o == root && relay >= 0) ? relay : o;
          if (pushes && sender == rank) S += sl * (size_t)(D - 1);
          if (!in_root_dom && owner_of(t, k, s) == rank) R += sl;
        }
      }
      // C: intra all-gather among the non-root members (the relay also forwards the root's region)
      if (!is_root)
        for (int i = 0; i < d; i++) {
          if (i == j) continue;
          const int peer = t.members[t.dom_first[k] + i];
          if (peer == root) continue;
          S += region(k, j);
          if (in_root_dom && rank == relay) S += region(k, rj);  // the root's region, on the root's behalf
          R += region(k, i);
          if (in_root_dom && peer == relay) R += region(k, rj);
        }
    }
  }
  *sent = S * (size_t)es;
  *recv = R * (size_t)es;
}

}  // namespace hetccl
