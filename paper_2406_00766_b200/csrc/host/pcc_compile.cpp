// Native core of the host compiler (compiler/build.py, restating
// pcirc/compiler/build.py:183-631 and blocks.py:73-148).
//
// The Python driver keeps the orchestration and the per-block / per-product
// tables; everything proportional to the edge count runs here:
//   * pcc_gather_layer  - one sum layer's edge arrays from its segments
//                         (build.py:195-222: child key, slot per edge);
//   * pcc_blocks_*      - connectivity-class block detection (blocks.py:73-148):
//                         product classes keyed by the sorted parent list in
//                         first-occurrence order over ascending key, sum classes
//                         keyed by the sorted child-block set in sum order,
//                         k-chunking with PAD tails, demotion to 1 x 1;
//   * pcc_tiles         - the layer's (sum block, product block) tiles
//                         (build.py:251-339): tile grids of slots, the tied
//                         rep-slot pattern dedupe (within the layer and against
//                         every earlier layer), theta fill, slot_phys, the
//                         parallel-edge and tying-alignment checks;
//   * pcc_sum_groups_multi / pcc_rows_* - the sorted physical positions of
//                         every sum row for the simplex groups (build.py:535-567),
//                         with overlap claims;
//   * pcc_hash_records_multi - the graph_hash byte records (build.py:634-657);
//   * pcc_depths, pcc_group_runs, pcc_minmax, pcc_narrow_i32 - graph depths and
//                         the device-plan table helpers.
// Orderings are the reference's (dict insertion = first occurrence, np.unique
// = ascending); grouping is exact (64-bit row hashes, then element-wise
// comparison with the group representative).  Parallel loops are plain
// std::thread workers over contiguous ranges; every parallel write is either
// to a disjoint range or an idempotent / compare-and-swap update, so the
// output is independent of the thread count.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../../include/pcirc_host.h"

namespace {
using i64 = int64_t;
using u64 = uint64_t;

int g_threads = 0;

int nthreads() {
  if (g_threads <= 0) {
    unsigned h = std::thread::hardware_concurrency();
    g_threads = h ? (int)std::min(h, 64u) : 1;
  }
  return g_threads;
}

// f(lo, hi, worker) over [0, n) split into contiguous ranges
template <class F>
void pfor(i64 n, F&& f, i64 grain = 1 << 14) {
  if (n <= 0) return;
  const int T = (int)std::min<i64>(nthreads(), (n + grain - 1) / grain);
  if (T <= 1) {
    f((i64)0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (int t = 0; t < T; ++t) {
    const i64 lo = n * t / T, hi = n * (t + 1) / T;
    th.emplace_back([&f, lo, hi, t] { f(lo, hi, t); });
  }
  for (auto& x : th) x.join();
}

inline u64 mix(u64 z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline u64 row_hash(const i64* v, i64 n) {
  u64 h = 0;
  for (i64 i = 0; i < n; ++i) h += mix((u64)v[i] ^ mix((u64)i));
  return mix(h ^ mix((u64)n * 0x94D049BB133111EBull));
}

// open-addressing map: 64-bit hash -> head of a chain of group ids
struct HashHeads {
  std::vector<u64> key;
  std::vector<i64> head;
  u64 mask = 0;
  void init(i64 n) {
    u64 cap = 16;
    while (cap < (u64)(2 * n + 16)) cap <<= 1;
    key.assign(cap, 0);
    head.assign(cap, -1);
    mask = cap - 1;
  }
  i64& at(u64 h) {  // creates an empty (-1) chain on first sight
    u64 i = mix(h) & mask;
    while (head[i] >= 0 && key[i] != h) i = (i + 1) & mask;
    key[i] = h;
    return head[i];
  }
};

struct Groups {
  std::vector<i64> gid;    // per row
  std::vector<i64> first;  // per group: its first row
};

// Exact grouping of rows 0..n-1 (row(i) -> {ptr, len}), numbered by first
// occurrence (the reference's dict-insertion order).
template <class Row>
Groups group_rows(i64 n, Row row) {
  Groups g;
  g.gid.resize(n);
  std::vector<u64> h(n);
  pfor(n, [&](i64 lo, i64 hi, int) {
    for (i64 i = lo; i < hi; ++i) {
      const auto r = row(i);
      h[i] = row_hash(r.first, r.second);
    }
  }, 1 << 10);
  HashHeads idx;
  idx.init(n);
  std::vector<i64> next;
  for (i64 i = 0; i < n; ++i) {
    i64& hd = idx.at(h[i]);
    const auto ri = row(i);
    i64 found = -1;
    for (i64 c = hd; c >= 0; c = next[c]) {
      const auto rc = row(g.first[c]);
      if (rc.second == ri.second &&
          (ri.second == 0 || std::memcmp(rc.first, ri.first, sizeof(i64) * ri.second) == 0)) {
        found = c;
        break;
      }
    }
    if (found < 0) {
      found = (i64)g.first.size();
      g.first.push_back(i);
      next.push_back(hd);
      hd = found;
    }
    g.gid[i] = found;
  }
  return g;
}

// blocks.py:50-70: chunk classes (first-occurrence numbered) into k-blocks,
// members in index order within a class.  blk / off per member, mat of
// member indices (-1 = PAD).
void chunk(i64 m, const std::vector<i64>& gid, i64 ncls, i64 k, std::vector<i64>& blk,
           std::vector<i64>& off, std::vector<i64>& mat, i64& nblk_total, double& pad) {
  std::vector<i64> size(ncls, 0), base(ncls), cur(ncls, 0);
  for (i64 i = 0; i < m; ++i) ++size[gid[i]];
  i64 b = 0;
  for (i64 c = 0; c < ncls; ++c) {
    base[c] = b;
    b += (size[c] + k - 1) / k;
  }
  nblk_total = b;
  blk.resize(m);
  off.resize(m);
  mat.assign(b * k, -1);
  for (i64 i = 0; i < m; ++i) {
    const i64 c = gid[i], r = cur[c]++;
    blk[i] = base[c] + r / k;
    off[i] = r % k;
    mat[blk[i] * k + off[i]] = i;
  }
  const i64 total = b * k;
  pad = total ? (double)(total - m) / (double)total : 0.0;
}

i64 pow2_floor(i64 n) {
  i64 p = 1;
  while (p * 2 <= n) p *= 2;
  return p;
}

// Uninitialised scratch reused across layers: no zero fill, and pages
// first-touched once by the parallel writers (released by pcc_release).
struct Scratch {
  std::unique_ptr<i64[]> p;
  size_t n = 0;
  i64* get(size_t m) {
    if (m > n) {
      p.reset(new i64[m]);
      n = m;
    }
    return p.get();
  }
  void release() {
    p.reset();
    n = 0;
  }
};
// per calling thread: concurrent compiles from several Python threads (ctypes
// releases the GIL) never share a buffer
thread_local Scratch g_tmp, g_par, g_grid, g_pat, g_rows;

struct Layer {
  // caller-owned inputs (kept alive by the Python layer object)
  i64 n = 0, E = 0;
  const i64* sids = nullptr;  // (n) sum ids, row order
  const i64* key = nullptr;   // (E) child keys
  const i64* off = nullptr;   // (n + 1)
  // products
  i64 kmin = 0;
  std::vector<int32_t> kix;  // key - kmin -> product index (ascending key)
  std::vector<i64> pkeys;
  Groups pcls;
  // blocking
  i64 km = 1, kn = 1, n_pb = 0, n_sb = 0;
  bool demoted = false;
  double spad = 0, ppad = 0;
  std::vector<i64> pblk, poff, pmat;  // per product / (n_pb, kn) product indices
  std::vector<i64> sblk, soff, smat;  // per row / (n_sb, km) row indices
  std::vector<i64> b2_off, b2;        // per row: sorted unique child blocks
  std::vector<i64> cb_off, cb_flat;   // per sum block (its first member's set)
  std::vector<i64> sorder;            // rows by ascending sum id (stable)
  // tiles
  std::vector<i64> pair_theta;
  i64 n_new_tiles = 0;
};

inline int32_t pidx(const Layer& L, i64 k) { return L.kix[(size_t)(k - L.kmin)]; }

void sum_sets(Layer& L) {
  const i64 n = L.n;
  i64* tmp = g_tmp.get((size_t)L.E);
  std::vector<i64> ulen(n);
  pfor(n, [&](i64 lo, i64 hi, int) {
    for (i64 r = lo; r < hi; ++r) {
      const i64 a = L.off[r], b = L.off[r + 1];
      i64 c = 0, last = -1;
      for (i64 e = a; e < b; ++e) {
        const i64 bl = L.pblk[pidx(L, L.key[e])];
        if (c == 0 || bl != last) tmp[a + c++] = bl;
        last = bl;
      }
      std::sort(tmp + a, tmp + a + c);
      ulen[r] = std::unique(tmp + a, tmp + a + c) - (tmp + a);
    }
  }, 1 << 8);
  L.b2_off.assign(n + 1, 0);
  for (i64 r = 0; r < n; ++r) L.b2_off[r + 1] = L.b2_off[r] + ulen[r];
  L.b2.resize(L.b2_off[n]);
  pfor(n, [&](i64 lo, i64 hi, int) {
    for (i64 r = lo; r < hi; ++r)
      std::copy(tmp + L.off[r], tmp + L.off[r] + ulen[r], L.b2.begin() + L.b2_off[r]);
  }, 1 << 10);
}

void block_pass(Layer& L, i64 km, i64 kn) {
  L.km = km;
  L.kn = kn;
  chunk((i64)L.pkeys.size(), L.pcls.gid, (i64)L.pcls.first.size(), kn, L.pblk, L.poff, L.pmat,
        L.n_pb, L.ppad);
  sum_sets(L);
  Groups s = group_rows(L.n, [&](i64 r) {
    return std::pair<const i64*, i64>(L.b2.data() + L.b2_off[r], L.b2_off[r + 1] - L.b2_off[r]);
  });
  chunk(L.n, s.gid, (i64)s.first.size(), km, L.sblk, L.soff, L.smat, L.n_sb, L.spad);
}

int blocks(Layer& L, i64 k, i64 k_n, double demote) {
  const i64 n = L.n, E = L.E;
  // product keys: dense index over the key range
  i64 kmin = 0, kmax = -1;
  if (E) {
    std::vector<i64> mn(nthreads(), INT64_MAX), mx(nthreads(), INT64_MIN);
    pfor(E, [&](i64 lo, i64 hi, int t) {
      i64 a = INT64_MAX, b = INT64_MIN;
      for (i64 e = lo; e < hi; ++e) a = std::min(a, L.key[e]), b = std::max(b, L.key[e]);
      mn[t] = std::min(mn[t], a), mx[t] = std::max(mx[t], b);
    });
    kmin = *std::min_element(mn.begin(), mn.end());
    kmax = *std::max_element(mx.begin(), mx.end());
  }
  const i64 R = kmax - kmin + 1;
  if (R > ((i64)1 << 31) - 2) return 3;
  L.kmin = kmin;
  L.kix.assign((size_t)std::max<i64>(R, 0), -1);
  pfor(E, [&](i64 lo, i64 hi, int) {
    for (i64 e = lo; e < hi; ++e) __atomic_store_n(&L.kix[L.key[e] - kmin], 0, __ATOMIC_RELAXED);
  });
  L.pkeys.clear();
  for (i64 j = 0; j < R; ++j)
    if (L.kix[j] == 0) {
      L.kix[j] = (int32_t)L.pkeys.size();
      L.pkeys.push_back(kmin + j);
    }
  const i64 P = (i64)L.pkeys.size();
  // sum rows by ascending sum id (stable); the product parent lists follow it
  L.sorder.resize(n);
  for (i64 r = 0; r < n; ++r) L.sorder[r] = r;
  bool asc = true;
  for (i64 r = 1; r < n && asc; ++r) asc = L.sids[r] > L.sids[r - 1];
  if (!asc)
    std::stable_sort(L.sorder.begin(), L.sorder.end(),
                     [&](i64 a, i64 b) { return L.sids[a] < L.sids[b]; });
  // parents per product key (counting sort, T row chunks in sum-id order)
  const int T = std::max(1, std::min<int>(nthreads(), (int)((n + 255) / 256)));
  std::vector<i64> cnt((size_t)T * P, 0);
  auto chunk_lo = [&](int t) { return n * t / T; };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        i64* c = cnt.data() + (size_t)t * P;
        for (i64 q = chunk_lo(t); q < chunk_lo(t + 1); ++q) {
          const i64 r = L.sorder[q];
          for (i64 e = L.off[r]; e < L.off[r + 1]; ++e) ++c[pidx(L, L.key[e])];
        }
      });
    for (auto& x : th) x.join();
  }
  std::vector<i64> poff_par(P + 1, 0);
  for (i64 p = 0; p < P; ++p) {
    i64 s = poff_par[p];
    for (int t = 0; t < T; ++t) {
      const i64 v = cnt[(size_t)t * P + p];
      cnt[(size_t)t * P + p] = s;
      s += v;
    }
    poff_par[p + 1] = s;
  }
  i64* par = g_par.get((size_t)E);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        i64* c = cnt.data() + (size_t)t * P;
        for (i64 q = chunk_lo(t); q < chunk_lo(t + 1); ++q) {
          const i64 r = L.sorder[q];
          for (i64 e = L.off[r]; e < L.off[r + 1]; ++e) par[c[pidx(L, L.key[e])]++] = L.sids[r];
        }
      });
    for (auto& x : th) x.join();
  }
  cnt = std::vector<i64>();
  L.pcls = group_rows(P, [&](i64 p) {
    return std::pair<const i64*, i64>(par + poff_par[p], poff_par[p + 1] - poff_par[p]);
  });
  const i64 kn0 = std::min(k_n, pow2_floor(std::max<i64>(P, 1)));
  const i64 km0 = std::min(k, pow2_floor(std::max<i64>(n, 1)));
  block_pass(L, km0, kn0);
  L.demoted = false;
  if (std::max(L.spad, L.ppad) > demote && std::max(km0, kn0) > 1) {
    block_pass(L, 1, 1);
    L.demoted = true;
  }
  // child blocks of each sum block = those of its first member
  L.cb_off.assign(L.n_sb + 1, 0);
  for (i64 b = 0; b < L.n_sb; ++b) {
    const i64 r = L.smat[b * L.km];
    L.cb_off[b + 1] = L.cb_off[b] + (L.b2_off[r + 1] - L.b2_off[r]);
  }
  L.cb_flat.resize(L.cb_off[L.n_sb]);
  for (i64 b = 0; b < L.n_sb; ++b) {
    const i64 r = L.smat[b * L.km];
    std::copy(L.b2.begin() + L.b2_off[r], L.b2.begin() + L.b2_off[r + 1], L.cb_flat.begin() + L.cb_off[b]);
  }
  return 0;
}

// ----------------------------------------------------------------- tiles
struct TileEntry {
  i64 start, tile;
  std::vector<i64> pattern;
};

struct TileTable {
  std::unordered_map<u64, std::vector<TileEntry>> by_hash;  // keyed by (tilesz, hash)
  std::vector<i64> starts, writers;                          // per tile, creation order
};


inline u64 table_key(i64 tilesz, u64 h) { return h ^ mix((u64)tilesz * 0x9E3779B97F4A7C15ull); }

}  // namespace

extern "C" {

int pcc_version() { return 1; }

void pcc_set_threads(int n) { g_threads = n; }

int pcc_threads() { return nthreads(); }

// One sum layer's per-edge sum ids / child ids / child keys / slots from its
// segments: segment s contributes rows rows[s][0..nrows[s]) (or 0..nrows[s]
// when rows[s] is null) of its (count, fan) children / slots matrices, in the
// given order; starts[s] is its first node id.  Children rows are
// ch_stride[s] elements apart (0: one row broadcast to every sum).
void pcc_gather_layer(int nseg, const i64* const* children, const i64* ch_stride,
                      const i64* const* slots, const i64* fan, const i64* const* rows,
                      const i64* nrows, const i64* starts,
                      const int8_t* kinds, int8_t product_kind, i64 vkey_base, i64* e_sum,
                      i64* e_child, i64* e_key, i64* e_slot) {
  std::vector<i64> rbase(nseg + 1, 0), ebase(nseg + 1, 0);
  for (int s = 0; s < nseg; ++s) {
    rbase[s + 1] = rbase[s] + nrows[s];
    ebase[s + 1] = ebase[s] + nrows[s] * fan[s];
  }
  const i64 nr_all = rbase[nseg];
  const i64 E = ebase[nseg];
  const i64 avg = nr_all ? std::max<i64>(1, E / nr_all) : 1;
  pfor(nr_all, [&](i64 lo, i64 hi, int) {
    int s = (int)(std::upper_bound(rbase.begin(), rbase.end(), lo) - rbase.begin()) - 1;
    for (i64 g = lo; g < hi; ++g) {
      while (g >= rbase[s + 1]) ++s;
      const i64 q = g - rbase[s], f = fan[s];
      const i64 r = rows[s] ? rows[s][q] : q;
      const i64* c = children[s] + r * ch_stride[s];
      const i64* sl = slots[s] + r * f;
      const i64 o = ebase[s] + q * f, sid = starts[s] + r;
      for (i64 j = 0; j < f; ++j) {
        const i64 ch = c[j];
        e_sum[o + j] = sid;
        e_child[o + j] = ch;
        e_key[o + j] = kinds[ch] == product_kind ? ch : vkey_base - ch;
        e_slot[o + j] = sl[j];
      }
    }
  }, std::max<i64>(1, (1 << 15) / avg));
}

void pcc_fill_i64(i64* p, i64 n, i64 v) {
  pfor(n, [&](i64 lo, i64 hi, int) { std::fill(p + lo, p + hi, v); }, 1 << 20);
}

// dst[dst_start[i] + j] = src[src_start[i] + j], j < len[i]
void pcc_copy_ranges(i64 n, const i64* src_start, const i64* len, const i64* dst_start,
                     const double* src, double* dst) {
  pfor(n, [&](i64 lo, i64 hi, int) {
    for (i64 i = lo; i < hi; ++i) std::memcpy(dst + dst_start[i], src + src_start[i], 8 * len[i]);
  }, 1 << 8);
}

// out[dst_off[i] + j] = start[i] + j, j < len[i]
void pcc_iota_ranges(i64 n, const i64* dst_off, const i64* start, const i64* len, i64* out) {
  pfor(n, [&](i64 lo, i64 hi, int) {
    for (i64 i = lo; i < hi; ++i)
      for (i64 j = 0; j < len[i]; ++j) out[dst_off[i] + j] = start[i] + j;
  }, 1 << 8);
}

// slot_phys[slot_start[i] + j] = phys_start[i] + j (in order when `ordered`:
// overlapping ranges, last write wins), and the tying check of each
// (slot, phys) against ref (null = none).  Returns 1 if misaligned.
int pcc_assign_ranges(i64 n, const i64* slot_start, const i64* len, const i64* phys_start,
                      int ordered, i64* slot_phys, const i64* rep, i64* ref) {
  std::atomic<int> bad{0};
  auto body = [&](i64 lo, i64 hi, int) {
    for (i64 i = lo; i < hi; ++i)
      for (i64 j = 0; j < len[i]; ++j) {
        const i64 sl = slot_start[i] + j, ph = phys_start[i] + j;
        slot_phys[sl] = ph;
        if (ref) {
          const i64 r = rep ? rep[sl] : sl;
          i64 expect = -1;
          if (!__atomic_compare_exchange_n(&ref[r], &expect, ph, false, __ATOMIC_RELAXED,
                                           __ATOMIC_RELAXED) &&
              expect != ph)
            bad.store(1, std::memory_order_relaxed);
        }
      }
  };
  if (ordered)
    body(0, n, 0);
  else
    pfor(n, body, 1 << 8);
  return bad.load();
}

// Claims the positions of n ranges in a bitset; 1 if any was claimed before.
int pcc_claim_ranges(i64 n, const i64* start, const i64* len, u64* bits) {
  std::atomic<int> bad{0};
  pfor(n, [&](i64 lo, i64 hi, int) {
    for (i64 i = lo; i < hi; ++i)
      for (i64 j = 0; j < len[i]; ++j) {
        const u64 p = (u64)(start[i] + j), bit = 1ull << (p & 63);
        if (__atomic_fetch_or(&bits[p >> 6], bit, __ATOMIC_RELAXED) & bit)
          bad.store(1, std::memory_order_relaxed);
      }
  }, 1 << 8);
  return bad.load();
}

void* pcc_layer_new(i64 n, const i64* sids, i64 E, const i64* key, const i64* off) {
  Layer* L = new Layer;
  L->n = n, L->E = E, L->sids = sids, L->key = key, L->off = off;
  return L;
}

void pcc_layer_free(void* h) { delete static_cast<Layer*>(h); }

// 0 ok, 3 key range too large
int pcc_blocks(void* h, i64 k, i64 k_n, double demote) {
  return blocks(*static_cast<Layer*>(h), k, k_n, demote);
}

// meta: km, kn, demoted, n_sb, n_pb, n_prod_keys, n_cb; pads
void pcc_blocks_meta(void* h, i64* meta, double* pads) {
  const Layer& L = *static_cast<Layer*>(h);
  meta[0] = L.km, meta[1] = L.kn, meta[2] = L.demoted, meta[3] = L.n_sb, meta[4] = L.n_pb;
  meta[5] = (i64)L.pkeys.size(), meta[6] = (i64)L.cb_flat.size();
  pads[0] = L.spad, pads[1] = L.ppad;
}

// copies: smat (n_sb * km sum keys, PAD -1), pmat (n_pb * kn product keys),
// cb_flat, cb_off, sum_keys / sum_blk / sum_off (ascending sum id),
// prod_keys / prod_blk / prod_off (ascending key)
void pcc_blocks_get(void* h, i64* smat, i64* pmat, i64* cb_flat, i64* cb_off, i64* sum_keys,
                    i64* sum_blk, i64* sum_off, i64* prod_keys, i64* prod_blk, i64* prod_off) {
  const Layer& L = *static_cast<Layer*>(h);
  for (size_t i = 0; i < L.smat.size(); ++i) smat[i] = L.smat[i] < 0 ? -1 : L.sids[L.smat[i]];
  for (size_t i = 0; i < L.pmat.size(); ++i) pmat[i] = L.pmat[i] < 0 ? -1 : L.pkeys[L.pmat[i]];
  std::copy(L.cb_flat.begin(), L.cb_flat.end(), cb_flat);
  std::copy(L.cb_off.begin(), L.cb_off.end(), cb_off);
  for (i64 q = 0; q < L.n; ++q) {
    const i64 r = L.sorder[q];
    sum_keys[q] = L.sids[r], sum_blk[q] = L.sblk[r], sum_off[q] = L.soff[r];
  }
  std::copy(L.pkeys.begin(), L.pkeys.end(), prod_keys);
  std::copy(L.pblk.begin(), L.pblk.end(), prod_blk);
  std::copy(L.poff.begin(), L.poff.end(), prod_off);
}

// Marks every rep slot used by a sum edge: bit r of `seen`, and of `multi`
// once it is used a second time (tile patterns containing a once-used rep
// slot cannot equal any other tile).
void pcc_slot_uses(i64 E, const i64* slots, const i64* rep, u64* seen, u64* multi) {
  pfor(E, [&](i64 lo, i64 hi, int) {
    for (i64 e = lo; e < hi; ++e) {
      const u64 r = (u64)(rep ? rep[slots[e]] : slots[e]);
      const u64 bit = 1ull << (r & 63);
      const u64 old = __atomic_fetch_or(&seen[r >> 6], bit, __ATOMIC_RELAXED);
      if (old & bit) __atomic_fetch_or(&multi[r >> 6], bit, __ATOMIC_RELAXED);
    }
  });
}

void* pcc_tiles_new() { return new TileTable; }

void pcc_tiles_free(void* t) { delete static_cast<TileTable*>(t); }

// frees the scratch buffers kept across the layers of one compile
void pcc_release() {
  for (Scratch* b : {&g_tmp, &g_par, &g_grid, &g_pat, &g_rows}) b->release();
}

i64 pcc_tiles_count(void* t) { return (i64)static_cast<TileTable*>(t)->starts.size(); }

void pcc_tiles_get(void* t, i64* starts, i64* writers) {
  const TileTable& T = *static_cast<TileTable*>(t);
  std::copy(T.starts.begin(), T.starts.end(), starts);
  std::copy(T.writers.begin(), T.writers.end(), writers);
}

// build.py:251-339 for one blocked layer.  slots: (E) param slot per edge;
// rep: tied representative per slot (null = identity); multi: bitset of rep
// slots used more than once by sum edges (null = none are); params: slot
// values; theta: output buffer of capacity theta_cap, *theta_size advanced
// by the new tiles; slot_phys updated; ref (null = no tying check): per rep
// slot its physical position.  pair_theta (n_cb) out: the tile start of
// every (sum block, child block) pair in cb order.
// Returns 0 ok, 1 parallel edge, 2 tying misaligned, 4 theta capacity.
int pcc_tiles(void* h, void* table, const i64* slots, const i64* rep, const u64* multi,
              const double* params, double* theta, i64 theta_cap, i64* theta_size,
              i64* slot_phys, i64* ref, i64* pair_theta) {
  Layer& L = *static_cast<Layer*>(h);
  TileTable& T = *static_cast<TileTable*>(table);
  const i64 km = L.km, kn = L.kn, tsz = km * kn;
  const i64 npair = (i64)L.cb_flat.size();
  i64* grid = g_grid.get((size_t)(npair * tsz));
  pfor(npair * tsz, [&](i64 lo, i64 hi, int) { std::fill(grid + lo, grid + hi, (i64)-1); }, 1 << 20);
  std::atomic<int> dup{0};
  pfor(L.n, [&](i64 lo, i64 hi, int) {
    for (i64 r = lo; r < hi; ++r) {
      const i64 sb = L.sblk[r], so = L.soff[r];
      const i64* cb = L.cb_flat.data() + L.cb_off[sb];
      const i64 ncb = L.cb_off[sb + 1] - L.cb_off[sb];
      i64 last_pb = -1, pair = -1;
      for (i64 e = L.off[r]; e < L.off[r + 1]; ++e) {
        const i64 p = pidx(L, L.key[e]);
        const i64 pb = L.pblk[p];
        if (pb != last_pb) {
          pair = L.cb_off[sb] + (std::lower_bound(cb, cb + ncb, pb) - cb);
          last_pb = pb;
        }
        i64* g = &grid[(size_t)(pair * tsz + so * kn + L.poff[p])];
        i64 expect = -1;
        if (!__atomic_compare_exchange_n(g, &expect, slots[e], false, __ATOMIC_RELAXED,
                                         __ATOMIC_RELAXED))
          dup.store(1, std::memory_order_relaxed);
      }
    }
  }, 1 << 6);
  if (dup.load()) return 1;
  // unique rows: some entry's rep slot is used once
  std::vector<uint8_t> uniq(npair, 1);
  if (multi) {
    pfor(npair, [&](i64 lo, i64 hi, int) {
      for (i64 q = lo; q < hi; ++q) {
        const i64* g = &grid[(size_t)(q * tsz)];
        bool u = false;
        for (i64 t = 0; t < tsz && !u; ++t)
          if (g[t] >= 0) {
            const u64 rr = (u64)(rep ? rep[g[t]] : g[t]);
            u = !((multi[rr >> 6] >> (rr & 63)) & 1);
          }
        uniq[q] = u;
      }
    }, 1 << 8);
  }
  // patterns (rep slot or -1) and hashes of the shared-able rows
  std::vector<i64> shared_rows;
  for (i64 q = 0; q < npair; ++q)
    if (!uniq[q]) shared_rows.push_back(q);
  const i64 ns = (i64)shared_rows.size();
  i64* pat = g_pat.get((size_t)(ns * tsz));
  std::vector<u64> hsh(ns);
  pfor(ns, [&](i64 lo, i64 hi, int) {
    for (i64 i = lo; i < hi; ++i) {
      const i64* g = &grid[(size_t)(shared_rows[i] * tsz)];
      i64* pp = &pat[(size_t)(i * tsz)];
      for (i64 t = 0; t < tsz; ++t) pp[t] = g[t] < 0 ? -1 : (rep ? rep[g[t]] : g[t]);
      hsh[i] = row_hash(pp, tsz);
    }
  }, 1 << 6);
  // tile starts in pair order (first occurrence within the layer, then the
  // global table of earlier layers' tied patterns)
  HashHeads local;
  local.init(ns);
  std::vector<i64> lnext, lfirst, lstart, ltile;
  std::vector<i64> new_rows;  // pair index of each new tile, in allocation order
  i64 ts = *theta_size;
  i64 si = 0;
  for (i64 q = 0; q < npair; ++q) {
    if (uniq[q]) {
      pair_theta[q] = ts;
      T.starts.push_back(ts);
      T.writers.push_back(1);
      new_rows.push_back(q);
      ts += tsz;
      continue;
    }
    const i64 i = si++;
    const i64* pp = &pat[(size_t)(i * tsz)];
    i64& hd = local.at(hsh[i]);
    i64 found = -1;
    for (i64 c = hd; c >= 0; c = lnext[c])
      if (std::memcmp(&pat[(size_t)(lfirst[c] * tsz)], pp, sizeof(i64) * tsz) == 0) {
        found = c;
        break;
      }
    if (found >= 0) {
      pair_theta[q] = lstart[found];
      ++T.writers[ltile[found]];
      continue;
    }
    // a new group of this layer: the global table, else a new tile
    auto& bucket = T.by_hash[table_key(tsz, hsh[i])];
    i64 start = -1, tile = -1;
    for (const auto& en : bucket)
      if ((i64)en.pattern.size() == tsz &&
          std::memcmp(en.pattern.data(), pp, sizeof(i64) * tsz) == 0) {
        start = en.start, tile = en.tile;
        break;
      }
    if (start < 0) {
      start = ts;
      tile = (i64)T.starts.size();
      T.starts.push_back(ts);
      T.writers.push_back(0);
      bucket.push_back(TileEntry{start, tile, std::vector<i64>(pp, pp + tsz)});
      new_rows.push_back(q);
      ts += tsz;
    }
    lfirst.push_back(i);
    lstart.push_back(start);
    ltile.push_back(tile);
    lnext.push_back(hd);
    hd = (i64)lfirst.size() - 1;
    pair_theta[q] = start;
    ++T.writers[tile];
  }
  if (ts > theta_cap) return 4;
  // theta of the new tiles
  const i64 nnew = (i64)new_rows.size();
  pfor(nnew, [&](i64 lo, i64 hi, int) {
    for (i64 j = lo; j < hi; ++j) {
      const i64* g = &grid[(size_t)(new_rows[j] * tsz)];
      double* out = theta + pair_theta[new_rows[j]];
      for (i64 t = 0; t < tsz; ++t) out[t] = g[t] >= 0 ? params[g[t]] : 0.0;
    }
  }, 1 << 6);
  *theta_size = ts;
  L.n_new_tiles = nnew;
  // slot_phys and the tying alignment check
  std::atomic<int> bad{0};
  pfor(npair, [&](i64 lo, i64 hi, int) {
    for (i64 q = lo; q < hi; ++q) {
      const i64* g = &grid[(size_t)(q * tsz)];
      const i64 st = pair_theta[q];
      for (i64 t = 0; t < tsz; ++t) {
        if (g[t] < 0) continue;
        const i64 phys = st + t;
        slot_phys[g[t]] = phys;
        if (ref) {
          const i64 r = rep ? rep[g[t]] : g[t];
          i64 expect = -1;
          if (!__atomic_compare_exchange_n(&ref[r], &expect, phys, false, __ATOMIC_RELAXED,
                                           __ATOMIC_RELAXED) &&
              expect != phys)
            bad.store(1, std::memory_order_relaxed);
        }
      }
    }
  }, 1 << 6);
  return bad.load() ? 2 : 0;
}

// ---------------------------------------------------------------- simplex
// Exact grouping of the sorted physical rows of non-contiguous sums
// (build.py:535-567, the general path): rows are added segment by segment in
// node-id order; contiguous rows are reported back as ranges.
struct RowGroups {
  HashHeads heads;
  std::vector<i64> next, first_id, off{0}, members;
  std::vector<u64> hash;
  i64 cap = 0;
};

void* pcc_rows_new() { return new RowGroups; }

void pcc_rows_free(void* h) { delete static_cast<RowGroups*>(h); }

// Rows of several segments of one fan-in (segment s: counts[s] rows of its
// (count, fan) slot matrix, node ids id0s[s] + i), in the order given (node-id
// order).  contig_start (one per row, concatenated): first position of a
// contiguous row, else -1.  Rows are sorted and hashed in parallel chunks;
// grouping is sequential in row order (first occurrence).
void pcc_rows_add_multi(void* h, i64 nseg, const i64* counts, i64 fan,
                        const i64* const* slot_ptrs, const i64* id0s, const i64* slot_phys,
                        i64* contig_start) {
  RowGroups& G = *static_cast<RowGroups*>(h);
  std::vector<i64> rbase(nseg + 1, 0);
  for (i64 s = 0; s < nseg; ++s) rbase[s + 1] = rbase[s] + counts[s];
  const i64 N = rbase[nseg];
  if (!N || fan <= 0) return;
  const i64 step = std::max<i64>(1, ((i64)1 << 25) / fan);
  std::vector<u64> hs;
  for (i64 q0 = 0; q0 < N; q0 += step) {
    const i64 q1 = std::min(N, q0 + step), nq = q1 - q0;
    i64* rows = g_rows.get((size_t)(nq * fan));
    hs.resize(nq);
    pfor(nq, [&](i64 lo, i64 hi, int) {
      i64 s = (i64)(std::upper_bound(rbase.begin(), rbase.end(), q0 + lo) - rbase.begin()) - 1;
      for (i64 i = lo; i < hi; ++i) {
        while (q0 + i >= rbase[s + 1]) ++s;
        i64* r = rows + i * fan;
        const i64* sl = slot_ptrs[s] + (q0 + i - rbase[s]) * fan;
        for (i64 j = 0; j < fan; ++j) r[j] = slot_phys[sl[j]];
        std::sort(r, r + fan);
        const bool contig = r[fan - 1] - r[0] == fan - 1 &&
                            std::adjacent_find(r, r + fan, [](i64 a, i64 b) { return b != a + 1; }) ==
                                r + fan;
        contig_start[q0 + i] = contig ? r[0] : -1;
        if (!contig) hs[i] = row_hash(r, fan);
      }
    }, std::max<i64>(1, (1 << 14) / fan));
    i64 ncontig = 0;
    for (i64 i = 0; i < nq; ++i) ncontig += contig_start[q0 + i] >= 0;
    const i64 need = (i64)G.first_id.size() + nq - ncontig;
    if (need > G.cap) {  // rehash into a larger table
      G.cap = std::max<i64>(2 * G.cap, need);
      G.heads.init(G.cap);
      for (i64 gi = 0; gi < (i64)G.first_id.size(); ++gi) {
        i64& hd = G.heads.at(G.hash[gi]);
        G.next[gi] = hd;
        hd = gi;
      }
    }
    i64 s = (i64)(std::upper_bound(rbase.begin(), rbase.end(), q0) - rbase.begin()) - 1;
    for (i64 i = 0; i < nq; ++i) {
      while (q0 + i >= rbase[s + 1]) ++s;
      if (contig_start[q0 + i] >= 0) continue;
      const i64* r = rows + i * fan;
      i64& hd = G.heads.at(hs[i]);
      bool found = false;
      for (i64 c = hd; c >= 0; c = G.next[c])
        if (G.off[c + 1] - G.off[c] == fan &&
            std::memcmp(G.members.data() + G.off[c], r, sizeof(i64) * fan) == 0) {
          found = true;
          break;
        }
      if (found) continue;
      G.first_id.push_back(id0s[s] + (q0 + i - rbase[s]));
      G.hash.push_back(hs[i]);
      G.members.insert(G.members.end(), r, r + fan);
      G.off.push_back((i64)G.members.size());
      G.next.push_back(hd);
      hd = (i64)G.first_id.size() - 1;
    }
  }
}

i64 pcc_rows_count(void* h, i64* n_members) {
  const RowGroups& G = *static_cast<RowGroups*>(h);
  *n_members = (i64)G.members.size();
  return (i64)G.first_id.size();
}

void pcc_rows_get(void* h, i64* first_id, i64* off, i64* members) {
  const RowGroups& G = *static_cast<RowGroups*>(h);
  std::copy(G.first_id.begin(), G.first_id.end(), first_id);
  std::copy(G.off.begin(), G.off.end(), off);
  std::copy(G.members.begin(), G.members.end(), members);
}

// claim[group_idx[e]] = group of e; 1 if a position is claimed by two groups
int pcc_claim_groups(i64 ngroups, const i64* group_off, const i64* group_idx, i64* claim) {
  std::atomic<int> bad{0};
  pfor(ngroups, [&](i64 lo, i64 hi, int) {
    for (i64 gi = lo; gi < hi; ++gi)
      for (i64 e = group_off[gi]; e < group_off[gi + 1]; ++e) {
        i64 expect = -1;
        if (!__atomic_compare_exchange_n(&claim[group_idx[e]], &expect, gi, false,
                                         __ATOMIC_RELAXED, __ATOMIC_RELAXED) &&
            expect != gi)
          bad.store(1, std::memory_order_relaxed);
      }
  }, 1 << 6);
  return bad.load();
}

// pcc_sum_groups over several segments (segment s: counts[s] rows of fan
// fans[s]); dst: one group_idx offset per row, concatenated.
int pcc_sum_groups_multi(i64 nseg, const i64* counts, const i64* fans, const i64* const* slot_ptrs,
                         const i64* slot_phys, u64* bits, const i64* dst, i64* group_idx) {
  std::vector<i64> rbase(nseg + 1, 0);
  i64 E = 0;
  for (i64 s = 0; s < nseg; ++s) rbase[s + 1] = rbase[s] + counts[s], E += counts[s] * fans[s];
  const i64 N = rbase[nseg];
  std::atomic<int> bad{0};
  pfor(N, [&](i64 lo, i64 hi, int) {
    i64 s = (i64)(std::upper_bound(rbase.begin(), rbase.end(), lo) - rbase.begin()) - 1;
    for (i64 q = lo; q < hi; ++q) {
      if (bad.load(std::memory_order_relaxed)) return;  // the general path takes over
      while (q >= rbase[s + 1]) ++s;
      const i64 fan = fans[s];
      i64* out = group_idx + dst[q];
      const i64* sl = slot_ptrs[s] + (q - rbase[s]) * fan;
      bool sorted = true;
      for (i64 j = 0; j < fan; ++j) {
        const i64 p = slot_phys[sl[j]];
        out[j] = p;
        if (j && p < out[j - 1]) sorted = false;
        const u64 bit = 1ull << ((u64)p & 63);
        if (__atomic_fetch_or(&bits[(u64)p >> 6], bit, __ATOMIC_RELAXED) & bit)
          bad.store(1, std::memory_order_relaxed);
      }
      if (!sorted) std::sort(out, out + fan);
    }
  }, std::max<i64>(1, (1 << 14) / std::max<i64>(1, N ? E / N : 1)));
  return bad.load();
}

// Depths (build.py:103-110) of segments given in dependency order: inputs 0,
// else 1 + the max child depth.  kinds[s] = 0 marks an input segment.
void pcc_depths(i64 nseg, const i64* starts, const i64* counts, const i64* fans,
                const int8_t* kinds, const i64* const* child_ptrs, const i64* strides,
                i64* depth) {
  for (i64 s = 0; s < nseg; ++s) {
    if (kinds[s] == 0) {
      std::fill(depth + starts[s], depth + starts[s] + counts[s], (i64)0);
      continue;
    }
    const i64 f = fans[s], st = strides[s];
    if (st == 0) {  // broadcast rows: one child list for the whole segment
      i64 m = -1;
      for (i64 j = 0; j < f; ++j) m = std::max(m, depth[child_ptrs[s][j]]);
      std::fill(depth + starts[s], depth + starts[s] + counts[s], m + 1);
      continue;
    }
    auto body = [&](i64 lo, i64 hi, int) {
      for (i64 i = lo; i < hi; ++i) {
        const i64* c = child_ptrs[s] + i * st;
        i64 m = -1;
        for (i64 j = 0; j < f; ++j) m = std::max(m, depth[c[j]]);
        depth[starts[s] + i] = m + 1;
      }
    };
    if (counts[s] * f >= (1 << 16))
      pfor(counts[s], body, std::max<i64>(1, (1 << 14) / std::max<i64>(f, 1)));
    else
      body(0, counts[s], 0);
  }
}

// graph_hash records of several segments, concatenated in order (see
// pcc_hash_records; a / b / c are var / ncat / slot for inputs, children /
// slots for sums, children for products; a_stride / b_stride: row strides in
// elements, 0 for broadcast rows).
void pcc_hash_records_multi(i64 nseg, const int8_t* kinds, const i64* counts, const i64* fans,
                            const i64* const* a, const i64* a_stride, const i64* const* b,
                            const i64* b_stride, const i64* const* c, uint8_t* out) {
  std::vector<i64> obase(nseg + 1, 0);
  for (i64 s = 0; s < nseg; ++s) {
    const i64 f = std::max<i64>(fans[s], 1);
    const i64 rec = kinds[s] == 0 ? 25 : (kinds[s] == 1 ? 1 + 8 * f : 1 + 16 * f);
    obase[s + 1] = obase[s] + rec * counts[s];
  }
  pfor(nseg, [&](i64 lo, i64 hi, int) {
    for (i64 s = lo; s < hi; ++s) {
      const i64 f = std::max<i64>(fans[s], 1);
      uint8_t* o = out + obase[s];
      for (i64 i = 0; i < counts[s]; ++i) {
        if (kinds[s] == 0) {
          *o++ = 'I';
          const i64 v[3] = {a[s][i], b[s][i], c[s][i]};
          std::memcpy(o, v, 24);
          o += 24;
        } else if (kinds[s] == 1) {
          *o++ = 'P';
          std::memcpy(o, a[s] + i * a_stride[s], 8 * f);
          o += 8 * f;
        } else {
          *o++ = 'S';
          std::memcpy(o, a[s] + i * a_stride[s], 8 * f);
          std::memcpy(o + 8 * f, b[s] + i * b_stride[s], 8 * f);
          o += 16 * f;
        }
      }
    }
  }, 64);
}

// Run-length encoding of the simplex-group table (runtime/plan.py
// group_runs): maximal runs of consecutive theta indices inside each group.
// Pass 1 (rs == null): runs per group into run_off[g + 1]; pass 2: run
// starts / lengths at the exclusive prefix run_off.
void pcc_group_runs(i64 ngroups, const i64* go, const i64* gi, i64* run_off, i64* rs, i64* rl) {
  pfor(ngroups, [&](i64 lo, i64 hi, int) {
    for (i64 g = lo; g < hi; ++g) {
      const i64 a = go[g], b = go[g + 1];
      if (!rs) {
        i64 n = a < b;
        for (i64 i = a + 1; i < b; ++i) n += gi[i] != gi[i - 1] + 1;
        run_off[g + 1] = n;
        continue;
      }
      i64 r = run_off[g];
      for (i64 i = a; i < b; ++i) {
        if (i == a || gi[i] != gi[i - 1] + 1) {
          rs[r] = gi[i];
          rl[r++] = 1;
        } else {
          ++rl[r - 1];
        }
      }
    }
  }, 1 << 10);
}

// min / max of an int64 array (the plan's int32 range check)
void pcc_minmax(const i64* a, i64 n, i64* out) {
  std::vector<i64> mn(nthreads(), INT64_MAX), mx(nthreads(), INT64_MIN);
  pfor(n, [&](i64 lo, i64 hi, int t) {
    i64 x = INT64_MAX, y = INT64_MIN;
    for (i64 i = lo; i < hi; ++i) x = std::min(x, a[i]), y = std::max(y, a[i]);
    mn[t] = std::min(mn[t], x), mx[t] = std::max(mx[t], y);
  }, 1 << 20);
  out[0] = *std::min_element(mn.begin(), mn.end());
  out[1] = *std::max_element(mx.begin(), mx.end());
}

// dst = int32(src), checked beforehand
void pcc_narrow_i32(const i64* src, i64 n, int32_t* dst) {
  pfor(n, [&](i64 lo, i64 hi, int) {
    for (i64 i = lo; i < hi; ++i) dst[i] = (int32_t)src[i];
  }, 1 << 20);
}

}  // extern "C"
