// Host-side (CPU) bookkeeping of the hot path, native so that the per-call
// overhead of Network.launch / contract stays in microseconds:
//   tnb_zero_flux_blocks  <- _zero_flux_combos      (pkg/src/tnkit/unitensor.py:31-45)
//   tnb_optimal_order     <- find_optimal_order     (pkg/src/tnkit/contract.py:271-343)
// Both are integer/text algorithms and must reproduce the reference bit for bit
// (enumeration order; DP cost and tie-break on the rendered order string).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tnb.h"

namespace tnb {
int fail(int code, const std::string& msg);
}

extern "C" int tnb_zero_flux_blocks(int nbonds, int nsyms, const int32_t* nsec, const int32_t* btype,
                                    const int64_t* charges, const int32_t* sym_n, int64_t max_out,
                                    int32_t* out_qn, int64_t* count) {
  if (nbonds < 1 || nbonds > TNB_MAX_RANK || nsyms < 1 || !nsec || !btype || !charges || !sym_n || !count)
    return tnb::fail(TNB_EINVAL, "zero_flux_blocks: bad arguments");
  std::vector<int64_t> off(nbonds + 1, 0);
  for (int b = 0; b < nbonds; ++b) {
    if (nsec[b] < 1) return tnb::fail(TNB_EINVAL, "zero_flux_blocks: bond without sectors");
    off[b + 1] = off[b] + nsec[b];
  }
  // per-bond signed contribution of each sector: IN adds q, OUT adds reverse(q)
  // (symmetry.py:49-66: U1 negation, Zn (-q) mod n; combine is + (mod n))
  std::vector<int64_t> contrib((size_t)off[nbonds] * nsyms);
  for (int b = 0; b < nbonds; ++b)
    for (int s = 0; s < nsec[b]; ++s)
      for (int y = 0; y < nsyms; ++y) {
        int64_t q = charges[(off[b] + s) * nsyms + y];
        if (btype[b] < 0) q = -q;
        if (sym_n[y] > 0) q = ((q % sym_n[y]) + sym_n[y]) % sym_n[y];
        contrib[(off[b] + s) * nsyms + y] = q;
      }
  // row-major product enumeration (itertools.product, first bond outermost) with
  // a running flux per prefix so each step costs O(nsyms)
  std::vector<int32_t> idx(nbonds, 0);
  std::vector<int64_t> flux((size_t)(nbonds + 1) * nsyms, 0);
  auto recompute_from = [&](int b0) {
    for (int b = b0; b < nbonds; ++b)
      for (int y = 0; y < nsyms; ++y) {
        int64_t v = flux[(size_t)b * nsyms + y] + contrib[(off[b] + idx[b]) * nsyms + y];
        if (sym_n[y] > 0) v %= sym_n[y];
        flux[(size_t)(b + 1) * nsyms + y] = v;
      }
  };
  recompute_from(0);
  int64_t found = 0;
  while (true) {
    bool zero = true;
    for (int y = 0; y < nsyms; ++y) zero = zero && (flux[(size_t)nbonds * nsyms + y] == 0);
    if (zero) {
      if (found < max_out && out_qn)
        for (int b = 0; b < nbonds; ++b) out_qn[found * nbonds + b] = idx[b];
      ++found;
    }
    int b = nbonds - 1;
    while (b >= 0 && idx[b] + 1 == nsec[b]) {
      idx[b] = 0;
      --b;
    }
    if (b < 0) break;
    ++idx[b];
    recompute_from(b);
  }
  *count = found;
  return TNB_OK;
}

namespace {

typedef unsigned __int128 u128;

std::string u128_str(u128 v) {
  if (v == 0) return "0";
  std::string s;
  while (v) {
    s.insert(s.begin(), char('0' + (int)(v % 10)));
    v /= 10;
  }
  return s;
}

struct Entry {
  bool set = false;
  u128 cost = 0;
  std::string rendered;
};

}  // namespace

extern "C" int tnb_optimal_order(int n, const char* names, const int32_t* nlab, const int32_t* labels,
                                 const int64_t* dims, char* out, int64_t cap_out, char* cost_out) {
  if (n < 1 || n > 16 || !names || !nlab || !labels || !dims || !out)
    return tnb::fail(TNB_EINVAL, "optimal_order: bad arguments (1 <= n <= 16)");
  std::vector<std::string> nm(n);
  const char* p = names;
  for (int i = 0; i < n; ++i) {
    nm[i] = std::string(p);
    p += nm[i].size() + 1;
  }
  int nl = 0;
  std::vector<std::vector<int>> lab(n);
  {
    int64_t o = 0;
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < nlab[i]; ++j) {
        int l = labels[o + j];
        if (l < 0) return tnb::fail(TNB_EINVAL, "optimal_order: negative label id");
        lab[i].push_back(l);
        if (l + 1 > nl) nl = l + 1;
      }
      o += nlab[i];
    }
  }
  auto put = [&](const std::string& s, const std::string& c) -> int {
    if ((int64_t)s.size() + 1 > cap_out) return tnb::fail(TNB_EINVAL, "optimal_order: output buffer too small");
    memcpy(out, s.c_str(), s.size() + 1);
    if (cost_out) {
      std::string cc = c.substr(0, 63);
      memcpy(cost_out, cc.c_str(), cc.size() + 1);
    }
    return TNB_OK;
  };
  if (n == 1) return put(nm[0], "0");
  const int W = (nl + 63) / 64;
  const int full = (1 << n) - 1;
  // free labels per subset: occurring exactly once
  std::vector<uint64_t> freebits((size_t)(full + 1) * W, 0);
  {
    std::vector<int> cnt(nl, 0);
    for (int mask = 1; mask <= full; ++mask) {
      std::fill(cnt.begin(), cnt.end(), 0);
      for (int i = 0; i < n; ++i)
        if (mask >> i & 1)
          for (int l : lab[i]) cnt[l]++;
      uint64_t* f = &freebits[(size_t)mask * W];
      for (int l = 0; l < nl; ++l)
        if (cnt[l] == 1) f[l >> 6] |= (1ull << (l & 63));
    }
  }
  bool overflow = false;
  auto pair_cost = [&](int m1, int m2) -> u128 {
    u128 c = 1;
    const uint64_t* f1 = &freebits[(size_t)m1 * W];
    const uint64_t* f2 = &freebits[(size_t)m2 * W];
    for (int w = 0; w < W; ++w) {
      uint64_t u = f1[w] | f2[w];
      while (u) {
        int b = __builtin_ctzll(u);
        u &= u - 1;
        u128 dmul = (u128)(uint64_t)dims[w * 64 + b];
        if (dmul != 0 && c > (~(u128)0) / dmul) overflow = true;
        c *= dmul;
      }
    }
    return c;
  };
  u128 cap = 0;
  bool first = true;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      u128 c = pair_cost(1 << i, 1 << j);
      if (first || c < cap) cap = c;
      first = false;
    }
  if (cap < 1) cap = 1;
  // masks by popcount (stable: ascending value within a popcount), popcount >= 2
  std::vector<int> order;
  for (int pc = 2; pc <= n; ++pc)
    for (int m = 1; m <= full; ++m)
      if (__builtin_popcount(m) == pc) order.push_back(m);
  std::vector<Entry> best(full + 1);
  while (true) {
    for (auto& e : best) e.set = false;
    for (int i = 0; i < n; ++i) {
      best[1 << i].set = true;
      best[1 << i].cost = 0;
      best[1 << i].rendered = nm[i];
    }
    for (int mask : order) {
      int sub = (mask - 1) & mask;
      while (sub) {
        int rest = mask ^ sub;
        int s1 = sub < rest ? sub : rest;
        int s2 = sub < rest ? rest : sub;
        sub = (sub - 1) & mask;
        if (!best[s1].set || !best[s2].set) continue;
        u128 pc = pair_cost(s1, s2);
        u128 cost = best[s1].cost + best[s2].cost + pc;
        if (cost < pc) overflow = true;
        if (cost > cap) continue;
        const std::string& r1 = best[s1].rendered;
        const std::string& r2 = best[s2].rendered;
        std::string rendered = (r1 <= r2) ? ("(" + r1 + "," + r2 + ")") : ("(" + r2 + "," + r1 + ")");
        Entry& cur = best[mask];
        if (!cur.set || cost < cur.cost || (cost == cur.cost && rendered < cur.rendered)) {
          cur.set = true;
          cur.cost = cost;
          cur.rendered = std::move(rendered);
        }
      }
    }
    if (overflow) return tnb::fail(TNB_EUNSUP, "optimal_order: cost exceeds 128 bits");
    if (best[full].set) return put(best[full].rendered, u128_str(best[full].cost));
    if (cap > (~(u128)0) / 2) return tnb::fail(TNB_EUNSUP, "optimal_order: cost cap overflow");
    cap *= 2;
  }
}
