// Device plan encoder; see device_plan.hpp and dev_plan.h for the layout.
#include "device_plan.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <cstring>
#include <string>

#include "model.hpp"

namespace pbn_b200 {

namespace {

std::uint32_t entry_log2(std::uint32_t members) {
  return members <= 8 ? 0 : members <= 16 ? 1 : members <= 32 ? 2 : 3;
}

std::size_t align16(std::size_t x) { return (x + 15) & ~std::size_t(15); }

template <class T>
void put(std::vector<std::uint8_t>& blob, std::size_t off, const std::vector<T>& v) {
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), sizeof(T) * v.size());
}

}  // namespace

// Exact restatement of the reference's combined-function choice for one
// draw r53 (engine.hpp:285-290): u = r53 * 2^-53, x = u * N in IEEE double
// (this file is compiled without FP contraction), c = trunc(x) clamped to
// N-1, pick c iff x - c < cut[c].
std::uint32_t alias53_cell(std::uint64_t r53, std::uint32_t n) {
  const double x = static_cast<double>(r53) * 0x1.0p-53 * static_cast<double>(n);
  const std::uint32_t c = static_cast<std::uint32_t>(x);
  return c >= n ? n - 1 : c;
}
double alias53_frac(std::uint64_t r53, std::uint32_t n) {
  const double x = static_cast<double>(r53) * 0x1.0p-53 * static_cast<double>(n);
  const std::uint32_t c = alias53_cell(r53, n);
  return x - static_cast<double>(c);
}

// For each cell c, the smallest r53 of the cell whose fraction reaches cut[c]
// (the cell's end when none does): within a cell the fraction is monotone in
// r53, so pick(r53) == c  <=>  r53 < C[c]. Binary searches over the exact rule.
std::vector<std::uint64_t> alias53_cut_points(const double* cut, std::uint32_t n) {
  auto first = [&](std::uint64_t lo, std::uint64_t hi, auto pred) {  // min r in [lo,hi) with pred, else hi
    while (lo < hi) {
      const std::uint64_t mid = lo + (hi - lo) / 2;
      if (pred(mid))
        hi = mid;
      else
        lo = mid + 1;
    }
    return lo;
  };
  const std::uint64_t end = 1ull << 53;
  std::vector<std::uint64_t> start(n + 1, end), C(n, end);
  start[0] = 0;
  for (std::uint32_t c = 1; c < n; ++c)
    start[c] = first(start[c - 1], end, [&](std::uint64_t r) { return alias53_cell(r, n) >= c; });
  for (std::uint32_t c = 0; c < n; ++c)
    C[c] = first(start[c], start[c + 1],
                 [&](std::uint64_t r) { return !(alias53_frac(r, n) < cut[c]); });
  return C;
}

std::vector<std::uint32_t> alias53_records(const double* cut, const std::uint32_t* alias,
                                           std::uint32_t n) {
  const std::vector<std::uint64_t> C = alias53_cut_points(cut, n);
  std::vector<std::uint32_t> rec(2 * static_cast<std::size_t>(n));
  for (std::uint32_t c = 0; c < n; ++c) {
    rec[2 * c] = alias[c];
    rec[2 * c + 1] = static_cast<std::uint32_t>(std::min<std::uint64_t>(C[c], (1ull << 53) - 1) >> 21);
  }
  return rec;
}

std::uint32_t alias53_pick_int(const std::uint32_t* rec, std::uint32_t n, std::uint32_t hi,
                               bool& rare) {
  const std::uint64_t P = static_cast<std::uint64_t>(hi) * n;
  const std::uint32_t e = static_cast<std::uint32_t>(P >> 32);
  const std::uint32_t chi = rec[2 * e + 1];
  rare = rare || static_cast<std::uint32_t>(P) > ~n || hi == chi;
  return hi < chi ? e : rec[2 * e];
}

void philox_round_keys(std::uint64_t seed, std::uint32_t rk0[10], std::uint32_t rk1[10]) {
  std::uint32_t k0 = static_cast<std::uint32_t>(seed), k1 = static_cast<std::uint32_t>(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    rk0[r] = k0;
    rk1[r] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

dev_predicate compile_dev_predicate(const std::uint32_t* bits, const std::uint8_t* vals,
                                    std::uint32_t n, std::uint32_t n_kept) {
  dev_predicate p{};
  bool contradiction = false;
  for (std::uint32_t i = 0; i < n; ++i) {
    if (bits[i] >= n_kept) throw model_error("predicate references a bit outside the state");
    const std::uint32_t w = bits[i] >> 5, m = 1u << (bits[i] & 31);
    std::uint32_t j = 0;
    while (j < p.n && p.w[j] != w) ++j;
    if (j == p.n) {
      if (p.n == kMaxPredWords) throw resource_error("predicate spans too many state words");
      p.w[j] = w;
      p.mask[j] = 0;
      p.want[j] = 0;
      ++p.n;
    }
    const std::uint32_t want = vals[i] ? m : 0u;
    if ((p.mask[j] & m) && (p.want[j] & m) != want) contradiction = true;
    p.mask[j] |= m;
    p.want[j] |= want;
  }
  if (contradiction) {  // "x == 0 and x == 1": never satisfied
    p = dev_predicate{};
    p.n = 1;
    p.w[0] = 0;
    p.mask[0] = 0;
    p.want[0] = 1;
  }
  return p;
}

encoded_plan encode_plan(const pbn_plan_view& v) {
  const std::uint32_t n = v.n_kept;
  if (n == 0) throw model_error("empty plan");
  if (n >= 65535) throw resource_error("device engine supports at most 65534 kept nodes");
  if (v.pert_k < 1 || v.pert_k > 24) throw resource_error("perturbation width must be in [1,24]");
  if (v.pert_size != (1u << v.pert_k)) throw model_error("perturbation table size != 2^k");

  encoded_plan ep;
  dev_plan_header& h = ep.h;
  h.n_kept = n;
  h.sw32 = 2 * (n / 64 + 1);
  h.g = v.pert_groups;
  h.k = v.pert_k;
  h.last_mask = static_cast<std::uint32_t>(v.pert_mask);
  h.n_groups = v.n_groups;
  h.rg_ok = h.sw32 <= 32 ? 1u : 0u;
  if (v.pert_mode > 1) throw model_error("unknown perturbation mode");
  // The grouped stepper always makes the leaf draw once no kept node flipped
  // (engine.hpp:268, also when t == 1); a grouped view without it would shift
  // every function-selection draw by one. Only Method_old (pert_mode 1) has
  // no leaf draw (engine.hpp:193-201).
  if (v.pert_mode == 0 && !v.has_leaf)
    throw std::invalid_argument(
        "plan view: grouped plans (pert_mode 0) need has_leaf = 1 (engine.hpp:268)");
  h.pert_mode = v.pert_mode;
  h.has_leaf = v.has_leaf ? 1u : 0u;
  if (v.pert_mode == 1) {
    if (!(v.pert_p > 0.0 && v.pert_p < 1.0)) throw model_error("perturbation rate must be in (0,1)");
    if (v.pert_k != 1) throw model_error("Bernoulli perturbation needs k = 1");
    // u < p  <=>  r < ceil(p * 2^bits)  (p * 2^bits is exact)
    h.pthr53 = static_cast<std::uint64_t>(std::ceil(std::ldexp(v.pert_p, 53))) << 11;
    h.pthr32 = static_cast<std::uint64_t>(std::ceil(std::ldexp(v.pert_p, 32)));
  }
  // leaf perturbation iff u > t  <=>  r > floor(t * 2^bits) (t*2^bits is exact)
  const double t53 = std::floor(std::ldexp(v.t, 53));
  h.leaf_thr53 = t53 >= 9007199254740992.0 ? ~0ull : (static_cast<std::uint64_t>(t53) << 11) | 0x7FFu;
  const double t32 = std::floor(std::ldexp(v.t, 32));
  h.leaf_never = v.t >= 1.0 ? 1u : 0u;
  h.leaf_thr32 = t32 >= 4294967295.0 ? 0xFFFFFFFFu : static_cast<std::uint32_t>(t32);

  // ---- perturbation cells
  const std::uint32_t k = v.pert_k;
  std::vector<std::uint64_t> pert53(v.pert_size);
  std::vector<std::uint32_t> pert32(v.pert_size);
  for (std::uint32_t c = 0; c < v.pert_size; ++c) {
    const double cut = v.pert_cut[c];
    const std::uint32_t al = v.pert_alias[c];
    {
      const double T = std::ceil(std::ldexp(cut, 53 - static_cast<int>(k)));
      const double full = std::ldexp(1.0, 53 - static_cast<int>(k));
      std::uint64_t tt = 0, aa = c;
      if (T < full) {
        tt = static_cast<std::uint64_t>(T);
        aa = al;
      }
      // raw-word form: compared against the draw's 64-bit word pair (r53 << 11 | noise)
      pert53[c] = (tt << 11) | (aa << (64 - k));
    }
    {
      const double T = std::ceil(std::ldexp(cut, 32 - static_cast<int>(k)));
      const double full = std::ldexp(1.0, 32 - static_cast<int>(k));
      std::uint32_t tt = 0, aa = c;
      if (T < full) {
        tt = static_cast<std::uint32_t>(T);
        aa = al;
      }
      pert32[c] = tt | (aa << (32 - k));
    }
  }

  // ---- groups, functions, gather records, tables
  std::vector<std::uint32_t> groups(4 * static_cast<std::size_t>(v.n_groups));
  std::vector<std::uint32_t> fns(4 * static_cast<std::size_t>(v.n_fns));
  std::vector<std::uint16_t> grec;
  std::vector<std::uint8_t> tables;
  std::vector<std::uint32_t> fn_members(v.n_fns, 0);
  h.max_alias = 0;
  h.n_alias_groups = 0;
  bool plain_seen = false;
  for (std::uint32_t gi = 0; gi < v.n_groups; ++gi) {
    const std::uint32_t off = v.grp_offset[gi];
    std::uint32_t members;
    if (v.grp_members) {
      members = v.grp_members[gi];
      if (members == 0 || members > 64 || off + members > n)
        throw model_error("group member count out of range");
    } else {
      const std::uint32_t end = gi + 1 < v.n_groups ? v.grp_offset[gi + 1] : n;
      if (end <= off || end - off > 64) throw model_error("group member count out of range");
      members = end - off;
    }
    const std::uint32_t asz = v.grp_alias_size[gi];
    if (asz >= (1u << 23)) throw resource_error("group alias table too large for the device");
    if (asz == 1) throw model_error("alias table of one cell");
    if (asz) {
      if (plain_seen) throw model_error("alias groups must precede single-function groups");
      ++h.n_alias_groups;
    } else {
      plain_seen = true;
    }
    h.max_alias = std::max(h.max_alias, asz);
    groups[4 * gi + 0] = off;
    groups[4 * gi + 1] = v.grp_fn_begin[gi];
    groups[4 * gi + 2] = v.grp_alias_begin[gi];
    groups[4 * gi + 3] = asz | ((members - 1) << 24);
    const std::uint32_t nf = asz ? asz : 1;
    for (std::uint32_t j = 0; j < nf; ++j) {
      const std::uint32_t f = v.grp_fn_begin[gi] + j;
      if (f >= v.n_fns) throw model_error("function index out of range");
      fn_members[f] = members;
    }
  }
  // leading single-node alias groups whose functions all have inline tables
  h.n_single_alias = 0;
  h.single_gc5 = 0;
  std::vector<std::uint32_t> arec;
  for (std::uint32_t gi = 0; gi < h.n_alias_groups; ++gi) {
    const std::uint32_t members = (groups[4 * gi + 3] >> 24) + 1;
    if (members != 1 || groups[4 * gi] != gi) break;
    if (v.grp_fn_begin[gi] != v.grp_alias_begin[gi] || v.grp_alias_size[gi] > 255 ||
        v.grp_fn_begin[gi] >= (1u << 24))
      break;
    bool ok = true, gc5 = false;
    for (std::uint32_t j = 0; j < v.grp_alias_size[gi]; ++j) {
      ok = ok && v.fn_gather_count[v.grp_fn_begin[gi] + j] <= 5;
      gc5 = gc5 || v.fn_gather_count[v.grp_fn_begin[gi] + j] == 5;
    }
    if (!ok) break;
    if (gc5) h.single_gc5 = 1;
    h.n_single_alias = gi + 1;
    arec.push_back(v.grp_fn_begin[gi] | (v.grp_alias_size[gi] << 24));
  }
  // single-node rounds end on a 32-group boundary unless they cover the whole
  // alias region, so the general path never sees a group below A1
  if (h.n_single_alias < h.n_alias_groups) {
    h.n_single_alias &= ~31u;
    arec.resize(h.n_single_alias);
  }
  if (arec.empty()) arec.push_back(0);
  auto record = [&](std::uint32_t f, std::uint32_t b) -> std::uint16_t {
    const std::uint32_t gc = v.fn_gather_count[f];
    const std::uint32_t pos = b < gc ? v.fn_gather[v.fn_gather_begin[f] + b] : n;
    if (pos > n) throw model_error("gather position out of range");
    return static_cast<std::uint16_t>(((pos >> 5) << 5) | (((pos & 31) - b) & 31));
  };
  for (std::uint32_t f = 0; f < v.n_fns; ++f) {
    const std::uint32_t gc = v.fn_gather_count[f];
    if (gc > 30) throw resource_error("gather list longer than 30 bits");
    if (v.fn_gather_begin[f] + gc > v.n_gather) throw model_error("gather range out of bounds");
    const std::uint32_t members = fn_members[f] ? fn_members[f] : 1;
    const std::uint32_t el2 = entry_log2(members);
    // table
    std::size_t tb = tables.size();
    const std::size_t align = el2 == 3 ? 8 : 4;
    tb = (tb + align - 1) & ~(align - 1);
    const std::uint64_t len = 1ull << gc;
    const std::size_t bytes = static_cast<std::size_t>(len) << el2;
    tables.resize(((tb + bytes) + 3) & ~std::size_t(3), 0);
    if (v.fn_table_begin[f] + len > v.n_table) throw model_error("table range out of bounds");
    for (std::uint64_t e = 0; e < len; ++e) {
      const std::uint64_t out = v.fn_tables[v.fn_table_begin[f] + e];
      std::memcpy(tables.data() + tb + (e << el2), &out, std::size_t(1) << el2);  // little endian
    }
    if (tb > 0xFFFFFFFFull) throw resource_error("function tables exceed 4 GiB");
    // records 0..3 inline, the rest in grec (4-aligned quads)
    std::uint32_t xq = 0;
    if (gc > 4) {
      while (grec.size() % 4) grec.push_back(0);
      xq = static_cast<std::uint32_t>(grec.size() / 4);
      if (xq >= (1u << 24)) throw resource_error("too many gather records");
      const std::uint32_t slots = (gc + 3) & ~3u;
      for (std::uint32_t b = 4; b < slots; ++b) grec.push_back(record(f, b));
    }
    // tables of at most 32 bits live inline in the record (entry e at bits
    // [e*members, (e+1)*members))
    std::uint32_t inl = 0, word = static_cast<std::uint32_t>(tb);
    if (static_cast<std::uint64_t>(members) << gc <= 32) {
      inl = 1;
      word = 0;
      for (std::uint64_t e = 0; e < len; ++e)
        word |= static_cast<std::uint32_t>(v.fn_tables[v.fn_table_begin[f] + e]) << (e * members);
    }
    fns[4 * f + 0] = word;
    fns[4 * f + 1] = gc | (el2 << 5) | (inl << 7) | (xq << 8);
    fns[4 * f + 2] = record(f, 0) | (static_cast<std::uint32_t>(record(f, 1)) << 16);
    fns[4 * f + 3] = record(f, 2) | (static_cast<std::uint32_t>(record(f, 3)) << 16);
  }
  if (grec.empty()) grec.assign(4, 0);

  // ---- group alias cells
  std::vector<double> acut(v.alias_cut, v.alias_cut + v.n_alias);
  std::vector<std::uint32_t> aidx(v.alias_idx, v.alias_idx + v.n_alias);
  // acell[c] = {U53: alias, hi32 of the cut point (dev_plan.h); U32: threshold, alias}
  std::vector<std::uint32_t> acell(4 * v.n_alias, 0);
  h.u32_ok = h.max_alias <= (1u << 21) ? 1u : 0u;
  for (std::uint32_t gi = 0; gi < v.n_groups; ++gi) {
    const std::uint32_t asz = v.grp_alias_size[gi], ab = v.grp_alias_begin[gi];
    if (static_cast<std::uint64_t>(ab) + asz > v.n_alias) throw model_error("alias range out of bounds");
    for (std::uint32_t c = 0; c < asz; ++c) {
      const double T = std::ceil(std::ldexp(v.alias_cut[ab + c], 32));
      std::uint32_t tt = 0, aa = c;
      if (T < 4294967296.0) {
        tt = static_cast<std::uint32_t>(T);
        aa = v.alias_idx[ab + c];
      }
      acell[4 * (ab + c) + 2] = tt;
      acell[4 * (ab + c) + 3] = aa;
    }
    if (asz == 0) continue;
    if (asz > kA53MaxCells) {
      groups[4 * gi + 3] |= kGroupExactAlias;  // this group always takes the FP64 path
      continue;
    }
    const std::vector<std::uint32_t> rec = alias53_records(v.alias_cut + ab, v.alias_idx + ab, asz);
    for (std::uint32_t c = 0; c < asz; ++c) {
      acell[4 * (ab + c) + 0] = rec[2 * c];
      acell[4 * (ab + c) + 1] = rec[2 * c + 1];
    }
  }

  // compact records of the leading single-node groups for the register gather
  // (n' <= 1023, at most 4 parents), in a bank-column layout (dev_plan.h scol):
  // group j owns 8-byte slot j % 16 of 128-byte rows, so the 16 lanes of each
  // half-warp of a round read 16 distinct bank pairs. Per group, N rows each of
  // U53 cells {alias, hi32(C)}, U32 cells {threshold, alias} and function
  // records {rec0 | rec1 << 10 | rec2 << 20, rec3 | table << 16} (10-bit
  // records word << 5 | rotation); arec4[j] = {byte offset of the U53 cells,
  // byte offset of the function records, N, ~N}.
  h.single_compact = h.rg_ok && h.n_single_alias >= 32 && !h.single_gc5 ? 1u : 0u;
  std::vector<std::uint32_t> scol, arec4;
  std::vector<std::uint32_t> scol_row0;  // per single group: first row
  if (h.single_compact) {
    std::uint32_t rows[kScolSlots] = {};
    scol_row0.resize(h.n_single_alias);
    for (std::uint32_t gi = 0; gi < h.n_single_alias; ++gi) {
      scol_row0[gi] = rows[gi % kScolSlots];
      rows[gi % kScolSlots] += 3 * v.grp_alias_size[gi];
    }
    const std::uint32_t nrows = *std::max_element(rows, rows + kScolSlots);
    scol.assign(static_cast<std::size_t>(nrows) * 2 * kScolSlots, 0);
    auto put2 = [&](std::uint32_t row, std::uint32_t slot, std::uint32_t x, std::uint32_t y) {
      const std::size_t w = (static_cast<std::size_t>(row) * kScolSlots + slot) * 2;
      scol[w] = x;
      scol[w + 1] = y;
    };
    for (std::uint32_t gi = 0; gi < h.n_single_alias; ++gi) {
      const std::uint32_t asz = v.grp_alias_size[gi], ab = v.grp_alias_begin[gi];
      const std::uint32_t slot = gi % kScolSlots, r0 = scol_row0[gi];
      for (std::uint32_t c = 0; c < asz; ++c) {
        put2(r0 + c, slot, acell[4 * (ab + c) + 0], acell[4 * (ab + c) + 1]);
        put2(r0 + asz + c, slot, acell[4 * (ab + c) + 2], acell[4 * (ab + c) + 3]);
        const std::uint32_t f = v.grp_fn_begin[gi] + c;
        const std::uint32_t gc = v.fn_gather_count[f];
        if (gc > 4 || fn_members[f] != 1) throw model_error("compact single-node record misuse");
        std::uint32_t rc[4];
        for (std::uint32_t b = 0; b < 4; ++b) rc[b] = record(f, b) & 0x3FFu;
        std::uint32_t table = 0;
        for (std::uint32_t e = 0; e < (1u << gc); ++e)
          table |= static_cast<std::uint32_t>(v.fn_tables[v.fn_table_begin[f] + e] & 1u) << e;
        put2(r0 + 2 * asz + c, slot, rc[0] | (rc[1] << 10) | (rc[2] << 20), rc[3] | (table << 16));
      }
    }
  }

  // Compact single-node records for networks too large for the register
  // gather (n' > 2047: the sub-warp kernel's shared-memory gather, GM 4;
  // dev_plan.h sgrp/sfn): sgrp[j] = the group's N <= 4 U53 cells, one word
  // each: hi32(C[c]) with the low 4 bits replaced by alias[c] << 2 (and N-1
  // in cell 0) — the kernel compares the high word's top 28 bits, a tie
  // being rare (redo); sfn[4j + c] = {1-bit inline table, records 0|1,
  // records 2|3, record 4 | gather count << 16} (16-bit records, as fns).
  h.single_compact_l = !h.single_compact && h.sw32 > 64 && h.n_single_alias >= 32 && n < 65536 ? 1u : 0u;
  for (std::uint32_t gi = 0; h.single_compact_l && gi < h.n_single_alias; ++gi)
    if (v.grp_alias_size[gi] > 4) h.single_compact_l = 0;
  std::vector<std::uint32_t> sgrp, sfn;
  if (h.single_compact_l) {
    const std::uint32_t A1 = h.n_single_alias;
    sgrp.assign(4 * static_cast<std::size_t>(A1), 0);
    sfn.assign(16 * static_cast<std::size_t>(A1), 0);
    for (std::uint32_t gi = 0; gi < A1; ++gi) {
      const std::uint32_t asz = v.grp_alias_size[gi], ab = v.grp_alias_begin[gi];
      for (std::uint32_t c = 0; c < asz; ++c) {
        const std::uint32_t al = acell[4 * (ab + c) + 0], hi = acell[4 * (ab + c) + 1];
        if (al >= asz) throw model_error("alias target out of range");
        sgrp[4 * gi + c] = (hi & ~0xFu) | (al << 2) | (c == 0 ? asz - 1 : 0u);
        const std::uint32_t f = v.grp_fn_begin[gi] + c;
        const std::uint32_t gc = v.fn_gather_count[f];
        if (gc > 5 || fn_members[f] != 1) throw model_error("compact single-node record misuse");
        std::uint32_t table = 0;
        for (std::uint32_t e = 0; e < (1u << gc); ++e)
          table |= static_cast<std::uint32_t>(v.fn_tables[v.fn_table_begin[f] + e] & 1u) << e;
        std::uint32_t* F = &sfn[16 * static_cast<std::size_t>(gi) + 4 * c];
        F[0] = table;
        F[1] = record(f, 0) | (static_cast<std::uint32_t>(record(f, 1)) << 16);
        F[2] = record(f, 2) | (static_cast<std::uint32_t>(record(f, 3)) << 16);
        F[3] = record(f, 4) | (gc << 16);
      }
    }
  }

  // With the compact records the single-node groups' fns/acell entries are
  // needed only by the fallback (non-compact) kernels: they move to an
  // unstaged tail (fns_s, acell_s) and the staged fns/acell start at the first
  // general group's entries (groups[].y/.z rebased).
  h.fn_base = 0;
  h.cell_base = 0;
  if (h.single_compact) {
    const std::uint32_t A1 = h.n_single_alias;
    std::uint32_t fb = v.n_fns, cb = static_cast<std::uint32_t>(v.n_alias);
    for (std::uint32_t gi = A1; gi < v.n_groups; ++gi) {
      fb = std::min(fb, v.grp_fn_begin[gi]);
      if (v.grp_alias_size[gi]) cb = std::min(cb, v.grp_alias_begin[gi]);
    }
    bool ok = true;
    for (std::uint32_t gi = 0; gi < A1; ++gi)
      ok = ok && v.grp_fn_begin[gi] + v.grp_alias_size[gi] <= fb &&
           v.grp_alias_begin[gi] + v.grp_alias_size[gi] <= cb;
    if (ok) {
      h.fn_base = fb;
      h.cell_base = cb;
      for (std::uint32_t gi = 0; gi < v.n_groups; ++gi) {
        groups[4 * gi + 1] = gi < A1 ? 0u : groups[4 * gi + 1] - fb;
        groups[4 * gi + 2] = gi < A1 || v.grp_alias_size[gi] == 0 ? 0u : groups[4 * gi + 2] - cb;
      }
    }
  }
  std::vector<std::uint32_t> fns_s(fns.begin(), fns.begin() + 4 * static_cast<std::size_t>(h.fn_base));
  std::vector<std::uint32_t> acell_s(acell.begin(), acell.begin() + 4 * static_cast<std::size_t>(h.cell_base));
  fns.erase(fns.begin(), fns.begin() + 4 * static_cast<std::size_t>(h.fn_base));
  acell.erase(acell.begin(), acell.begin() + 4 * static_cast<std::size_t>(h.cell_base));

  // ---- assemble
  std::size_t off = 0;
  auto section = [&](std::size_t bytes) {
    const std::size_t o = off;
    off = align16(off + bytes);
    return static_cast<std::uint32_t>(o);
  };
  // placement prefixes: [core | tables | pert32 | pert53] — a launch stages
  // the longest prefix that fits in shared memory and reads the rest via L1/L2
  h.off_sgrp = section(4 * sgrp.size());  // 0: staged by every GM 4 launch
  h.off_sfn = section(4 * sfn.size());
  h.off_groups = section(4 * groups.size());
  h.off_fns = section(4 * fns.size());
  h.off_grec = section(2 * grec.size());
  h.off_acell = section(4 * acell.size());
  h.off_arec = section(4 * arec.size());
  h.off_scol = section(4 * scol.size());
  h.off_arec4 = section(16 * static_cast<std::size_t>(h.single_compact ? h.n_single_alias : 0));
  h.core_bytes = static_cast<std::uint32_t>(off);
  h.off_tables = section(tables.size());
  h.table_bytes = static_cast<std::uint32_t>(off) - h.off_tables;
  h.off_pert32 = section(4 * pert32.size());
  h.off_pert53 = section(8 * pert53.size());
  h.blob_bytes = static_cast<std::uint32_t>(off);  // end of the stageable prefix
  // FP64 cut-offs for the rare exact path: read through L1/L2, never staged
  h.off_acut = section(8 * acut.size());
  h.off_aidx = section(4 * aidx.size());
  std::vector<std::uint32_t> pert53h(pert53.size());
  for (std::size_t c = 0; c < pert53.size(); ++c) pert53h[c] = static_cast<std::uint32_t>(pert53[c] >> 32);
  h.off_pert53h = section(4 * pert53h.size());
  if (h.fn_base || h.cell_base) {
    h.off_fns_s = section(4 * fns_s.size());
    h.off_acell_s = section(4 * acell_s.size());
  } else {  // nothing moved: the fallback paths read the staged arrays
    h.off_fns_s = h.off_fns;
    h.off_acell_s = h.off_acell;
  }
  if (off > 0xFFFFFFF0ull) throw resource_error("device plan exceeds 4 GiB");
  ep.total_bytes = static_cast<std::uint32_t>(off);
  ep.blob.assign(off, 0);
  put(ep.blob, h.off_sgrp, sgrp);
  put(ep.blob, h.off_sfn, sfn);
  put(ep.blob, h.off_pert53, pert53);
  put(ep.blob, h.off_pert32, pert32);
  put(ep.blob, h.off_pert53h, pert53h);
  put(ep.blob, h.off_groups, groups);
  put(ep.blob, h.off_fns, fns);
  put(ep.blob, h.off_grec, grec);
  put(ep.blob, h.off_acut, acut);
  put(ep.blob, h.off_aidx, aidx);
  put(ep.blob, h.off_acell, acell);
  if (h.fn_base || h.cell_base) {
    put(ep.blob, h.off_fns_s, fns_s);
    put(ep.blob, h.off_acell_s, acell_s);
  }
  put(ep.blob, h.off_arec, arec);
  put(ep.blob, h.off_scol, scol);
  if (h.single_compact) {
    arec4.assign(4 * static_cast<std::size_t>(h.n_single_alias), 0);
    auto addr = [&](std::uint32_t row, std::uint32_t slot) {
      return h.off_scol + (row * kScolSlots + slot) * 8;
    };
    for (std::uint32_t gi = 0; gi < h.n_single_alias; ++gi) {
      const std::uint32_t asz = v.grp_alias_size[gi], slot = gi % kScolSlots, r0 = scol_row0[gi];
      arec4[4 * gi + 0] = addr(r0, slot);
      arec4[4 * gi + 1] = addr(r0 + 2 * asz, slot);
      arec4[4 * gi + 2] = asz;
      arec4[4 * gi + 3] = ~asz;
    }
    put(ep.blob, h.off_arec4, arec4);
  }
  put(ep.blob, h.off_tables, tables);
  return ep;
}

}  // namespace pbn_b200
