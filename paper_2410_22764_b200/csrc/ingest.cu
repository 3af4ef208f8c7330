// LTS ingestion front-end: parse_lts / determinize / complete
// of the reference's ingest.hpp:130-284, host-side as the survey recommends (the
// subset construction is sequential by definition: states are numbered in
// breadth-first discovery order).  Same results, same errors (ParseError line
// numbers and messages, SubsetBudgetExceeded), but:
//   * parse_lts runs multi-threaded: the body is cut at line boundaries into
//     chunks parsed in parallel, each with its own label table; labels are then
//     interned in global first-appearance order (chunk order, then order inside a
//     chunk) and the transitions remapped — identical to the sequential intern;
//     the reported error is the first one in file order;
//   * determinize keeps the transitions in one CSR by source state, sorted by
//     label (not the reference's n x labels vectors), expands a subset over all
//     labels in one sweep, and interns subsets in a flat pool behind an
//     open-addressing table.
// The completed automaton goes straight to the minimizers (dfm_sort_pr & co).
#include <algorithm>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "dfm_internal.cuh"

namespace dfm {
namespace ingest {

struct ParseFail {
  uint64_t line;
  std::string what;
};

struct Lts {
  uint32_t num_states = 0, initial = 0;
  std::vector<std::string> labels;
  std::vector<uint32_t> src, label, dst;
};

struct PartialDfa {
  uint32_t n = 0, k = 0, initial = 0;
  std::vector<uint32_t> delta;  // [k][n], kMissing = 0xFFFFFFFF
};

namespace {

struct Cursor {  // ingest.hpp detail::LineCursor
  std::string_view text;
  size_t pos = 0;
  uint64_t line;
  Cursor(std::string_view t, uint64_t l) : text(t), line(l) {}
  [[noreturn]] void fail(const std::string& w) const { throw ParseFail{line, w}; }
  void skip_ws() {
    while (pos < text.size() && (text[pos] == ' ' || text[pos] == '\t')) ++pos;
  }
  bool at_end() {
    skip_ws();
    return pos >= text.size();
  }
  void expect(char c, const char* what) {
    skip_ws();
    if (pos >= text.size() || text[pos] != c) fail(std::string("expected '") + c + "' " + what);
    ++pos;
  }
  uint64_t parse_uint(const char* what) {
    skip_ws();
    if (pos >= text.size() || text[pos] < '0' || text[pos] > '9')
      fail(std::string("expected number for ") + what);
    uint64_t v = 0;
    while (pos < text.size() && text[pos] >= '0' && text[pos] <= '9') {
      v = v * 10 + (uint64_t)(text[pos] - '0');
      if (v > 0xFFFFFFFFull) fail(std::string(what) + " out of range");
      ++pos;
    }
    return v;
  }
  std::string_view parse_label() {
    skip_ws();
    if (pos < text.size() && text[pos] == '"') {
      ++pos;
      const size_t close = text.find('"', pos);
      if (close == std::string_view::npos) fail("unterminated label quote");
      const std::string_view l = text.substr(pos, close - pos);
      pos = close + 1;
      return l;
    }
    const size_t stop = text.find(',', pos);
    if (stop == std::string_view::npos) fail("missing label field");
    size_t end = stop;
    while (end > pos && (text[end - 1] == ' ' || text[end - 1] == '\t')) --end;
    if (end == pos) fail("empty label");
    const std::string_view l = text.substr(pos, end - pos);
    pos = stop;
    return l;
  }
};

bool blank(std::string_view l) {
  for (char c : l)
    if (c != ' ' && c != '\t') return false;
  return true;
}

// next line of text[i..): returns its view without '\n' / trailing '\r'; i advances
std::string_view next_line(std::string_view text, size_t& i, bool& last) {
  const size_t nl = text.find('\n', i);
  const size_t end = nl == std::string_view::npos ? text.size() : nl;
  std::string_view l = text.substr(i, end - i);
  if (!l.empty() && l.back() == '\r') l.remove_suffix(1);
  last = nl == std::string_view::npos;
  i = last ? text.size() : nl + 1;
  return l;
}

struct Chunk {
  size_t begin = 0, end = 0;      // byte range, starts at a line start
  uint64_t first_line = 0;        // line number of its first line
  std::vector<std::string_view> labels;  // local table, first-appearance order
  std::vector<uint32_t> src, lab, dst;
  bool has_error = false;
  ParseFail err;
  uint64_t last_nonempty = 0;     // line number of the chunk's last non-blank line
};

void parse_chunk(std::string_view text, uint64_t num_states, Chunk& c) {
  std::unordered_map<std::string_view, uint32_t> local;
  size_t i = c.begin;
  uint64_t line = c.first_line;
  while (i < c.end) {
    bool last;
    const std::string_view l = next_line(text, i, last);
    const uint64_t ln = line++;
    if (blank(l)) continue;
    c.last_nonempty = ln;
    try {
      Cursor cur(l, ln);
      cur.expect('(', "starting transition");
      const uint64_t s = cur.parse_uint("source state");
      cur.expect(',', "after source state");
      const std::string_view label = cur.parse_label();
      cur.expect(',', "after label");
      const uint64_t d = cur.parse_uint("target state");
      cur.expect(')', "closing transition");
      if (!cur.at_end()) cur.fail("trailing characters after transition");
      if (s >= num_states) cur.fail("source state out of range");
      if (d >= num_states) cur.fail("target state out of range");
      auto it = local.find(label);
      uint32_t id;
      if (it == local.end()) {
        id = (uint32_t)c.labels.size();
        local.emplace(label, id);
        c.labels.push_back(label);
      } else {
        id = it->second;
      }
      c.src.push_back((uint32_t)s);
      c.lab.push_back(id);
      c.dst.push_back((uint32_t)d);
    } catch (const ParseFail& f) {
      c.has_error = true;
      c.err = f;
      return;
    }
    if (last) break;
  }
}

unsigned parse_threads(size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return (unsigned)std::max<size_t>(1, std::min<size_t>(std::min(hw, 32u), bytes >> 20));
}

}  // namespace

Lts parse_lts(std::string_view text) {
  // header: the first non-blank line (ingest.hpp:130-154)
  size_t i = 0;
  uint64_t line = 1;
  std::string_view head;
  uint64_t head_line = 0;
  bool found = false;
  while (i <= text.size()) {
    bool last;
    const std::string_view l = next_line(text, i, last);
    const uint64_t ln = line++;
    if (!blank(l)) {
      head = l;
      head_line = ln;
      found = true;
      break;
    }
    if (last) break;
  }
  if (!found) throw ParseFail{1, "missing des header"};
  Cursor h(head, head_line);
  h.skip_ws();
  if (h.text.substr(h.pos, 3) != "des") h.fail("expected des header");
  h.pos += 3;
  h.expect('(', "after des");
  const uint64_t initial = h.parse_uint("initial state");
  h.expect(',', "after initial state");
  const uint64_t num_t = h.parse_uint("transition count");
  h.expect(',', "after transition count");
  const uint64_t num_states = h.parse_uint("state count");
  h.expect(')', "closing header");
  if (!h.at_end()) h.fail("trailing characters after header");
  if (num_states == 0) h.fail("state count must be positive");
  if (initial >= num_states) h.fail("initial state out of range");

  // body [i, size): chunks at line boundaries, line numbers from newline counts
  const size_t body = i;
  const unsigned T = parse_threads(text.size() - body);
  std::vector<Chunk> chunks(T);
  size_t at = body;
  for (unsigned t = 0; t < T; ++t) {
    chunks[t].begin = at;
    size_t cut = t + 1 == T ? text.size() : body + (text.size() - body) * (t + 1) / T;
    if (cut < at) cut = at;
    if (t + 1 < T) {
      const size_t nl = text.find('\n', cut);
      cut = nl == std::string_view::npos ? text.size() : nl + 1;
    }
    chunks[t].end = cut;
    at = cut;
  }
  {
    std::vector<uint64_t> nls(T, 0);
    auto count = [&](unsigned t) {
      nls[t] = (uint64_t)std::count(text.begin() + chunks[t].begin, text.begin() + chunks[t].end, '\n');
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(count, t);
    count(0);
    for (auto& x : th) x.join();
    uint64_t ln = line;  // the line after the header
    for (unsigned t = 0; t < T; ++t) {
      chunks[t].first_line = ln;
      ln += nls[t];
    }
  }
  {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t)
      th.emplace_back([&, t] { parse_chunk(text, num_states, chunks[t]); });
    parse_chunk(text, num_states, chunks[0]);
    for (auto& x : th) x.join();
  }
  for (auto& c : chunks)
    if (c.has_error) throw c.err;  // first error in file order
  Lts lts;
  lts.num_states = (uint32_t)num_states;
  lts.initial = (uint32_t)initial;
  // global label ids in first-appearance order; per-chunk remap tables
  std::unordered_map<std::string_view, uint32_t> global;
  std::vector<std::vector<uint32_t>> remap(T);
  uint64_t total = 0, last_line = head_line;
  for (unsigned t = 0; t < T; ++t) {
    auto& c = chunks[t];
    remap[t].resize(c.labels.size());
    for (size_t j = 0; j < c.labels.size(); ++j) {
      auto it = global.find(c.labels[j]);
      if (it == global.end()) {
        const uint32_t id = (uint32_t)lts.labels.size();
        global.emplace(c.labels[j], id);
        lts.labels.emplace_back(c.labels[j]);
        remap[t][j] = id;
      } else {
        remap[t][j] = it->second;
      }
    }
    total += c.src.size();
    if (c.last_nonempty) last_line = c.last_nonempty;
  }
  if (total != num_t)
    throw ParseFail{last_line, "header declares " + std::to_string(num_t) + " transitions, found " +
                                   std::to_string(total)};
  lts.src.resize(total);
  lts.label.resize(total);
  lts.dst.resize(total);
  std::vector<uint64_t> off(T + 1, 0);
  for (unsigned t = 0; t < T; ++t) off[t + 1] = off[t] + chunks[t].src.size();
  std::vector<std::thread> th;
  auto place = [&](unsigned t) {
    const auto& c = chunks[t];
    for (size_t j = 0; j < c.src.size(); ++j) {
      lts.src[off[t] + j] = c.src[j];
      lts.label[off[t] + j] = remap[t][c.lab[j]];
      lts.dst[off[t] + j] = c.dst[j];
    }
  };
  for (unsigned t = 1; t < T; ++t) th.emplace_back(place, t);
  place(0);
  for (auto& x : th) x.join();
  return lts;
}

struct BudgetExceeded {
  uint64_t budget;
};

PartialDfa determinize(const Lts& lts, uint64_t max_subsets) {
  const uint32_t n = lts.num_states, L = (uint32_t)lts.labels.size();
  const uint64_t m = lts.src.size();
  // CSR by source, each state's transitions ordered by label (stable)
  std::vector<uint64_t> off(n + 1, 0);
  for (uint64_t j = 0; j < m; ++j) ++off[lts.src[j] + 1];
  for (uint32_t s = 0; s < n; ++s) off[s + 1] += off[s];
  std::vector<uint32_t> tl(m), td(m);
  {
    std::vector<uint64_t> cur(off.begin(), off.end() - 1);
    for (uint64_t j = 0; j < m; ++j) {
      const uint64_t p = cur[lts.src[j]]++;
      tl[p] = lts.label[j];
      td[p] = lts.dst[j];
    }
    for (uint32_t s = 0; s < n; ++s) {
      // stable sort of the segment by label (counting order of labels)
      const uint64_t a = off[s], b = off[s + 1];
      if (b - a < 2) continue;
      std::vector<std::pair<uint32_t, uint32_t>> seg(b - a);
      for (uint64_t p = a; p < b; ++p) seg[p - a] = {tl[p], td[p]};
      std::stable_sort(seg.begin(), seg.end(),
                       [](const auto& x, const auto& y) { return x.first < y.first; });
      for (uint64_t p = a; p < b; ++p) {
        tl[p] = seg[p - a].first;
        td[p] = seg[p - a].second;
      }
    }
  }
  // subsets: flat pool + open-addressing intern table
  std::vector<uint32_t> pool;
  std::vector<uint64_t> sub_off{0};
  std::vector<uint32_t> table(1024, 0xFFFFFFFFu);
  auto hash_of = [](const uint32_t* p, size_t len) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ len;
    for (size_t i = 0; i < len; ++i) {
      h ^= p[i] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
      h *= 0xBF58476D1CE4E5B9ull;
    }
    return h ^ (h >> 31);
  };
  auto count = [&]() { return (uint64_t)(sub_off.size() - 1); };
  auto grow = [&]() {
    std::vector<uint32_t> t2(table.size() * 2, 0xFFFFFFFFu);
    for (uint64_t id = 0; id < count(); ++id) {
      const uint32_t* p = pool.data() + sub_off[id];
      uint64_t x = hash_of(p, sub_off[id + 1] - sub_off[id]) & (t2.size() - 1);
      while (t2[x] != 0xFFFFFFFFu) x = (x + 1) & (t2.size() - 1);
      t2[x] = (uint32_t)id;
    }
    table.swap(t2);
  };
  // intern the sorted subset stored at the pool's tail (length len)
  auto intern_tail = [&](size_t len) -> uint32_t {
    const uint32_t* p = pool.data() + pool.size() - len;
    uint64_t x = hash_of(p, len) & (table.size() - 1);
    while (table[x] != 0xFFFFFFFFu) {
      const uint32_t id = table[x];
      const uint64_t a = sub_off[id], b = sub_off[id + 1];
      if (b - a == len && std::equal(p, p + len, pool.data() + a)) {
        pool.resize(pool.size() - len);  // known subset: drop the tail
        return id;
      }
      x = (x + 1) & (table.size() - 1);
    }
    if (count() >= max_subsets) throw BudgetExceeded{max_subsets};
    const uint32_t id = (uint32_t)count();
    table[x] = id;
    sub_off.push_back(pool.size());
    if (count() * 2 > table.size()) grow();
    return id;
  };
  pool.push_back(lts.initial);
  intern_tail(1);
  PartialDfa out;
  out.k = L;
  out.initial = 0;
  std::vector<std::vector<uint32_t>> rows(L);
  std::vector<std::vector<uint32_t>> tgt(L);
  std::vector<uint32_t> touched;
  for (uint64_t cur = 0; cur < count(); ++cur) {
    touched.clear();
    for (uint64_t e = sub_off[cur]; e < sub_off[cur + 1]; ++e) {
      const uint32_t s = pool[e];
      for (uint64_t p = off[s]; p < off[s + 1]; ++p) {
        if (tgt[tl[p]].empty()) touched.push_back(tl[p]);
        tgt[tl[p]].push_back(td[p]);
      }
    }
    for (uint32_t a = 0; a < L; ++a) rows[a].push_back(0xFFFFFFFFu);  // kMissing by default
    std::sort(touched.begin(), touched.end());  // labels in index order
    for (uint32_t a : touched) {
      auto& v = tgt[a];
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      pool.insert(pool.end(), v.begin(), v.end());
      rows[a].back() = intern_tail(v.size());
      v.clear();
    }
  }
  out.n = (uint32_t)count();
  out.delta.resize((uint64_t)L * out.n);
  for (uint32_t a = 0; a < L; ++a)
    std::copy(rows[a].begin(), rows[a].end(), out.delta.begin() + (uint64_t)a * out.n);
  return out;
}

}  // namespace ingest
}  // namespace dfm

// ------------------------------------------------------------------ C-ABI
using namespace dfm::ingest;

struct dfm_lts {
  Lts v;
};
struct dfm_pdfa {
  PartialDfa v;
};

namespace {
void set_err(char* err, uint32_t cap, const std::string& m) {
  if (err && cap) {
    std::strncpy(err, m.c_str(), cap - 1);
    err[cap - 1] = 0;
  }
}
}  // namespace

extern "C" {

int dfm_lts_parse(const char* text, uint64_t len, dfm_lts** out, uint64_t* err_line, char* err,
                  uint32_t err_cap) {
  if (out == nullptr || (text == nullptr && len)) return DFM_ERR_INVALID;
  *out = nullptr;
  try {
    auto* l = new dfm_lts{parse_lts(std::string_view(text ? text : "", len))};
    *out = l;
    return DFM_OK;
  } catch (const ParseFail& f) {
    if (err_line) *err_line = f.line;
    set_err(err, err_cap, "line " + std::to_string(f.line) + ": " + f.what);
    return DFM_ERR_PARSE;
  } catch (const std::bad_alloc&) {
    return DFM_ERR_NO_MEMORY;
  }
}

int dfm_lts_info(const dfm_lts* l, uint32_t* num_states, uint32_t* initial, uint32_t* num_labels,
                 uint64_t* num_transitions) {
  if (l == nullptr) return DFM_ERR_INVALID;
  if (num_states) *num_states = l->v.num_states;
  if (initial) *initial = l->v.initial;
  if (num_labels) *num_labels = (uint32_t)l->v.labels.size();
  if (num_transitions) *num_transitions = l->v.src.size();
  return DFM_OK;
}

int dfm_lts_label(const dfm_lts* l, uint32_t i, const char** data, uint64_t* len) {
  if (l == nullptr || i >= l->v.labels.size()) return DFM_ERR_INVALID;
  if (data) *data = l->v.labels[i].data();
  if (len) *len = l->v.labels[i].size();
  return DFM_OK;
}

int dfm_lts_transitions(const dfm_lts* l, uint32_t* src, uint32_t* label, uint32_t* dst) {
  if (l == nullptr) return DFM_ERR_INVALID;
  const size_t m = l->v.src.size();
  if (src) std::memcpy(src, l->v.src.data(), m * 4);
  if (label) std::memcpy(label, l->v.label.data(), m * 4);
  if (dst) std::memcpy(dst, l->v.dst.data(), m * 4);
  return DFM_OK;
}

void dfm_lts_free(dfm_lts* l) { delete l; }

int dfm_lts_build(uint32_t num_states, uint32_t initial, uint32_t num_labels,
                  const char* const* labels, const uint64_t* label_lens, uint64_t m,
                  const uint32_t* src, const uint32_t* label, const uint32_t* dst, dfm_lts** out) {
  if (out == nullptr || num_states == 0 || initial >= num_states) return DFM_ERR_INVALID;
  *out = nullptr;
  auto* l = new dfm_lts;
  l->v.num_states = num_states;
  l->v.initial = initial;
  for (uint32_t i = 0; i < num_labels; ++i)
    l->v.labels.emplace_back(labels ? std::string(labels[i], label_lens[i]) : std::to_string(i));
  l->v.src.assign(src, src + m);
  l->v.label.assign(label, label + m);
  l->v.dst.assign(dst, dst + m);
  for (uint64_t j = 0; j < m; ++j)
    if (src[j] >= num_states || dst[j] >= num_states || label[j] >= num_labels) {
      delete l;
      return DFM_ERR_INVALID;
    }
  *out = l;
  return DFM_OK;
}

int dfm_determinize(const dfm_lts* l, uint64_t max_subset_states, dfm_pdfa** out,
                    uint64_t* budget_out) {
  if (l == nullptr || out == nullptr) return DFM_ERR_INVALID;
  *out = nullptr;
  try {
    *out = new dfm_pdfa{determinize(l->v, max_subset_states)};
    return DFM_OK;
  } catch (const BudgetExceeded& b) {
    if (budget_out) *budget_out = b.budget;
    return DFM_ERR_BUDGET;
  } catch (const std::bad_alloc&) {
    return DFM_ERR_NO_MEMORY;
  }
}

int dfm_pdfa_shape(const dfm_pdfa* p, uint32_t* n, uint32_t* k, uint32_t* initial) {
  if (p == nullptr) return DFM_ERR_INVALID;
  if (n) *n = p->v.n;
  if (k) *k = p->v.k;
  if (initial) *initial = p->v.initial;
  return DFM_OK;
}

int dfm_pdfa_rows(const dfm_pdfa* p, uint32_t* delta_flat) {
  if (p == nullptr || (delta_flat == nullptr && !p->v.delta.empty())) return DFM_ERR_INVALID;
  std::memcpy(delta_flat, p->v.delta.data(), p->v.delta.size() * 4);
  return DFM_OK;
}

int dfm_complete(const dfm_pdfa* p, uint32_t* num_states_out, uint32_t* delta_flat,
                 uint8_t* accepting) {
  // ingest.hpp:253-284: one rejecting sink appended iff a transition is missing
  if (p == nullptr || num_states_out == nullptr) return DFM_ERR_INVALID;
  const auto& v = p->v;
  const bool missing =
      std::find(v.delta.begin(), v.delta.end(), 0xFFFFFFFFu) != v.delta.end();
  const uint32_t n = v.n + (missing ? 1 : 0);
  *num_states_out = n;
  if (delta_flat) {
    for (uint32_t a = 0; a < v.k; ++a) {
      for (uint32_t q = 0; q < v.n; ++q) {
        const uint32_t t = v.delta[(uint64_t)a * v.n + q];
        delta_flat[(uint64_t)a * n + q] = t == 0xFFFFFFFFu ? v.n : t;
      }
      if (missing) delta_flat[(uint64_t)a * n + v.n] = v.n;
    }
  }
  if (accepting) {
    std::memset(accepting, 1, n);
    if (missing) accepting[v.n] = 0;
  }
  return DFM_OK;
}

void dfm_pdfa_free(dfm_pdfa* p) { delete p; }

int dfm_pdfa_build(uint32_t num_states, uint32_t alphabet_size, uint32_t initial,
                   const uint32_t* delta_flat, dfm_pdfa** out) {
  if (out == nullptr || num_states == 0 || initial >= num_states) return DFM_ERR_INVALID;
  auto* p = new dfm_pdfa;
  p->v.n = num_states;
  p->v.k = alphabet_size;
  p->v.initial = initial;
  p->v.delta.assign(delta_flat, delta_flat + (uint64_t)num_states * alphabet_size);
  for (uint32_t t : p->v.delta)
    if (t != 0xFFFFFFFFu && t >= num_states) {
      delete p;
      return DFM_ERR_INVALID;
    }
  *out = p;
  return DFM_OK;
}

}  // extern "C"
