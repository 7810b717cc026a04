// Native reader of the reference's line-oriented design format (SURVEY 8f
// rank 2): model.py:423-571 parse_design + the Design checks it runs
// (model.py:121-190 _validate) + the flat arrays of NetlistArrays
// (model.py:231-275), in one O(text) host pass.  At 800k instances the
// reference spends ~28 s parsing and ~9 s in NetlistArrays' per-pin Python
// loop; this reader hands the GP loop its arrays directly.
//
// Host code only (no kernels).  Errors carry the reference's messages
// ("line N: ..." for ParseError, the bare DesignError text otherwise), so the
// Python wrapper raises the same exceptions with the same text.  Numbers are
// read with strtod (Python's float() also accepts '_' digit separators; the
// generator and the reference's writers never emit them).
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

struct Kind {
  std::string name;
  double w = 0, h = 0;
  std::vector<std::string> pins;
  std::vector<double> dx, dy;
};

struct Tech {
  std::vector<Kind> kinds;  // insertion order (the reference's dict order)
  std::unordered_map<std::string, int> index;
};

struct Parsed {
  double die_w = 0, die_h = 0, row_t = 0, row_b = 0, util_t = 0, util_b = 0;
  double pitch = 0, spacing = 0, cost = 0;
  Tech tech[2];  // 0 bottom, 1 top
  std::vector<std::string> inst_name, inst_kind;
  std::vector<uint8_t> inst_macro;
  std::vector<std::string> net_name;
  std::vector<int64_t> net_ptr;
  std::vector<int64_t> pin_inst;
  std::vector<std::string> pin_name;
  // resolved per instance / pin
  std::vector<int> kind_top, kind_bot;
  std::vector<int> pin_idx;  // index of the pin name in its kind's (bottom) pin list
};

struct Fail {
  std::string msg;
};

[[noreturn]] void fail_line(long line, const std::string& msg) {
  throw Fail{"line " + std::to_string(line) + ": " + msg};
}
[[noreturn]] void fail(const std::string& msg) { throw Fail{msg}; }

bool to_num(std::string_view tok, double& v) {
  std::string s(tok);
  char* end = nullptr;
  v = strtod(s.c_str(), &end);
  return end && *end == '\0' && !s.empty();
}

double num(std::string_view tok, long line, const char* what = "number") {
  double v;
  if (!to_num(tok, v)) fail_line(line, std::string("expected ") + what + ", got '" + std::string(tok) + "'");
  return v;
}

// Python's repr of a float for the messages that print one (model.py:_validate)
std::string pyfloat(double v) {
  if (v == floor(v) && fabs(v) < 1e16) {
    char b[64];
    snprintf(b, sizeof b, "%.1f", v);
    return b;
  }
  char b[64];
  for (int p = 1; p <= 17; ++p) {
    snprintf(b, sizeof b, "%.*g", p, v);
    if (strtod(b, nullptr) == v) break;
  }
  return b;
}

void split(std::string_view line, std::vector<std::string_view>& toks) {
  toks.clear();
  size_t i = 0, n = line.size();
  while (i < n) {
    while (i < n && (line[i] == ' ' || line[i] == '\t' || line[i] == '\r' || line[i] == '\f' ||
                     line[i] == '\v'))
      ++i;
    if (i >= n) break;
    size_t j = i;
    while (j < n && !(line[j] == ' ' || line[j] == '\t' || line[j] == '\r' || line[j] == '\f' ||
                      line[j] == '\v'))
      ++j;
    toks.push_back(line.substr(i, j - i));
    i = j;
  }
}

void parse(const char* text, int64_t len, Parsed& P) {
  bool have_die = false, have_ut = false, have_ub = false, have_rt = false, have_rb = false,
       have_hbt = false;
  int cur_tech = -1;
  // open Cell / Net blocks
  bool in_cell = false, in_net = false;
  Kind cell;
  long cell_want = 0;
  std::string net_nm;
  long net_want = 0;
  std::vector<std::pair<long, std::string>> net_refs;
  std::vector<std::vector<std::pair<long, std::string>>> all_refs;
  std::unordered_map<std::string, int> inst_idx;

  auto finish_cell = [&](long line) {
    if (!in_cell) return;
    if ((long)cell.pins.size() != cell_want)
      fail_line(line, "cell " + cell.name + ": expected " + std::to_string(cell_want) +
                          " pins, got " + std::to_string(cell.pins.size()));
    Tech& t = P.tech[cur_tech];
    auto it = t.index.find(cell.name);
    if (it == t.index.end()) {
      t.index[cell.name] = (int)t.kinds.size();
      t.kinds.push_back(cell);
    } else {
      t.kinds[it->second] = cell;  // a dict re-assignment keeps the first position
    }
    in_cell = false;
  };
  auto finish_net = [&](long line) {
    if (!in_net) return;
    if ((long)net_refs.size() != net_want)
      fail_line(line, "net " + net_nm + ": expected " + std::to_string(net_want) + " pins, got " +
                          std::to_string(net_refs.size()));
    P.net_name.push_back(net_nm);
    all_refs.push_back(std::move(net_refs));
    net_refs.clear();
    in_net = false;
  };

  std::vector<std::string_view> toks;
  long line_no = 0, last_line = 0;
  int64_t pos = 0;
  while (pos < len) {
    int64_t e = pos;
    while (e < len && text[e] != '\n') ++e;
    ++line_no;
    std::string_view raw(text + pos, (size_t)(e - pos));
    pos = e + 1;
    const size_t hash = raw.find('#');
    if (hash != std::string_view::npos) raw = raw.substr(0, hash);
    split(raw, toks);
    if (toks.empty()) continue;
    last_line = line_no;
    const std::string_view key = toks[0];
    if (key == "Pin") {
      if (in_cell) {
        if (toks.size() != 4) fail_line(line_no, "Pin inside a Cell needs: Pin name ox oy");
        cell.pins.emplace_back(toks[1]);
        cell.dx.push_back(num(toks[2], line_no));
        cell.dy.push_back(num(toks[3], line_no));
      } else if (in_net) {
        if (toks.size() != 2 || toks[1].find('/') == std::string_view::npos)
          fail_line(line_no, "Pin inside a Net needs: Pin inst/pin");
        net_refs.emplace_back(line_no, std::string(toks[1]));
      } else {
        fail_line(line_no, "Pin outside of a Cell or Net block");
      }
      continue;
    }
    finish_cell(line_no);
    finish_net(line_no);
    if (key == "DieSize") {
      if (toks.size() != 3) fail_line(line_no, "DieSize needs two extents");
      P.die_w = num(toks[1], line_no);
      P.die_h = num(toks[2], line_no);
      have_die = true;
    } else if (key == "TopDieMaxUtil" || key == "BottomDieMaxUtil") {
      if (toks.size() < 2) fail_line(line_no, "expected number");
      const double v = num(toks[1], line_no);
      if (key[0] == 'T') { P.util_t = v; have_ut = true; } else { P.util_b = v; have_ub = true; }
    } else if (key == "TopDieRowHeight" || key == "BottomDieRowHeight") {
      if (toks.size() < 2) fail_line(line_no, "expected number");
      const double v = num(toks[1], line_no);
      if (key[0] == 'T') { P.row_t = v; have_rt = true; } else { P.row_b = v; have_rb = true; }
    } else if (key == "TopDieTech" || key == "BottomDieTech") {
      cur_tech = key[0] == 'T' ? 1 : 0;
    } else if (key == "Cell") {
      if (cur_tech < 0) fail_line(line_no, "Cell outside of a tech block");
      if (toks.size() != 5) fail_line(line_no, "Cell needs: Cell name w h npins");
      const double w = num(toks[2], line_no), h = num(toks[3], line_no);
      if (w <= 0 || h <= 0) fail_line(line_no, "cell " + std::string(toks[1]) + ": non-positive dimension");
      cell = Kind();
      cell.name = std::string(toks[1]);
      cell.w = w;
      cell.h = h;
      cell_want = (long)num(toks[4], line_no, "pin count");
      in_cell = true;
    } else if (key == "Inst") {
      if (toks.size() != 4) fail_line(line_no, "Inst needs: Inst name kind isMacro");
      std::string flag(toks[3]);
      for (auto& c : flag) c = (char)tolower((unsigned char)c);
      if (flag != "0" && flag != "1" && flag != "true" && flag != "false")
        fail_line(line_no, "bad isMacro flag '" + std::string(toks[3]) + "'");
      std::string nm(toks[1]);
      if (inst_idx.count(nm)) fail_line(line_no, "duplicate instance " + nm);
      inst_idx[nm] = (int)P.inst_name.size();
      P.inst_name.push_back(nm);
      P.inst_kind.emplace_back(toks[2]);
      P.inst_macro.push_back(flag == "1" || flag == "true");
    } else if (key == "Net") {
      if (toks.size() != 3) fail_line(line_no, "Net needs: Net name npins");
      net_nm = std::string(toks[1]);
      net_want = (long)num(toks[2], line_no, "pin count");
      in_net = true;
    } else if (key == "HBT") {
      if (toks.size() != 4) fail_line(line_no, "HBT needs: HBT pitch spacing cost");
      P.pitch = num(toks[1], line_no);
      P.spacing = num(toks[2], line_no);
      P.cost = num(toks[3], line_no);
      have_hbt = true;
    } else {
      fail_line(line_no, "unknown directive '" + std::string(key) + "'");
    }
  }
  finish_cell(last_line + 1);
  finish_net(last_line + 1);
  if (!have_die) fail_line(last_line + 1, "missing DieSize");
  if (!have_ut || !have_ub) fail_line(last_line + 1, "missing die utilization");
  if (!have_rt || !have_rb) fail_line(last_line + 1, "missing row heights");
  if (!have_hbt) fail_line(last_line + 1, "missing HBT line");
  // net pins -> (instance, pin name)
  P.net_ptr.assign(1, 0);
  for (size_t j = 0; j < all_refs.size(); ++j) {
    for (const auto& r : all_refs[j]) {
      const size_t slash = r.second.find('/');
      const std::string in = r.second.substr(0, slash), pn = r.second.substr(slash + 1);
      auto it = inst_idx.find(in);
      if (it == inst_idx.end())
        fail_line(r.first, "net " + P.net_name[j] + ": unknown instance '" + in + "'");
      P.pin_inst.push_back(it->second);
      P.pin_name.push_back(pn);
    }
    P.net_ptr.push_back((int64_t)P.pin_inst.size());
  }
  // Design(...): duplicate net names, then _validate (model.py:121-190)
  {
    std::unordered_map<std::string, int> seen;
    for (size_t j = 0; j < P.net_name.size(); ++j)
      if (!seen.emplace(P.net_name[j], (int)j).second) fail("duplicate net name");
  }
  if (P.die_w <= 0 || P.die_h <= 0) fail("die extents must be positive");
  for (double u : {P.util_t, P.util_b})
    if (!(0 < u && u <= 1)) fail("utilization " + pyfloat(u) + " outside (0, 1]");
  for (double rh : {P.row_t, P.row_b}) {
    if (rh <= 0) fail("row height must be positive");
    const double n = P.die_h / rh;
    if (fabs(n - nearbyint(n)) > 1e-9)
      fail("rows of height " + pyfloat(rh) + " do not tile die height " + pyfloat(P.die_h));
  }
  if (P.pitch <= 0 || P.spacing < 0 || P.cost < 0) fail("bad HBT spec");
  for (int d : {1, 0}) {
    const char* tag = d ? "top" : "bottom";
    for (const Kind& k : P.tech[d].kinds) {
      if (k.w <= 0 || k.h <= 0) fail(std::string(tag) + " kind " + k.name + " has non-positive dimensions");
      for (size_t p = 0; p < k.pins.size(); ++p)
        if (fabs(k.dx[p]) > k.w / 2 + 1e-9 || fabs(k.dy[p]) > k.h / 2 + 1e-9)
          fail("pin " + k.name + "/" + k.pins[p] + " offset outside the " + tag + " footprint");
    }
  }
  const size_t n = P.inst_name.size();
  P.kind_top.resize(n);
  P.kind_bot.resize(n);
  for (size_t i = 0; i < n; ++i) {
    auto t = P.tech[1].index.find(P.inst_kind[i]);
    auto b = P.tech[0].index.find(P.inst_kind[i]);
    if (t == P.tech[1].index.end() || b == P.tech[0].index.end())
      fail("instance " + P.inst_name[i] + ": kind " + P.inst_kind[i] + " missing from a die tech");
    P.kind_top[i] = t->second;
    P.kind_bot[i] = b->second;
    if (P.tech[1].kinds[t->second].pins != P.tech[0].kinds[b->second].pins)
      fail("kind " + P.inst_kind[i] + ": pin lists differ between dies");
  }
  P.pin_idx.resize(P.pin_inst.size());
  for (size_t j = 0; j + 1 < P.net_ptr.size(); ++j) {
    if (P.net_ptr[j + 1] == P.net_ptr[j]) fail("net " + P.net_name[j] + " has no pins");
    for (int64_t p = P.net_ptr[j]; p < P.net_ptr[j + 1]; ++p) {
      const Kind& k = P.tech[0].kinds[P.kind_bot[P.pin_inst[p]]];
      int idx = -1;  // CellKind.pin_offset: the first pin of that name
      for (size_t q = 0; q < k.pins.size(); ++q)
        if (k.pins[q] == P.pin_name[p]) { idx = (int)q; break; }
      if (idx < 0)
        fail("net " + P.net_name[j] + ": pin " + P.inst_name[P.pin_inst[p]] + "/" + P.pin_name[p] + " undefined");
      P.pin_idx[p] = idx;
    }
  }
}

}  // namespace

}  // namespace p3d

extern "C" {

int p3d_parse_design(const char* text, int64_t len, void** handle) {
  using namespace p3d;
  if (!text || len < 0 || !handle) { set_error("parse_design: bad args"); return P3D_ERR_ARG; }
  *handle = nullptr;
  Parsed* P = new Parsed();
  try {
    parse(text, len, *P);
  } catch (const Fail& f) {
    delete P;
    set_error("%s", f.msg.c_str());
    return P3D_ERR_ARG;
  } catch (...) {
    delete P;
    set_error("parse_design: out of memory");
    return P3D_ERR_CUDA;
  }
  *handle = P;
  return P3D_OK;
}

int p3d_parsed_counts(const void* handle, int64_t* counts, double* scalars) {
  using namespace p3d;
  const Parsed* P = static_cast<const Parsed*>(handle);
  if (!P || !counts || !scalars) { set_error("parsed_counts: bad args"); return P3D_ERR_ARG; }
  int64_t ib = 0, nb = 0;
  for (const auto& s : P->inst_name) ib += (int64_t)s.size() + 1;
  for (const auto& s : P->net_name) nb += (int64_t)s.size() + 1;
  counts[0] = (int64_t)P->inst_name.size();
  counts[1] = (int64_t)P->net_name.size();
  counts[2] = (int64_t)P->pin_inst.size();
  counts[3] = ib;
  counts[4] = nb;
  const double s[9] = {P->die_w, P->die_h, P->row_t, P->row_b, P->util_t, P->util_b,
                       P->pitch, P->spacing, P->cost};
  memcpy(scalars, s, sizeof s);
  return P3D_OK;
}

int p3d_parsed_fill(const void* handle, uint8_t* is_macro, double* w_top, double* h_top,
                    double* w_bot, double* h_bot, int64_t* net_ptr, int64_t* pin_inst,
                    double* ox_top, double* oy_top, double* ox_bot, double* oy_bot,
                    char* inst_names, char* net_names) {
  using namespace p3d;
  const Parsed* P = static_cast<const Parsed*>(handle);
  if (!P || !is_macro || !w_top || !h_top || !w_bot || !h_bot || !net_ptr || !pin_inst ||
      !ox_top || !oy_top || !ox_bot || !oy_bot || !inst_names || !net_names) {
    set_error("parsed_fill: bad args");
    return P3D_ERR_ARG;
  }
  const size_t n = P->inst_name.size();
  for (size_t i = 0; i < n; ++i) {
    const Kind& kt = P->tech[1].kinds[P->kind_top[i]];
    const Kind& kb = P->tech[0].kinds[P->kind_bot[i]];
    is_macro[i] = P->inst_macro[i];
    w_top[i] = kt.w; h_top[i] = kt.h;
    w_bot[i] = kb.w; h_bot[i] = kb.h;
  }
  memcpy(net_ptr, P->net_ptr.data(), P->net_ptr.size() * sizeof(int64_t));
  for (size_t p = 0; p < P->pin_inst.size(); ++p) {
    const int64_t i = P->pin_inst[p];
    const int q = P->pin_idx[p];
    const Kind& kt = P->tech[1].kinds[P->kind_top[i]];
    const Kind& kb = P->tech[0].kinds[P->kind_bot[i]];
    pin_inst[p] = i;
    ox_top[p] = kt.dx[q]; oy_top[p] = kt.dy[q];
    ox_bot[p] = kb.dx[q]; oy_bot[p] = kb.dy[q];
  }
  char* o = inst_names;
  for (const auto& s : P->inst_name) { memcpy(o, s.data(), s.size()); o += s.size(); *o++ = '\n'; }
  o = net_names;
  for (const auto& s : P->net_name) { memcpy(o, s.data(), s.size()); o += s.size(); *o++ = '\n'; }
  return P3D_OK;
}

void p3d_parsed_free(void* handle) { delete static_cast<p3d::Parsed*>(handle); }

}  // extern "C"
