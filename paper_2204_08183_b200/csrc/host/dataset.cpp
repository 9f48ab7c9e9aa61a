// dataset.cpp — sorted host layout, COO ingestion, subsetting, persistence and
// the lazily created device copy of a SurvivalDataset.
#include "survscan/dataset.hpp"

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <string_view>
#include <unordered_set>
#include <cmath>
#include <fstream>
#include <numeric>
#include <sstream>

#include "../../../include/gss.h"
#include "survscan/engine.hpp"  // default_device()
#include "survscan/errors.hpp"

namespace survscan {

struct SurvivalDataset::DeviceCache {
  std::mutex mu;
  std::vector<gss_dataset*> by_device;
  ~DeviceCache() {
    for (gss_dataset* d : by_device)
      if (d) gss_dataset_release(d);
  }
};

SurvivalDataset::SurvivalDataset(const SurvivalDataset& o)
    : times_(o.times_), status_(o.status_), row_ids_(o.row_ids_), col_ptr_(o.col_ptr_),
      row_idx_(o.row_idx_), vals_(o.vals_), stratum_start_(o.stratum_start_),
      n_events_(o.n_events_), has_competing_(o.has_competing_), dev_(o.dev_) {}
SurvivalDataset& SurvivalDataset::operator=(const SurvivalDataset& o) {
  if (this != &o) {
    SurvivalDataset tmp(o);
    *this = std::move(tmp);
  }
  return *this;
}
SurvivalDataset::SurvivalDataset(SurvivalDataset&&) noexcept = default;
SurvivalDataset& SurvivalDataset::operator=(SurvivalDataset&&) noexcept = default;
SurvivalDataset::~SurvivalDataset() = default;

SurvivalDataset SurvivalDataset::assemble(
    std::vector<double> times, std::vector<int> status, std::vector<std::int64_t> row_ids,
    std::size_t n_cols, std::vector<std::vector<std::pair<std::uint32_t, double>>> cols,
    std::vector<std::uint8_t> stratum_start) {
  SurvivalDataset ds;
  ds.times_ = std::move(times);
  ds.status_ = std::move(status);
  ds.row_ids_ = std::move(row_ids);
  ds.stratum_start_ = std::move(stratum_start);
  for (int s : ds.status_) {
    if (s == 1) ++ds.n_events_;
    if (s == 2) ds.has_competing_ = true;
  }
  ds.col_ptr_.assign(n_cols + 1, 0);
  for (std::size_t j = 0; j < n_cols; ++j)
    ds.col_ptr_[j + 1] = ds.col_ptr_[j] + static_cast<std::int64_t>(cols[j].size());
  ds.row_idx_.reserve(static_cast<std::size_t>(ds.col_ptr_[n_cols]));
  ds.vals_.reserve(static_cast<std::size_t>(ds.col_ptr_[n_cols]));
  for (auto& c : cols)
    for (const auto& [i, v] : c) {
      ds.row_idx_.push_back(static_cast<std::int32_t>(i));
      ds.vals_.push_back(v);
    }
  ds.dev_ = std::make_shared<DeviceCache>();
  return ds;
}

SurvivalDataset SurvivalDataset::assemble_csc(std::vector<double> times, std::vector<int> status,
                                              std::vector<std::int64_t> row_ids,
                                              std::vector<std::int64_t> col_ptr,
                                              std::vector<std::int32_t> row_idx,
                                              std::vector<double> vals,
                                              std::vector<std::uint8_t> stratum_start) {
  SurvivalDataset ds;
  ds.times_ = std::move(times);
  ds.status_ = std::move(status);
  ds.row_ids_ = std::move(row_ids);
  ds.stratum_start_ = std::move(stratum_start);
  for (int s : ds.status_) {
    if (s == 1) ++ds.n_events_;
    if (s == 2) ds.has_competing_ = true;
  }
  ds.col_ptr_ = std::move(col_ptr);
  ds.row_idx_ = std::move(row_idx);
  ds.vals_ = std::move(vals);
  ds.dev_ = std::make_shared<DeviceCache>();
  return ds;
}

std::uint64_t SurvivalDataset::content_hash() const {
  // FNV-1a over the sorted layout (times, status, CSC structure and values)
  std::uint64_t h = 0xcbf29ce484222325ULL;
  auto feed = [&h](const void* data, std::size_t bytes) {
    const auto* q = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < bytes; ++i) {
      h ^= q[i];
      h *= 0x100000001b3ULL;
    }
  };
  feed(times_.data(), times_.size() * sizeof(double));
  feed(status_.data(), status_.size() * sizeof(int));
  feed(col_ptr_.data(), col_ptr_.size() * sizeof(std::int64_t));
  feed(row_idx_.data(), row_idx_.size() * sizeof(std::int32_t));
  feed(vals_.data(), vals_.size() * sizeof(double));
  feed(stratum_start_.data(), stratum_start_.size());
  return h;
}

double SurvivalDataset::covariate(std::size_t i, std::size_t j) const {
  if (j >= p()) throw InvalidColumnError("covariate: column " + std::to_string(j) + " outside dataset");
  if (i >= n()) throw IndexError("covariate: row " + std::to_string(i) + " outside dataset");
  const auto b = row_idx_.begin() + col_ptr_[j], e = row_idx_.begin() + col_ptr_[j + 1];
  const auto it = std::lower_bound(b, e, static_cast<std::int32_t>(i));
  if (it == e || *it != static_cast<std::int32_t>(i)) return 0.0;
  return vals_[static_cast<std::size_t>(it - row_idx_.begin())];
}

SurvivalDataset SurvivalDataset::subset_rows(const std::vector<std::uint32_t>& positions,
                                             bool fresh_row_ids) const {
  const std::size_t m = positions.size();
  for (std::size_t i = 0; i + 1 < m; ++i)
    if (positions[i] > positions[i + 1])
      throw DomainError("subset_rows: positions must be non-decreasing");
  if (!positions.empty() && positions.back() >= n())
    throw IndexError("subset_rows: position outside dataset");
  if (!fresh_row_ids)
    for (std::size_t i = 0; i + 1 < m; ++i)
      if (positions[i] == positions[i + 1])
        throw DuplicateEntryError("subset_rows: repeated position needs fresh ids");
  std::vector<double> t(m);
  std::vector<int> s(m);
  std::vector<std::int64_t> ids(m);
  std::vector<std::uint8_t> ss;
  if (has_strata()) ss.assign(m, 0);
  for (std::size_t i = 0; i < m; ++i) {
    t[i] = times_[positions[i]];
    s[i] = status_[positions[i]];
    ids[i] = fresh_row_ids ? static_cast<std::int64_t>(i) : row_ids_[positions[i]];
  }
  if (has_strata()) {
    // a new stratum starts where the source stratum ordinal changes
    std::vector<std::int64_t> ord(n());
    std::int64_t k = -1;
    for (std::size_t i = 0; i < n(); ++i) ord[i] = (k += (i == 0 || stratum_start_[i]) ? 1 : 0);
    for (std::size_t i = 0; i < m; ++i)
      ss[i] = (i == 0 || ord[positions[i]] != ord[positions[i - 1]]) ? 1 : 0;
  }
  std::vector<std::vector<std::pair<std::uint32_t, double>>> cols(p());
  for (std::size_t j = 0; j < p(); ++j) {
    std::size_t pi = 0, ci = static_cast<std::size_t>(col_ptr_[j]);
    const std::size_t ce = static_cast<std::size_t>(col_ptr_[j + 1]);
    while (pi < m && ci < ce) {
      const std::uint32_t r = static_cast<std::uint32_t>(row_idx_[ci]);
      if (positions[pi] < r) {
        ++pi;
      } else if (positions[pi] > r) {
        ++ci;
      } else {
        cols[j].emplace_back(static_cast<std::uint32_t>(pi), vals_[ci]);
        ++pi;
        while (pi < m && positions[pi] == positions[pi - 1]) {
          cols[j].emplace_back(static_cast<std::uint32_t>(pi), vals_[ci]);
          ++pi;
        }
        ++ci;
      }
    }
  }
  return assemble(std::move(t), std::move(s), std::move(ids), p(), std::move(cols), std::move(ss));
}

gss_dataset* SurvivalDataset::device(int device) const {
  if (!dev_) dev_ = std::make_shared<DeviceCache>();
  std::lock_guard<std::mutex> lock(dev_->mu);
  if (device < 0) throw DomainError("negative device index");
  if (static_cast<std::size_t>(device) >= dev_->by_device.size())
    dev_->by_device.resize(static_cast<std::size_t>(device) + 1, nullptr);
  if (!dev_->by_device[device]) {
    gss_host_dataset h{};
    h.n = static_cast<int64_t>(n());
    h.p = static_cast<int64_t>(p());
    h.times = times_.data();
    std::vector<int32_t> st(status_.begin(), status_.end());
    h.status = st.data();
    h.col_ptr = col_ptr_.data();
    h.row_idx = row_idx_.data();
    h.vals = vals_.data();
    h.col_indicator = nullptr;  // derived: all-ones and density < 25% (src/dataset.cpp:126-157)
    h.stratum_start = has_strata() ? stratum_start_.data() : nullptr;
    gss_dataset* d = nullptr;
    check(gss_dataset_pack(&h, device, &d));
    dev_->by_device[device] = d;
  }
  return dev_->by_device[device];
}

SurvivalDataset dataset_from_coo(const std::vector<double>& times, const std::vector<int>& status,
                                 const std::vector<std::int64_t>& rows,
                                 const std::vector<std::int64_t>& cols,
                                 const std::vector<double>& values, std::size_t n_cols,
                                 const std::vector<std::int64_t>& strata) {
  const std::size_t n = times.size();
  if (status.size() != n) throw DomainError("times and status lengths differ");
  if (rows.size() != cols.size() || rows.size() != values.size())
    throw DomainError("rows, cols, values lengths differ");
  if (!strata.empty() && strata.size() != n) throw DomainError("strata length differs from times");
  if (n >= (std::size_t(1) << 31)) throw DomainError("dataset too large for 32-bit row offsets");
  for (std::size_t i = 0; i < n; ++i) {
    if (!std::isfinite(times[i]) || times[i] < 0.0)
      throw DomainError("observation time must be finite and >= 0");
    if (status[i] != 0 && status[i] != 1 && status[i] != 2)
      throw DomainError("status must be 0, 1 or 2");
  }
  // Device ingestion when a GPU is present (gss_coo_sort: CUB radix sorts,
  // same order, same first-error semantics); SURVSCAN_HOST_INGEST=1 forces
  // the host sort below.
  if (gss_device_count() > 0 && !std::getenv("SURVSCAN_HOST_INGEST")) {
    const std::size_t k = rows.size();
    std::vector<std::int64_t> order(n), col_ptr(n_cols + 1);
    std::vector<std::int32_t> rp(k);
    std::vector<double> vv(k);
    std::int64_t m = 0, err[2] = {-1, -1};
    const int rc = gss_coo_sort(default_device(), static_cast<std::int64_t>(n), times.data(),
                                strata.empty() ? nullptr : strata.data(),
                                static_cast<std::int64_t>(k), rows.data(), cols.data(),
                                values.data(), static_cast<std::int64_t>(n_cols), order.data(),
                                col_ptr.data(), rp.data(), vv.data(), &m, err);
    if (rc == GSS_ERR_INDEX || (rc == GSS_ERR_DOMAIN && err[0] >= 0)) {
      const std::size_t e = static_cast<std::size_t>(err[0]);
      if (rows[e] < 0 || static_cast<std::size_t>(rows[e]) >= n)
        throw IndexError("matrix row " + std::to_string(rows[e]) + " outside [0, " +
                         std::to_string(n) + ")");
      if (cols[e] < 0 || static_cast<std::size_t>(cols[e]) >= n_cols)
        throw IndexError("matrix column " + std::to_string(cols[e]) + " outside [0, " +
                         std::to_string(n_cols) + ")");
      throw DomainError("matrix value must be finite");
    }
    if (rc == GSS_ERR_DUPLICATE)
      throw DuplicateEntryError("matrix cell (" + std::to_string(order[err[0]]) + ", " +
                                std::to_string(err[1]) + ") appears more than once");
    check(rc);
    std::vector<double> t(n);
    std::vector<int> s(n);
    std::vector<std::uint8_t> ss;
    if (!strata.empty()) ss.assign(n, 0);
    for (std::size_t i = 0; i < n; ++i) {
      const std::size_t o = static_cast<std::size_t>(order[i]);
      t[i] = times[o];
      s[i] = status[o];
      if (!strata.empty())
        ss[i] = (i == 0 || strata[o] != strata[static_cast<std::size_t>(order[i - 1])]) ? 1 : 0;
    }
    rp.resize(static_cast<std::size_t>(m));
    vv.resize(static_cast<std::size_t>(m));
    return SurvivalDataset::assemble_csc(std::move(t), std::move(s), std::move(order),
                                         std::move(col_ptr), std::move(rp), std::move(vv),
                                         std::move(ss));
  }
  // (stratum asc,) time desc, row id asc
  std::vector<std::size_t> order(n);
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
    if (!strata.empty() && strata[a] != strata[b]) return strata[a] < strata[b];
    if (times[a] != times[b]) return times[a] > times[b];
    return a < b;
  });
  std::vector<double> t(n);
  std::vector<int> s(n);
  std::vector<std::int64_t> ids(n);
  std::vector<std::uint32_t> pos_of(n);
  std::vector<std::uint8_t> ss;
  if (!strata.empty()) ss.assign(n, 0);
  for (std::size_t i = 0; i < n; ++i) {
    const std::size_t o = order[i];
    t[i] = times[o];
    s[i] = status[o];
    ids[i] = static_cast<std::int64_t>(o);
    pos_of[o] = static_cast<std::uint32_t>(i);
    if (!strata.empty()) ss[i] = (i == 0 || strata[o] != strata[order[i - 1]]) ? 1 : 0;
  }
  std::vector<std::vector<std::pair<std::uint32_t, double>>> cl(n_cols);
  for (std::size_t k = 0; k < rows.size(); ++k) {
    if (rows[k] < 0 || static_cast<std::size_t>(rows[k]) >= n)
      throw IndexError("matrix row " + std::to_string(rows[k]) + " outside [0, " +
                       std::to_string(n) + ")");
    if (cols[k] < 0 || static_cast<std::size_t>(cols[k]) >= n_cols)
      throw IndexError("matrix column " + std::to_string(cols[k]) + " outside [0, " +
                       std::to_string(n_cols) + ")");
    if (!std::isfinite(values[k])) throw DomainError("matrix value must be finite");
    if (values[k] == 0.0) continue;  // absent cells are exact zeros
    cl[static_cast<std::size_t>(cols[k])].emplace_back(pos_of[rows[k]], values[k]);
  }
  for (std::size_t j = 0; j < n_cols; ++j) {
    auto& c = cl[j];
    std::sort(c.begin(), c.end());
    for (std::size_t k = 1; k < c.size(); ++k)
      if (c[k].first == c[k - 1].first)
        throw DuplicateEntryError("matrix cell (" + std::to_string(ids[c[k].first]) + ", " +
                                  std::to_string(j) + ") appears more than once");
  }
  return SurvivalDataset::assemble(std::move(t), std::move(s), std::move(ids), n_cols,
                                   std::move(cl), std::move(ss));
}

// ---- plain-text persistence ------------------------------------------------
// The reference's two formats (src/dataset.cpp:82-117, 363-556), so files move
// between the two implementations unchanged:
//   * sparse COO pair: "row_id,time,status" lines + "row_id,col_id,value"
//     lines, '#' comments, an optional "# cols: P" width declaration
//     (otherwise the width is max col + 1), duplicate cells rejected;
//   * dense CSV with a header naming "time" and "status" anywhere; every other
//     column is a covariate; row ids are the line order.
// Strata are a rebuild feature with no file representation: they are not
// written (a stratified dataset round-trips as unstratified).
namespace {

std::string where(const std::string& path, std::size_t line_no) {
  return path + ":" + std::to_string(line_no);
}

template <class T>
T parse_number(std::string_view tok, const std::string& path, std::size_t line_no,
               const char* what) {
  if (tok.empty()) throw ParseError("missing value at " + where(path, line_no));
  T out{};
  const char* end = tok.data() + tok.size();
  const auto res = std::from_chars(tok.data(), end, out);
  if (res.ec != std::errc{} || res.ptr != end)
    throw ParseError(std::string("bad ") + what + " '" + std::string(tok) + "' at " +
                     where(path, line_no));
  return out;
}

double time_field(std::string_view tok, const std::string& path, std::size_t line_no) {
  const double t = parse_number<double>(tok, path, line_no, "numeric value");
  if (!std::isfinite(t) || t < 0.0)
    throw DomainError("time must be finite and >= 0 at " + where(path, line_no));
  return t;
}

int status_field(std::string_view tok, const std::string& path, std::size_t line_no) {
  const double v = parse_number<double>(tok, path, line_no, "numeric value");
  if (v != 0.0 && v != 1.0 && v != 2.0)
    throw DomainError("status must be 0, 1 or 2 at " + where(path, line_no));
  return static_cast<int>(v);
}

std::vector<std::string_view> fields(std::string_view line) {
  std::vector<std::string_view> out;
  for (std::size_t a = 0;;) {
    const std::size_t b = line.find(',', a);
    out.push_back(line.substr(a, b == std::string_view::npos ? std::string_view::npos : b - a));
    if (b == std::string_view::npos) return out;
    a = b + 1;
  }
}

// payload lines of a text file: '\r' stripped, blank and '#' lines skipped;
// "# cols: P" reported through `declared`
template <class Fn>
void data_lines(const std::string& path, Fn&& fn, std::size_t* declared = nullptr) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open '" + path + "'");
  std::string line;
  for (std::size_t no = 1; std::getline(in, line); ++no) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::string_view v(line);
    const std::size_t k = v.find_first_not_of(" \t");
    if (k == std::string_view::npos) continue;
    v.remove_prefix(k);
    if (v.front() == '#') {
      constexpr std::string_view tag = "# cols:";
      if (declared && v.starts_with(tag)) {
        std::string_view rest = v.substr(tag.size());
        const std::size_t w = rest.find_first_not_of(" \t");
        if (w != std::string_view::npos)
          *declared = static_cast<std::size_t>(
              parse_number<std::int64_t>(rest.substr(w), path, no, "integer"));
      }
      continue;
    }
    fn(std::string_view(line), no);
  }
}

void put_double(std::string& out, double v) {
  char buf[32];
  const int len = std::snprintf(buf, sizeof(buf), "%.17g", v);
  out.append(buf, static_cast<std::size_t>(len));
}

}  // namespace

SurvivalDataset sort_and_block(RawData raw) {
  // ids must be a permutation of [0, n) (src/dataset.cpp:212-262); the
  // builder below orders ties by position, so place each observation at its id
  const std::size_t n = raw.obs.size();
  for (const auto& o : raw.obs) {
    if (!std::isfinite(o.time) || o.time < 0.0)
      throw DomainError("observation time must be finite and >= 0");
    if (o.status != 0 && o.status != 1 && o.status != 2)
      throw DomainError("status must be 0, 1 or 2");
  }
  std::vector<double> t(n);
  std::vector<int> s(n);
  std::vector<unsigned char> seen(n, 0);
  for (const auto& o : raw.obs) {
    if (o.row_id < 0 || static_cast<std::size_t>(o.row_id) >= n)
      throw IndexError("row id " + std::to_string(o.row_id) + " outside [0, " +
                       std::to_string(n) + ")");
    if (seen[static_cast<std::size_t>(o.row_id)]++)
      throw DuplicateEntryError("row id " + std::to_string(o.row_id) + " appears more than once");
    t[static_cast<std::size_t>(o.row_id)] = o.time;
    s[static_cast<std::size_t>(o.row_id)] = o.status;
  }
  std::vector<std::int64_t> r, c;
  std::vector<double> v;
  r.reserve(raw.entries.size());
  c.reserve(raw.entries.size());
  v.reserve(raw.entries.size());
  for (const auto& e : raw.entries) {
    if (e.col >= raw.n_cols)
      throw IndexError("matrix column " + std::to_string(e.col) + " outside [0, " +
                       std::to_string(raw.n_cols) + ")");
    r.push_back(e.row);
    c.push_back(static_cast<std::int64_t>(e.col));
    v.push_back(e.value);
  }
  return dataset_from_coo(t, s, r, c, v, raw.n_cols);
}

SurvivalDataset load_sparse_coo(const std::string& obs_path, const std::string& matrix_path) {
  RawData raw;
  data_lines(obs_path, [&](std::string_view line, std::size_t no) {
    const auto f = fields(line);
    if (f.size() != 3)
      throw ParseError("expected 'row_id,time,status' at " + where(obs_path, no));
    Observation o;
    o.row_id = parse_number<std::int64_t>(f[0], obs_path, no, "integer");
    o.time = time_field(f[1], obs_path, no);
    o.status = status_field(f[2], obs_path, no);
    raw.obs.push_back(o);
  });
  const std::size_t n = raw.obs.size();
  std::unordered_set<std::uint64_t> cells;
  std::size_t declared = 0, width = 0;
  data_lines(
      matrix_path,
      [&](std::string_view line, std::size_t no) {
        const auto f = fields(line);
        if (f.size() != 3)
          throw ParseError("expected 'row_id,col_id,value' at " + where(matrix_path, no));
        const auto row = parse_number<std::int64_t>(f[0], matrix_path, no, "integer");
        const auto col = parse_number<std::int64_t>(f[1], matrix_path, no, "integer");
        const double value = parse_number<double>(f[2], matrix_path, no, "numeric value");
        if (row < 0 || static_cast<std::size_t>(row) >= n)
          throw IndexError("matrix row " + std::to_string(row) + " outside [0, " +
                           std::to_string(n) + ") at " + where(matrix_path, no));
        if (col < 0) throw IndexError("negative column at " + where(matrix_path, no));
        const std::uint64_t key =
            (static_cast<std::uint64_t>(row) << 32) | static_cast<std::uint64_t>(col);
        if (!cells.insert(key).second)
          throw DuplicateEntryError("cell (" + std::to_string(row) + "," + std::to_string(col) +
                                    ") given twice at " + where(matrix_path, no));
        if (!std::isfinite(value))
          throw DomainError("matrix value must be finite at " + where(matrix_path, no));
        width = std::max(width, static_cast<std::size_t>(col) + 1);
        if (value != 0.0) raw.entries.push_back({row, static_cast<std::size_t>(col), value});
      },
      &declared);
  if (declared > 0 && width > declared)
    throw IndexError("matrix column " + std::to_string(width - 1) + " outside declared width " +
                     std::to_string(declared) + " in '" + matrix_path + "'");
  raw.n_cols = std::max(declared, width);
  return sort_and_block(std::move(raw));
}

void write_sparse_coo(const SurvivalDataset& ds, const std::string& obs_path,
                      const std::string& matrix_path) {
  // sorted order with explicit row ids (ids need not be a permutation of
  // [0, n): subset_rows keeps the parent's ids)
  std::string buf;
  {
    std::ofstream fo(obs_path);
    if (!fo) throw ParseError("cannot write '" + obs_path + "'");
    fo << "# row_id,time,status\n";
    for (std::size_t i = 0; i < ds.n(); ++i) {
      buf = std::to_string(ds.row_ids()[i]);
      buf += ',';
      put_double(buf, ds.times()[i]);
      buf += ',';
      buf += std::to_string(ds.status()[i]);
      buf += '\n';
      fo << buf;
    }
    if (!fo) throw ParseError("short write to '" + obs_path + "'");
  }
  std::ofstream fm(matrix_path);
  if (!fm) throw ParseError("cannot write '" + matrix_path + "'");
  fm << "# row_id,col_id,value\n# cols: " << ds.p() << '\n';
  for (std::size_t j = 0; j < ds.p(); ++j)
    for (std::int64_t k = ds.col_ptr()[j]; k < ds.col_ptr()[j + 1]; ++k) {
      buf = std::to_string(ds.row_ids()[static_cast<std::size_t>(ds.row_idx()[k])]);
      buf += ',';
      buf += std::to_string(j);
      buf += ',';
      put_double(buf, ds.values()[static_cast<std::size_t>(k)]);
      buf += '\n';
      fm << buf;
    }
  if (!fm) throw ParseError("short write to '" + matrix_path + "'");
}

SurvivalDataset load_dense_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open '" + path + "'");
  std::string line;
  if (!std::getline(in, line)) throw SchemaError("empty file '" + path + "'");
  if (!line.empty() && line.back() == '\r') line.pop_back();
  const std::string header_line = line;
  const auto head = fields(header_line);
  std::size_t tcol = head.size(), scol = head.size();
  std::vector<std::size_t> xcols;
  for (std::size_t i = 0; i < head.size(); ++i) {
    if (head[i] == "time") {
      if (tcol != head.size()) throw SchemaError("duplicate 'time' column in '" + path + "'");
      tcol = i;
    } else if (head[i] == "status") {
      if (scol != head.size()) throw SchemaError("duplicate 'status' column in '" + path + "'");
      scol = i;
    } else {
      xcols.push_back(i);
    }
  }
  if (tcol == head.size()) throw SchemaError("'" + path + "' has no 'time' column");
  if (scol == head.size()) throw SchemaError("'" + path + "' has no 'status' column");
  RawData raw;
  raw.n_cols = xcols.size();
  for (std::size_t no = 2; std::getline(in, line); ++no) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const auto f = fields(line);
    if (f.size() != head.size())
      throw ParseError("expected " + std::to_string(head.size()) + " cells, got " +
                       std::to_string(f.size()) + " at " + where(path, no));
    Observation o;
    o.row_id = static_cast<std::int64_t>(raw.obs.size());
    o.time = time_field(f[tcol], path, no);
    o.status = status_field(f[scol], path, no);
    for (std::size_t j = 0; j < xcols.size(); ++j) {
      const double x = parse_number<double>(f[xcols[j]], path, no, "numeric value");
      if (!std::isfinite(x)) throw DomainError("covariate must be finite at " + where(path, no));
      if (x != 0.0) raw.entries.push_back({o.row_id, j, x});
    }
    raw.obs.push_back(o);
  }
  return sort_and_block(std::move(raw));
}

void write_dense_csv(const SurvivalDataset& ds, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw ParseError("cannot write '" + path + "'");
  std::string buf = "time,status";
  for (std::size_t j = 0; j < ds.p(); ++j) buf += ",x" + std::to_string(j);
  buf += '\n';
  f << buf;
  for (std::size_t i = 0; i < ds.n(); ++i) {  // sorted order, like the reference
    buf.clear();
    put_double(buf, ds.times()[i]);
    buf += ',';
    buf += std::to_string(ds.status()[i]);
    for (std::size_t j = 0; j < ds.p(); ++j) {
      buf += ',';
      put_double(buf, ds.covariate(i, j));
    }
    buf += '\n';
    f << buf;
  }
  if (!f) throw ParseError("short write to '" + path + "'");
}

}  // namespace survscan
