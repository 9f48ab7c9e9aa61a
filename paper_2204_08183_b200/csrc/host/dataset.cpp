// dataset.cpp — sorted host layout, COO ingestion, subsetting, persistence and
// the lazily created device copy of a SurvivalDataset.
#include "survscan/dataset.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <numeric>
#include <sstream>

#include "../../../include/gss.h"
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

// ---- plain-text persistence -------------------------------------------------
SurvivalDataset load_sparse_coo(const std::string& obs_path, const std::string& matrix_path) {
  std::ifstream fo(obs_path), fm(matrix_path);
  if (!fo) throw ParseError("cannot open " + obs_path);
  if (!fm) throw ParseError("cannot open " + matrix_path);
  std::vector<double> t;
  std::vector<int> s;
  std::string line;
  std::size_t n_cols = 0;
  while (std::getline(fo, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream is(line);
    double ti;
    int si;
    if (!(is >> ti >> si)) throw ParseError("bad observation line: " + line);
    t.push_back(ti);
    s.push_back(si);
  }
  std::vector<std::int64_t> r, c;
  std::vector<double> v;
  while (std::getline(fm, line)) {
    if (line.empty()) continue;
    if (line[0] == '#') {
      std::istringstream is(line.substr(1));
      std::string key;
      if (is >> key && key == "n_cols") is >> n_cols;
      continue;
    }
    std::istringstream is(line);
    std::int64_t ri, ci;
    double vi;
    if (!(is >> ri >> ci >> vi)) throw ParseError("bad matrix line: " + line);
    r.push_back(ri);
    c.push_back(ci);
    v.push_back(vi);
  }
  return dataset_from_coo(t, s, r, c, v, n_cols);
}

void write_sparse_coo(const SurvivalDataset& ds, const std::string& obs_path,
                      const std::string& matrix_path) {
  // rows are written in original row-id order, so a reload sorts identically
  std::vector<std::size_t> pos_of(ds.n());
  for (std::size_t i = 0; i < ds.n(); ++i) pos_of[static_cast<std::size_t>(ds.row_ids()[i])] = i;
  std::ofstream fo(obs_path), fm(matrix_path);
  if (!fo || !fm) throw ParseError("cannot write dataset files");
  fo.precision(17);
  fm.precision(17);
  for (std::size_t id = 0; id < ds.n(); ++id)
    fo << ds.times()[pos_of[id]] << ' ' << ds.status()[pos_of[id]] << '\n';
  fm << "# n_cols " << ds.p() << '\n';
  for (std::size_t j = 0; j < ds.p(); ++j)
    for (std::int64_t k = ds.col_ptr()[j]; k < ds.col_ptr()[j + 1]; ++k)
      fm << ds.row_ids()[static_cast<std::size_t>(ds.row_idx()[k])] << ' ' << j << ' '
         << ds.values()[static_cast<std::size_t>(k)] << '\n';
}

SurvivalDataset load_dense_csv(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw ParseError("cannot open " + path);
  std::vector<double> t;
  std::vector<int> s;
  std::vector<std::int64_t> r, c;
  std::vector<double> v;
  std::string line;
  std::size_t n_cols = 0, row = 0;
  bool header = true;
  while (std::getline(f, line)) {
    if (line.empty()) continue;
    std::vector<std::string> cells;
    std::stringstream ss(line);
    std::string cell;
    while (std::getline(ss, cell, ',')) cells.push_back(cell);
    if (header) {
      header = false;
      if (cells.size() < 2) throw SchemaError("csv needs time,status,x0,... columns");
      n_cols = cells.size() - 2;
      continue;
    }
    if (cells.size() != n_cols + 2) throw ParseError("ragged csv row " + std::to_string(row));
    try {
      t.push_back(std::stod(cells[0]));
      s.push_back(std::stoi(cells[1]));
      for (std::size_t j = 0; j < n_cols; ++j) {
        const double x = std::stod(cells[2 + j]);
        if (x != 0.0) {
          r.push_back(static_cast<std::int64_t>(row));
          c.push_back(static_cast<std::int64_t>(j));
          v.push_back(x);
        }
      }
    } catch (const std::logic_error&) {
      throw ParseError("bad csv value in row " + std::to_string(row));
    }
    ++row;
  }
  return dataset_from_coo(t, s, r, c, v, n_cols);
}

void write_dense_csv(const SurvivalDataset& ds, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw ParseError("cannot write " + path);
  f.precision(17);
  f << "time,status";
  for (std::size_t j = 0; j < ds.p(); ++j) f << ",x" << j;
  f << '\n';
  std::vector<std::size_t> pos_of(ds.n());
  for (std::size_t i = 0; i < ds.n(); ++i) pos_of[static_cast<std::size_t>(ds.row_ids()[i])] = i;
  for (std::size_t id = 0; id < ds.n(); ++id) {
    const std::size_t i = pos_of[id];
    f << ds.times()[i] << ',' << ds.status()[i];
    for (std::size_t j = 0; j < ds.p(); ++j) f << ',' << ds.covariate(i, j);
    f << '\n';
  }
}

}  // namespace survscan
