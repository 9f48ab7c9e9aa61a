// survscan/dataset.hpp — the reference's in-memory dataset contract
// (/root/reference/proj/include/survscan/dataset.hpp:14-111): rows sorted by
// (stratum asc,) time desc, original row id asc; CSC columns over sorted
// positions.  The device copy (gss_dataset_pack) is created lazily per device
// and shared by every Engine on that device.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <vector>

struct gss_dataset;

namespace survscan {

// Raw input of the reference's dataset builder (dataset.hpp:16-20, 56-61).
struct Observation {
  double time = 0.0;
  int status = 0;
  std::int64_t row_id = 0;
};

struct RawData {
  std::vector<Observation> obs;
  std::size_t n_cols = 0;
  struct Entry {
    std::int64_t row;  // refers to Observation::row_id
    std::size_t col;
    double value;
  };
  std::vector<Entry> entries;
};

class SurvivalDataset {
 public:
  SurvivalDataset() = default;
  SurvivalDataset(const SurvivalDataset& o);
  SurvivalDataset& operator=(const SurvivalDataset& o);
  SurvivalDataset(SurvivalDataset&&) noexcept;
  SurvivalDataset& operator=(SurvivalDataset&&) noexcept;
  ~SurvivalDataset();

  std::size_t n() const { return times_.size(); }
  std::size_t p() const { return col_ptr_.empty() ? 0 : col_ptr_.size() - 1; }
  std::size_t n_events() const { return n_events_; }
  bool has_competing() const { return has_competing_; }
  bool has_strata() const { return !stratum_start_.empty(); }
  std::size_t nnz_total() const { return row_idx_.size(); }
  std::uint64_t content_hash() const;

  const std::vector<double>& times() const { return times_; }
  const std::vector<int>& status() const { return status_; }
  const std::vector<std::int64_t>& row_ids() const { return row_ids_; }
  const std::vector<std::int64_t>& col_ptr() const { return col_ptr_; }
  const std::vector<std::int32_t>& row_idx() const { return row_idx_; }
  const std::vector<double>& values() const { return vals_; }
  const std::vector<std::uint8_t>& stratum_start() const { return stratum_start_; }
  double covariate(std::size_t i, std::size_t j) const;

  // src/dataset.cpp:268-322: rows at non-decreasing sorted positions (repeats
  // allowed with fresh ids, e.g. bootstrap resamples).
  SurvivalDataset subset_rows(const std::vector<std::uint32_t>& positions,
                              bool fresh_row_ids) const;
  SurvivalDataset subset_rows(std::span<const std::uint32_t> positions,
                              bool fresh_row_ids = false) const {
    return subset_rows(std::vector<std::uint32_t>(positions.begin(), positions.end()),
                       fresh_row_ids);
  }

  // Device-resident packed copy (created on first use; thread safe).
  gss_dataset* device(int device) const;

  // Build from sorted observations + per-column (position, value) lists.
  // sorted layout already in CSC form (device ingestion, gss_coo_sort)
  static SurvivalDataset assemble_csc(std::vector<double> times, std::vector<int> status,
                                      std::vector<std::int64_t> row_ids,
                                      std::vector<std::int64_t> col_ptr,
                                      std::vector<std::int32_t> row_idx, std::vector<double> vals,
                                      std::vector<std::uint8_t> stratum_start = {});
  static SurvivalDataset assemble(std::vector<double> times, std::vector<int> status,
                                  std::vector<std::int64_t> row_ids, std::size_t n_cols,
                                  std::vector<std::vector<std::pair<std::uint32_t, double>>> cols,
                                  std::vector<std::uint8_t> stratum_start = {});

 private:
  std::vector<double> times_;
  std::vector<int> status_;
  std::vector<std::int64_t> row_ids_;
  std::vector<std::int64_t> col_ptr_;
  std::vector<std::int32_t> row_idx_;
  std::vector<double> vals_;
  std::vector<std::uint8_t> stratum_start_;
  std::size_t n_events_ = 0;
  bool has_competing_ = false;
  struct DeviceCache;
  mutable std::shared_ptr<DeviceCache> dev_;
};

// sort_and_block (src/dataset.cpp:212-262): validate, sort by (stratum asc,)
// time desc, row id asc; absent cells are exact zeros.  `strata` optional
// (one integer per observation; a rebuild feature, SPEC.md:174 non-goal).
SurvivalDataset dataset_from_coo(const std::vector<double>& times, const std::vector<int>& status,
                                 const std::vector<std::int64_t>& rows,
                                 const std::vector<std::int64_t>& cols,
                                 const std::vector<double>& values, std::size_t n_cols,
                                 const std::vector<std::int64_t>& strata = {});

// sort_and_block (src/dataset.cpp:212-262): row ids must be a permutation of
// [0, n); ties in time keep ascending row id.
SurvivalDataset sort_and_block(RawData raw);

// Plain-text persistence in the reference's formats (src/dataset.cpp:363-556):
// "row_id,time,status" + "row_id,col_id,value" (with "# cols: P"), dense CSV
// with "time" and "status" header columns.
SurvivalDataset load_sparse_coo(const std::string& obs_path, const std::string& matrix_path);
void write_sparse_coo(const SurvivalDataset& ds, const std::string& obs_path,
                      const std::string& matrix_path);
SurvivalDataset load_dense_csv(const std::string& path);
void write_dense_csv(const SurvivalDataset& ds, const std::string& path);

}  // namespace survscan
