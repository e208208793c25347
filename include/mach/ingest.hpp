// Drop-in mirror of /root/reference/proj/include/mach/ingest.hpp:11-55, plus
// the streaming sample-on-arrival form of it (PAPER Remark 2).
// The name -> axis maps and the CSV text are host work; the cell means, the
// carry-forward fill and the sampling run on the B200 (mach_stream_*).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "mach/sampling.hpp"
#include "mach/tensor.hpp"

namespace mach {

struct MeasurementRecord {
    std::string machine_id;
    std::string metric;
    std::int64_t timestamp = 0;  // epoch seconds
    double value = 0.0;          // must be finite
};

enum class MissingPolicy { zero, carry_forward };

struct TensorBuildSpec {
    std::int64_t time_bucket_seconds = 300;
    MissingPolicy missing_policy = MissingPolicy::zero;
    std::vector<std::string> machine_order;
    std::vector<std::string> metric_order;
};

struct IngestResult {
    DenseTensor tensor;
    std::vector<std::string> machines;
    std::vector<std::string> metrics;
    std::vector<std::int64_t> bucket_starts;
};

IngestResult ingest(const std::vector<MeasurementRecord>& records, const TensorBuildSpec& spec);
std::vector<MeasurementRecord> read_measurements_csv(const std::string& path);
void write_measurements_csv(const std::vector<MeasurementRecord>& records, const std::string& path);

/// Sample-on-arrival: a machines x metrics x time tensor that grows along
/// time.  Records are handed over one closed time window at a time (any order
/// inside the window); each window is binned, filled and sampled on the
/// device, and the sampled tensor so far is identical to
/// sparsify(ingest(all records so far).tensor, cfg).  The axes are fixed up
/// front (explicit orderings, as with TensorBuildSpec's).
class StreamingIngest {
public:
    StreamingIngest(std::vector<std::string> machines, std::vector<std::string> metrics, std::int64_t first_bucket_start,
                    std::int64_t time_bucket_seconds, int capacity_buckets, MissingPolicy policy,
                    const SparsifyConfig& cfg);
    ~StreamingIngest();
    StreamingIngest(const StreamingIngest&) = delete;
    StreamingIngest& operator=(const StreamingIngest&) = delete;
    /// Appends `buckets` time buckets following the ones seen so far; every
    /// record must fall inside them.
    void append_window(const std::vector<MeasurementRecord>& records, int buckets);
    std::int64_t buckets() const;
    std::int64_t nnz() const;
    SparseTensor sampled() const;
    /// HOOI on the sampled tensor seen so far, without leaving the device.
    TuckerModel hooi(const std::vector<int>& ranks, const HooiConfig& cfg) const;

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace mach
