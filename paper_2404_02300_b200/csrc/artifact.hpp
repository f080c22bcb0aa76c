// Host reader of the reference's on-disk partition artifact (the contract the
// training path consumes):
//   manifest.json                 store.cpp:177-220 (written last = commit point)
//   part-<i>/edges.bin            "EDG1" + LE u64 pairs, edge_stream.cpp:174-183
//   part-<i>/nodes.tsv            ext \t owner \t role, store.cpp:241-245
//   part-<i>/features.bin         FEA1 (20-byte header + f32 rows), store.cpp:15-47
//   labels.tsv                    node \t label \t role, store.cpp:118-154
// Count verification and error messages follow read_partitions
// (store.cpp:269-333).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace catgnn {

struct PartTable {
  std::string dir;
  uint64_t m_nodes = 0, m_owned = 0, m_edges = 0;  // manifest counts
  std::vector<uint64_t> edges;                    // 2*E external ids, stream order
  std::vector<uint64_t> ext;                      // node table, ascending ext id
  std::vector<uint8_t> owner, role;
};

struct MetaEntry {
  uint64_t node;
  int32_t label;
  uint8_t role;
};

struct FeatureFile {
  uint64_t rows = 0;
  uint32_t dim = 0;
};

// FEA1 header check (store.cpp:31-47).
FeatureFile read_feature_header(const std::string& path);
// Whole-file read of a FEA1 matrix (rows x dim f32) into out.
void read_feature_matrix(const std::string& path, std::vector<float>& out, FeatureFile* info);
// Edge stream (TSV or EDG1 by extension), add_reverse as EdgeReader::next
// (edge_stream.cpp:138-148).  Appends pairs to out.
void read_edge_stream(const std::string& path, bool add_reverse, std::vector<uint64_t>& out);
uint8_t parse_role(const std::string& s);
// common.hpp:27-39 (splitmix64 finalizer and per-stream seed derivation).
uint64_t mix64(uint64_t x);
uint64_t seed_for(uint64_t seed, uint64_t stream);

}  // namespace catgnn

struct catgnn_artifact_s {
  std::string dir;
  uint32_t num_partitions = 0;
  uint64_t num_nodes = 0, num_edges = 0;
  uint32_t feature_dim = 0;
  bool has_features = false, has_meta = false, add_reverse = false;
  double manifest_rf = 0.0;
  std::string input, features;  // params.input / params.features
  std::vector<catgnn::PartTable> parts;
  std::vector<catgnn::MetaEntry> meta;  // sorted by node
  const catgnn::MetaEntry* find_meta(uint64_t node) const;
  double replication_factor() const;
};

namespace catgnn {
void open_artifact(catgnn_artifact_s* a, const std::string& dir);
}
