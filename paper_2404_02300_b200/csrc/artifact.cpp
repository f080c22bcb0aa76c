// Artifact reader — see artifact.hpp.  Plain C++ (no reference code): bulk
// reads instead of the reference's buffered per-record streams and row seeks.
#include "artifact.hpp"

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <nlohmann/json.hpp>

namespace fs = std::filesystem;

namespace catgnn {

uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t seed_for(uint64_t seed, uint64_t stream) { return mix64(seed ^ mix64(stream + 0x51ed2701)); }

namespace {

[[noreturn]] void corrupt(const std::string& what) { throw DataError("corrupt artifact: " + what); }

bool slurp(const std::string& path, std::string& out) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? (size_t)n : 0);
  size_t got = n > 0 ? std::fread(out.data(), 1, (size_t)n, f) : 0;
  std::fclose(f);
  return got == out.size();
}

// Iterate the lines of a text buffer, handling a trailing '\r' like the
// reference's getline loops.
template <typename Fn>
void for_lines(const std::string& buf, Fn&& fn) {
  size_t pos = 0;
  while (pos < buf.size()) {
    size_t nl = buf.find('\n', pos);
    size_t end = nl == std::string::npos ? buf.size() : nl;
    size_t e = end;
    if (e > pos && buf[e - 1] == '\r') --e;
    fn(buf.data() + pos, buf.data() + e);
    pos = nl == std::string::npos ? buf.size() : nl + 1;
  }
}

void read_binary_edges(const std::string& path, std::vector<uint64_t>& out, bool add_reverse) {
  std::error_code ec;
  if (!fs::is_regular_file(path, ec)) throw DataError("edge file not readable: " + path);
  std::string buf;
  if (!slurp(path, buf)) throw DataError("cannot open edge file: " + path);
  size_t off = 0;
  if (buf.size() >= 4 && std::memcmp(buf.data(), "EDG1", 4) == 0) off = 4;
  if ((buf.size() - off) % 16 != 0)
    throw DataError("binary edge file has truncated record: " + path);
  const size_t n = (buf.size() - off) / 16;
  const size_t base = out.size();
  if (!add_reverse) {
    out.resize(base + 2 * n);
    std::memcpy(out.data() + base, buf.data() + off, n * 16);
    return;
  }
  out.reserve(base + 4 * n);
  for (size_t k = 0; k < n; ++k) {
    uint64_t u, v;
    std::memcpy(&u, buf.data() + off + 16 * k, 8);
    std::memcpy(&v, buf.data() + off + 16 * k + 8, 8);
    out.push_back(u);
    out.push_back(v);
    if (u != v) {
      out.push_back(v);
      out.push_back(u);
    }
  }
}

void read_text_edges(const std::string& path, std::vector<uint64_t>& out, bool add_reverse) {
  std::error_code ec;
  if (!fs::is_regular_file(path, ec)) throw DataError("edge file not readable: " + path);
  std::string buf;
  if (!slurp(path, buf)) throw DataError("cannot open edge file: " + path);
  for_lines(buf, [&](const char* b, const char* e) {
    if (b == e || *b == '#') return;
    uint64_t u = 0, v = 0;
    auto r1 = std::from_chars(b, e, u);
    if (r1.ec != std::errc() || r1.ptr == e || *r1.ptr != '\t') return;  // malformed: skipped
    auto r2 = std::from_chars(r1.ptr + 1, e, v);
    if (r2.ec != std::errc() || r2.ptr != e) return;
    out.push_back(u);
    out.push_back(v);
    if (add_reverse && u != v) {
      out.push_back(v);
      out.push_back(u);
    }
  });
}

}  // namespace

uint8_t parse_role(const std::string& name) {
  if (name == "train") return 1;
  if (name == "val") return 2;
  if (name == "test") return 3;
  if (name == "none" || name.empty()) return 0;
  throw DataError("unknown node role: " + name);
}

void read_edge_stream(const std::string& path, bool add_reverse, std::vector<uint64_t>& out) {
  if (fs::path(path).extension() == ".bin") read_binary_edges(path, out, add_reverse);
  else read_text_edges(path, out, add_reverse);
}

FeatureFile read_feature_header(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open feature file: " + path);
  char magic[4];
  FeatureFile info;
  uint32_t dtype = 0;
  in.read(magic, 4);
  in.read(reinterpret_cast<char*>(&info.rows), 8);
  in.read(reinterpret_cast<char*>(&info.dim), 4);
  in.read(reinterpret_cast<char*>(&dtype), 4);
  if (!in || std::memcmp(magic, "FEA1", 4) != 0) throw DataError("bad feature header: " + path);
  if (dtype != 1) throw DataError("unsupported feature dtype: " + path);
  if (fs::file_size(path) != 20 + info.rows * (uint64_t)info.dim * 4)
    throw DataError("feature file size mismatch: " + path);
  return info;
}

void read_feature_matrix(const std::string& path, std::vector<float>& out, FeatureFile* info) {
  FeatureFile h = read_feature_header(path);
  out.resize(h.rows * (size_t)h.dim);
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw DataError("cannot open feature file: " + path);
  std::fseek(f, 20, SEEK_SET);
  size_t got = out.empty() ? 0 : std::fread(out.data(), 4, out.size(), f);
  std::fclose(f);
  if (got != out.size()) throw DataError("short feature read: " + path);
  if (info) *info = h;
}

void open_artifact(catgnn_artifact_s* a, const std::string& dir) {
  a->dir = dir;
  std::string text;
  if (!slurp((fs::path(dir) / "manifest.json").string(), text))
    throw DataError("missing manifest (incomplete artifact): " + dir);
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    corrupt(std::string("unparseable manifest: ") + e.what());
  }
  try {
    if (j.at("schema").get<int>() != 1) throw DataError("unsupported manifest schema");
    a->num_partitions = j.at("num_partitions").get<uint32_t>();
    a->num_nodes = j.at("num_nodes").get<uint64_t>();
    a->num_edges = j.at("num_edges").get<uint64_t>();
    a->feature_dim = j.at("feature_dim").get<uint32_t>();
    a->manifest_rf = j.at("replication_factor").get<double>();
    a->has_features = j.at("has_features").get<bool>();
    a->has_meta = j.at("has_meta").get<bool>();
    const auto& params = j.at("params");
    a->input = params.value("input", std::string{});
    a->features = params.value("features", std::string{});
    a->add_reverse = params.value("add_reverse", false);
    for (const auto& row : j.at("partitions")) {
      PartTable t;
      t.dir = row.at("dir").get<std::string>();
      t.m_nodes = row.at("nodes").get<uint64_t>();
      t.m_owned = row.at("owned").get<uint64_t>();
      t.m_edges = row.at("edges").get<uint64_t>();
      a->parts.push_back(std::move(t));
    }
  } catch (const nlohmann::json::exception& e) {
    throw DataError(std::string("bad manifest: ") + e.what());
  }
  if (a->parts.size() != a->num_partitions) corrupt("partition list length mismatch");
  uint64_t owned_total = 0;
  for (auto& t : a->parts) {
    fs::path pd = fs::path(dir) / t.dir;
    read_binary_edges((pd / "edges.bin").string(), t.edges, false);
    if (t.edges.size() / 2 != t.m_edges) corrupt("edge count mismatch in " + t.dir);
    std::string nodes;
    if (!slurp((pd / "nodes.tsv").string(), nodes)) corrupt("missing node table in " + t.dir);
    uint64_t owned = 0;
    for_lines(nodes, [&](const char* b, const char* e) {
      if (b == e) return;
      uint64_t node = 0;
      int flag = 0;
      auto r1 = std::from_chars(b, e, node);
      if (r1.ec != std::errc() || r1.ptr == e || *r1.ptr != '\t') corrupt("bad node record in " + t.dir);
      auto r2 = std::from_chars(r1.ptr + 1, e, flag);
      if (r2.ec != std::errc() || r2.ptr == e || *r2.ptr != '\t') corrupt("bad node record in " + t.dir);
      t.ext.push_back(node);
      t.owner.push_back(flag != 0 ? 1 : 0);
      t.role.push_back(parse_role(std::string(r2.ptr + 1, e)));
      owned += flag != 0 ? 1 : 0;
    });
    if (t.ext.size() != t.m_nodes) corrupt("node count mismatch in " + t.dir);
    if (owned != t.m_owned) corrupt("owner count mismatch in " + t.dir);
    if (a->has_features) {
      FeatureFile info = read_feature_header((pd / "features.bin").string());
      if (info.rows != t.m_nodes || info.dim != a->feature_dim)
        corrupt("feature shape mismatch in " + t.dir);
    }
    owned_total += owned;
  }
  if (owned_total != a->num_nodes) corrupt("ownership does not cover the node set");
  if (a->has_meta) {
    std::string lab;
    std::string path = (fs::path(dir) / "labels.tsv").string();
    if (!slurp(path, lab)) throw DataError("cannot open node meta file: " + path);
    for_lines(lab, [&](const char* b, const char* e) {
      if (b == e || *b == '#') return;
      uint64_t node = 0;
      int32_t label = 0;
      auto r1 = std::from_chars(b, e, node);
      if (r1.ec != std::errc() || r1.ptr == e || *r1.ptr != '\t')
        throw DataError("bad node meta line: " + std::string(b, e));
      auto r2 = std::from_chars(r1.ptr + 1, e, label);
      if (r2.ec != std::errc() || r2.ptr == e || *r2.ptr != '\t')
        throw DataError("bad node meta line: " + std::string(b, e));
      a->meta.push_back(MetaEntry{node, label, parse_role(std::string(r2.ptr + 1, e))});
    });
    // NodeMetaMap is a map: a later line for the same node overwrites (store.cpp:152)
    std::stable_sort(a->meta.begin(), a->meta.end(),
                     [](const MetaEntry& x, const MetaEntry& y) { return x.node < y.node; });
    std::vector<MetaEntry> dedup;
    for (size_t i = 0; i < a->meta.size(); ++i) {
      if (!dedup.empty() && dedup.back().node == a->meta[i].node) dedup.back() = a->meta[i];
      else dedup.push_back(a->meta[i]);
    }
    a->meta.swap(dedup);
  }
}

}  // namespace catgnn

const catgnn::MetaEntry* catgnn_artifact_s::find_meta(uint64_t node) const {
  auto it = std::lower_bound(meta.begin(), meta.end(), node,
                             [](const catgnn::MetaEntry& m, uint64_t n) { return m.node < n; });
  return (it != meta.end() && it->node == node) ? &*it : nullptr;
}

double catgnn_artifact_s::replication_factor() const {
  if (num_nodes == 0) throw catgnn::DataError("replication factor undefined for an empty graph");
  uint64_t total = 0;
  for (const auto& p : parts) total += p.ext.size();
  return static_cast<double>(total) / static_cast<double>(num_nodes);
}
