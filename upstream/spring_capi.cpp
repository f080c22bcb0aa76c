// Upstream partitioner used to PREPARE benchmark inputs: the reference's own
// SPRING (proj/src/spring.cpp) and degree pass (proj/src/edge_stream.cpp),
// compiled unmodified from /root/reference by upstream/Makefile.  The north
// star consumes "the reference's SPRING edge-to-partition assignment
// unchanged"; this wrapper only exposes that assignment as a plain array.  It
// runs before any timed region and is never part of the training path.
#include <cstdint>
#include <exception>
#include <string>

#include "gnnpart/edge_stream.hpp"
#include "gnnpart/spring.hpp"

using namespace gnnpart;

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* spring_last_error() { return g_err.c_str(); }

// home_by_ext[ext] = SPRING partition of every node seen in the stream
// (ids must be < capacity).  Returns 0, 2 (ConfigError), 3 (DataError) or 4.
int spring_homes(const char* input, int add_reverse, std::uint32_t partitions, double beta,
                 std::uint64_t tau_vol, std::uint64_t seed, std::uint32_t* home_by_ext,
                 std::uint64_t capacity, std::uint64_t* tau_used) {
  try {
    std::string in(input);
    EdgeFormat fmt = in.size() > 4 && in.substr(in.size() - 4) == ".bin" ? EdgeFormat::binary_u64
                                                                         : EdgeFormat::text_tsv;
    EdgeStream stream(in, fmt, add_reverse != 0);
    GraphIndex index = compute_degrees(stream);
    SpringParams sp;
    sp.partitions = partitions;
    sp.beta = beta;
    sp.tau_vol = tau_vol;
    sp.seed = seed;
    if (tau_used) *tau_used = tau_vol ? tau_vol : default_tau_vol(index.num_edges, partitions);
    PartitionAssignment pa = spring_partition(stream, index, sp);
    for (NodeId v = 0; v < index.num_nodes(); ++v) {
      ExtNodeId e = index.dense_to_ext[v];
      if (e >= capacity) throw ConfigError("home buffer too small");
      home_by_ext[e] = pa.node_part[v];
    }
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}
}
