// oracle/trace_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI veneer over the UNMODIFIED reference trace checker: seqpar::read_trace and
// seqpar::validate_trace (simhost.cpp:567-686), compiled with the reference sources where
// they lie (oracle/Makefile -> oracle/_ref/libseqpar_trace.so, nlohmann json.hpp from the
// venv's cudnn_frontend tree as SURVEY.md s0 records).  tests/ feed it the Event JSONL the
// GPU layer runtime emits (spava_host_trace_read) to check the overlap schedule with the
// reference's own happens-before rules.
#include <cstring>
#include <sstream>
#include <string>

#include "seqpar/simhost.hpp"

extern "C" int ref_validate_trace_jsonl(const char* jsonl, char* out, int cap) {
  try {
    std::istringstream is(jsonl);
    seqpar::EventTrace t = seqpar::read_trace(is);
    const auto v = seqpar::validate_trace(t);
    std::string all;
    for (const auto& s : v) all += s + "\n";
    if (out && cap > 0) {
      std::strncpy(out, all.c_str(), cap - 1);
      out[cap - 1] = 0;
    }
    return static_cast<int>(v.size());
  } catch (const std::exception& e) {
    if (out && cap > 0) {
      std::strncpy(out, e.what(), cap - 1);
      out[cap - 1] = 0;
    }
    return -1;
  }
}
