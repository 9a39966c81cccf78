// `ising-model v1` text documents <-> HostModel.  The format is the reference's
// (ref: proj/include/isingmc/model_io.hpp:10-20): a header line, `spins <n>`, optionally
// `layers <L> <P>`, one `h <i> <hex-float>` line per non-zero field and one
// `edge <i> <j> <hex-float> <space|tau>` line per undirected edge with i < j.  Hex-float literals make
// the round trip bit-exact.  Loading canonicalises the adjacency (space edges by target, then tau
// edges next layer first) and runs the structural checks of finalize_model.
#pragma once

#include <string>
#include <string_view>

#include "host_model.hpp"

namespace isingb200 {

struct ParseError : Error {  // maps to ISING_ERR_PARSE; message starts "line N: " (ref: model_io.cpp:28-30)
    using Error::Error;
};
struct IoError : Error {  // maps to ISING_ERR_IO
    using Error::Error;
};

std::string model_to_text(const HostModel& m);
HostModel model_from_text(std::string_view text);
void save_model_text(const HostModel& m, const std::string& path);
HostModel load_model_text(const std::string& path);

}  // namespace isingb200
