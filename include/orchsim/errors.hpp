// orchsim error classes -- the exception contract of the reference API
// (/root/reference/proj/include/orchsim/errors.hpp). The B200 library reports
// them through C-ABI return codes (include/orchsim_capi.h) that the host
// adapter (paper_2503_23830_b200/csrc/host/runtime.cpp) maps back to these.
#pragma once

#include <stdexcept>
#include <string>

namespace orchsim {

struct ConfigError : std::runtime_error {        // ORCH_CONFIG_ERROR
  using std::runtime_error::runtime_error;
};
struct VerificationError : std::runtime_error {  // verification sweeps (not on this path)
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {            // trace / report I/O (not on this path)
  using std::runtime_error::runtime_error;
};
struct SizeCapError : std::invalid_argument {    // ORCH_SIZE_CAP
  using std::invalid_argument::invalid_argument;
};

}  // namespace orchsim
