// Force-included (-include) when compiling the UNMODIFIED reference sources
// under /root/reference/proj (and the reference's own tests) into oracle/_ref.
//
// Why: the reference calls `apply(re, vec)` unqualified inside namespace
// orchsim (proj/src/orchestrator.cpp:467, proj/src/verify.cpp:252-256,
// proj/tests/test_balancers.cpp:35). With libstdc++ 13 argument-dependent
// lookup also finds the template std::apply through std::vector, which wins
// overload resolution for non-const / rvalue arguments and then fails hard
// ("incomplete type std::tuple_size<std::vector<MiniBatch>>").
//
// Fix without touching the reference: declare non-template overloads for every
// {R&, const R&, R&&} x {V&, const V&, V&&} combination except const/const
// (which the reference declares itself, proj/include/orchsim/core.hpp:121).
// A non-template exact match beats the template in overload resolution.
#pragma once

#include <utility>
#include <vector>

#include "orchsim/core.hpp"

namespace orchsim {

#define ORCH_ADL_FWD(RQ, VQ)                                                        \
  inline std::vector<MiniBatch> apply(Rearrangement RQ re, std::vector<MiniBatch> VQ b) { \
    return apply(static_cast<const Rearrangement&>(re),                            \
                 static_cast<const std::vector<MiniBatch>&>(b));                   \
  }

ORCH_ADL_FWD(&, &)
ORCH_ADL_FWD(&, &&)
ORCH_ADL_FWD(&, const&)
ORCH_ADL_FWD(const&, &)
ORCH_ADL_FWD(const&, &&)
ORCH_ADL_FWD(&&, &)
ORCH_ADL_FWD(&&, &&)
ORCH_ADL_FWD(&&, const&)

#undef ORCH_ADL_FWD

}  // namespace orchsim
