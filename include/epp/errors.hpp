// epp-b200 planner: exception taxonomy.
//
// Drop-in for the reference's error header (reference:
// proj/include/epp/errors.hpp:11-42).  Every planner entry point reports
// failures by throwing one of these; the C ABI (include/epp_c.h) maps each
// class to a distinct integer code.
#pragma once

#include <stdexcept>
#include <string>

namespace epp {

// Root of the hierarchy; thrown bare for internal invariant failures
// (schedule deadlock, simplex iteration cap, packing retry).
struct Error : std::runtime_error {
    explicit Error(const std::string& what_arg) : std::runtime_error(what_arg) {}
};

struct ConfigError : Error {      // invalid cluster / model / cost document
    using Error::Error;
};
struct ParseError : Error {       // malformed workload / plan / trace input
    using Error::Error;
};
struct InfeasibleError : Error {  // memory constraints admit no plan
    using Error::Error;
};
struct IoError : Error {          // filesystem failure
    using Error::Error;
};
struct ContractError : Error {    // caller broke a documented precondition
    using Error::Error;
};
struct FitError : Error {         // cost regression is rank deficient
    using Error::Error;
};

}  // namespace epp
