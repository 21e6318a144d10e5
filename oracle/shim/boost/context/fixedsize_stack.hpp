// Boost.Context stand-in (see continuation.hpp): stack size is ignored.
#pragma once
#include <cstddef>
namespace boost {
namespace context {
struct fixedsize_stack {
    explicit fixedsize_stack(std::size_t = 0) {}
};
}  // namespace context
}  // namespace boost
