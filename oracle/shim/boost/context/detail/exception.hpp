// Boost.Context stand-in (see ../continuation.hpp).
#pragma once
namespace boost {
namespace context {
namespace detail {
struct forced_unwind {};
}  // namespace detail
}  // namespace context
}  // namespace boost
