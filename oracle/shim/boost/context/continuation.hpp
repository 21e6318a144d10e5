// Minimal Boost.Context stand-in used ONLY to compile the read-only reference
// (proj/src/fabric.cpp:12-14, :197-198, :428-461) into oracle/_ref. Boost is not in
// this image. Each "fiber" is an OS thread; control is handed back and forth
// with binary semaphores so exactly one side runs at a time, which preserves
// the deterministic round-robin scheduling the reference fabric relies on.
//
// Contract honoured:
//   * callcc(allocator_arg, stack, fn) enters fn(sink) at once and returns when
//     fn first calls sink.resume();
//   * handle.resume() runs the fiber until its next sink.resume(), and returns
//     an empty continuation when fn returns;
//   * destroying a suspended handle unwinds the fiber by throwing
//     detail::forced_unwind out of its pending sink.resume().
// Test infrastructure, not product code.
#pragma once

#include <memory>
#include <semaphore>
#include <thread>
#include <utility>

#include "boost/context/detail/exception.hpp"
#include "boost/context/fixedsize_stack.hpp"

namespace boost {
namespace context {

namespace shim {
struct FiberState {
    std::thread thread;
    std::binary_semaphore to_fiber{0};
    std::binary_semaphore to_main{0};
    bool finished = false;
    bool unwinding = false;
};
}  // namespace shim

class continuation {
  public:
    continuation() = default;
    continuation(std::shared_ptr<shim::FiberState> st, bool sink) : st_(std::move(st)), sink_(sink) {}
    continuation(continuation&& o) noexcept : st_(std::move(o.st_)), sink_(o.sink_) {}
    continuation& operator=(continuation&& o) noexcept {
        if (this != &o) {
            release();
            st_ = std::move(o.st_);
            sink_ = o.sink_;
        }
        return *this;
    }
    continuation(const continuation&) = delete;
    continuation& operator=(const continuation&) = delete;
    ~continuation() { release(); }

    explicit operator bool() const noexcept { return st_ != nullptr; }

    continuation resume() {
        auto st = std::move(st_);
        if (sink_) {
            // fiber side: hand control to the scheduler and wait to be resumed
            st->to_main.release();
            st->to_fiber.acquire();
            if (st->unwinding) throw detail::forced_unwind{};
            return continuation(std::move(st), true);
        }
        st->to_fiber.release();
        st->to_main.acquire();
        if (st->finished) {
            if (st->thread.joinable()) st->thread.join();
            return continuation();
        }
        return continuation(std::move(st), false);
    }

  private:
    void release() {
        if (!st_ || sink_) {
            st_.reset();
            return;
        }
        auto st = std::move(st_);
        if (!st->finished) {
            st->unwinding = true;
            st->to_fiber.release();
            st->to_main.acquire();
        }
        if (st->thread.joinable()) st->thread.join();
    }

    std::shared_ptr<shim::FiberState> st_;
    bool sink_ = false;
};

template <typename StackAlloc, typename Fn>
continuation callcc(std::allocator_arg_t, StackAlloc&&, Fn&& fn) {
    auto st = std::make_shared<shim::FiberState>();
    st->thread = std::thread([st, f = std::forward<Fn>(fn)]() mutable {
        st->to_fiber.acquire();
        try {
            continuation back = f(continuation(st, true));
            (void)back;
        } catch (const detail::forced_unwind&) {
        }
        st->finished = true;
        st->to_main.release();
    });
    st->to_fiber.release();
    st->to_main.acquire();
    if (st->finished) {
        st->thread.join();
        return continuation();
    }
    return continuation(std::move(st), false);
}

}  // namespace context
}  // namespace boost
