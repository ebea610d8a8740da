// Exception -> return-code translation shared by the C-ABI translation units.
#pragma once

#include <exception>
#include <new>
#include <string>

#include "foundry/errors.hpp"

namespace foundry {

void fdy_set_last_error(const std::string& msg);

// Runs fn; maps foundry::Error to 1 + Errc and anything else to invalid-argument.
template <typename Fn>
int fdy_guard(Fn&& fn) noexcept {
    try {
        fn();
        return 0;
    } catch (const Error& e) {
        fdy_set_last_error(e.what());
        return 1 + static_cast<int>(e.code());
    } catch (const std::bad_alloc&) {
        fdy_set_last_error("invalid-argument: host allocation failed");
        return 1 + static_cast<int>(Errc::invalid_argument);
    } catch (const std::exception& e) {
        fdy_set_last_error(std::string("invalid-argument: ") + e.what());
        return 1 + static_cast<int>(Errc::invalid_argument);
    }
}

}  // namespace foundry
