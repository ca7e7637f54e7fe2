// oracle/shim.hpp -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// Forced-include shim used when compiling the read-only reference sources
// under /root/reference/proj/src out of tree.  The reference header
// include/larch/core/device_array.hpp:36-50 declares element_kind_of<T> for
// double/int32/int64 but not for their const-qualified forms, so every
// `as_span<const double>()` in device_array.cpp, reference.cpp, parallel.cpp
// and sim_device.cpp fails to compile as shipped.  This
// file adds the three missing specialisations without touching the reference.
#pragma once
#include "larch/core/device_array.hpp"

namespace larch {
template <>
struct element_kind_of<const double> {
    static constexpr ElementKind value = ElementKind::float64;
};
template <>
struct element_kind_of<const std::int32_t> {
    static constexpr ElementKind value = ElementKind::int32;
};
template <>
struct element_kind_of<const std::int64_t> {
    static constexpr ElementKind value = ElementKind::int64;
};
}  // namespace larch
