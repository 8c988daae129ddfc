// Former location of the C++ mirror; the drop-in header is now at the
// reference's own path, sgl/sgl_transform.hpp.
#pragma once

#include "sgl/sgl_transform.hpp"
