// Umbrella header: the whole reference-compatible C++ API.
//
// Code written against the reference (`#include "dwt2d/executor.hpp"`,
// `dwt2d::compile<float>(...)`) switches by including this header instead;
// the namespace alias keeps every `dwt2d::` name valid. See INTEGRATION.md.
#pragma once

#include "dwt2d_b200.h"
#include "dwt2d_b200/algebra.hpp"
#include "dwt2d_b200/executor.hpp"
#include "dwt2d_b200/image.hpp"
#include "dwt2d_b200/lowering.hpp"
#include "dwt2d_b200/schemes.hpp"

namespace dwt2d = dwt2d_b200;
