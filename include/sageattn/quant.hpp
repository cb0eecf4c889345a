// sageattn/quant.hpp -- B200 drop-in: the quantization dtype tag of the
// reference's public API (/root/reference/proj/include/sageattn/quant.hpp:22).
//
// The reference's CPU quantizers (quantize, smooth_k, fold_scale_into_q,
// quantize_p_static) are not re-exported: on this path they run inside K1 and
// K2 (paper_2410_02367_b200/csrc), bit-identical to the reference, behind
// sageattn::sage_attention.
#pragma once

#include <cstdint>

#include "tensor.hpp"

namespace sageattn {

enum class QuantDtype : uint8_t { Int8, FpE4M3, FpE5M2 };

}  // namespace sageattn
