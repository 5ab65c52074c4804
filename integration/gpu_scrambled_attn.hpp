// gpu_scrambled_attn.hpp -- reference-side adapter: the B200 path behind the reference's own
// pluggable attention provider (AttnFn, model.hpp:75-85).
//
// A maintainer of the reference adds this file (and links libsdattn_b200.so) to get a
// drop-in for sdattn::scrambled_attn (model.cpp:353-401): same options, same key derivation
// (request_id 1, domain 0, derive_seed chain), same per-segment span permutations, same merge
// -- with the scramble (K1), the keyless partial attention (K2), the local causal shard and the
// unscramble + merge (K3) executed on the GPU through the C ABI (include/sdattn_b200.h).
// Host f64 Matrix <-> device conversion happens only here.
#pragma once

#include "sdattn/model.hpp"

namespace sdattn_b200 {

// wire_fmt f64 or f32 -> FP32 device mode (Q'/K'/V' kept in f32); bf16 -> BF16 device mode
// (Q'/K'/V' rounded once to bf16, O' and the stats rounded to the bf16 grid as the reference's
// wire_round / wire_round_stat do, sda_wire_round); quant_bits in [2, 8] -> Q', K', V', O'
// quantised per tensor on the device (sda_quant_roundtrip), stats at f32. f16 wires throw
// std::invalid_argument, as do head dims outside {4, 8, ..., 256}.
sdattn::AttnFn gpu_scrambled_attn(const sdattn::ScrambledAttnOptions& opt);

}  // namespace sdattn_b200
