// Include-path forwarder: code written against the reference's "tgformer/sampler.hpp" compiles
// unchanged against the B200 host API (one header, include/tgfx/tgformer.hpp).
#pragma once
#include "tgfx/tgformer.hpp"
