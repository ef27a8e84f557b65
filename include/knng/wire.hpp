// The reference's header name (knng/wire.hpp), forwarded to the B200 drop-in:
// code written against the reference compiles unchanged with -I include and
// links libknng_b200.so.
#pragma once
#include "../knng_b200.hpp"
