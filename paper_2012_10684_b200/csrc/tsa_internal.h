// tsa_internal.h -- library-internal declarations shared by the translation
// units of libtsa (not part of the C ABI in include/tsa.h).
#pragma once
#include <stdint.h>

extern "C" {
// tsa_default_units with an explicit SM count (tsa_default_units passes the
// current device's; the sharded path a fixed one, so every rank agrees).
int32_t tsa_units_for_sms(int64_t nz, int32_t bins, int32_t k, int32_t enumeration, int32_t sms);
// set the thread-local detail string returned by tsa_last_error()
void tsa_internal_set_error(const char *msg);
}
