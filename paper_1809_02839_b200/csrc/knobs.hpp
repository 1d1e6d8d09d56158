// Development knobs: A/B timing switches and opt-in kernel variants that measured no
// faster than the defaults. The product library reads NO environment
// for them — every knob is its default. A development build (-DST_DEV_KNOBS:
// build.build_dev() → paper_1809_02839_b200/_var/dev/libspectrain.so) reads each one
// from the environment variable of the same name; tests/test_gpu_variants.py runs the
// parity tests against that build so the variant code paths stay correct.
#pragma once

#include <cstdlib>

namespace st {

inline int dev_knob(const char* name, int def) {
#ifdef ST_DEV_KNOBS
  const char* e = getenv(name);
  return e ? atoi(e) : def;
#else
  (void)name;
  return def;
#endif
}

}  // namespace st
