// Tuning / A-B experiment switches.
//
// The production library (the default Makefile build) compiles every switch to
// its measured default: no environment variable can change what a launch does.
// Tuning builds (`make TUNING=1`, tools/build_variant.sh) define PB_TUNING and
// read the PB_* variables once, at first use ("Tuning / A-B
// switches").
#pragma once
#include <stdlib.h>

namespace pb {

#ifdef PB_TUNING
inline int tune_int(const char* name, int def) {
  const char* e = getenv(name);
  return e ? atoi(e) : def;
}
inline double tune_dbl(const char* name, double def) {
  const char* e = getenv(name);
  return e ? atof(e) : def;
}
inline bool tune_flag(const char* name) { return getenv(name) != nullptr; }
#define PB_TUNE_INT(name, def) ([] { static const int v_ = ::pb::tune_int(name, def); return v_; }())
#define PB_TUNE_DBL(name, def) ([] { static const double v_ = ::pb::tune_dbl(name, def); return v_; }())
#define PB_TUNE_FLAG(name) ([] { static const bool v_ = ::pb::tune_flag(name); return v_; }())
// profiling bits of DictGramArgs::dbg (4: skip the bulk copies, 8: skip the element phase,
// 16: atomic-exchange grid barrier) — they skip work, so they exist in tuning builds only
#define PB_DBG(args, bit) ((args).dbg & (bit))
#else
#define PB_DBG(args, bit) 0
#define PB_TUNE_INT(name, def) (def)
#define PB_TUNE_DBL(name, def) (def)
#define PB_TUNE_FLAG(name) (false)
#endif

}  // namespace pb
