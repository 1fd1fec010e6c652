// knobs.h — the MM_* tuning / diagnostic environment knobs, read with one scan of the environment
// per ABI call (knobs_refresh) instead of one getenv() per knob per call.
#pragma once
#include <cstring>

extern char** environ;

namespace mmb {

struct KnobSnap {
  int n = 0;
  const char* name[48];  // "MM_X=value" entries of environ (valid for the duration of the call)
};
inline KnobSnap& knob_snap() {
  static thread_local KnobSnap s;
  return s;
}
// Snapshot the MM_* entries of the environment (call at the top of each ABI entry point).
inline void knobs_refresh() {
  KnobSnap& s = knob_snap();
  s.n = 0;
  for (char** e = environ; e && *e && s.n < 48; ++e)
    if ((*e)[0] == 'M' && (*e)[1] == 'M' && (*e)[2] == '_') s.name[s.n++] = *e;
}
// Value of knob `name` ("MM_..."), or nullptr when unset.
inline const char* knob(const char* name) {
  const KnobSnap& s = knob_snap();
  const size_t len = strlen(name);
  for (int i = 0; i < s.n; ++i)
    if (strncmp(s.name[i], name, len) == 0 && s.name[i][len] == '=') return s.name[i] + len + 1;
  return nullptr;
}

}  // namespace mmb
