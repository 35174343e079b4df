// errors.cpp -- thread-local error message, option defaults, ABI version.
#include <string>

#include "dm_internal.h"

namespace dm {

static thread_local std::string g_last_error;

dm_status fail(dm_status code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

void clear_error() { g_last_error.clear(); }

}  // namespace dm

extern "C" {

const char *dm_last_error(void) { return dm::g_last_error.c_str(); }

int32_t dm_abi_version(void) { return DM_ABI_VERSION; }

void dm_match_opts_init(dm_match_opts *opt) {
  if (!opt) return;
  opt->mode = DM_MONO;
  opt->output = DM_OUT_COUNT;
  opt->motifs = DM_MOTIF_M2 | DM_MOTIF_M3 | DM_MOTIF_M3O;
  opt->flags = 0;
  opt->row_budget = 0;
  opt->mem_budget = 0;
  opt->seed_begin = 0;
  opt->seed_end = -1;
  opt->cuda_stream = nullptr;
}

}  // extern "C"
