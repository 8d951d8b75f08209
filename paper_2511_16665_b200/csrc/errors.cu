// Thread-local last-error channel of the C-ABI (status code + message).
#include <string>
#include "../../include/tlt_b200.h"

namespace {
thread_local std::string g_last_error;
}

extern "C" TLT_API void tlt_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }
extern "C" TLT_API const char* tlt_version(void) { return "tlt_b200 0.1 sm_100a"; }

namespace tlt {
const char* thread_last_error() { return g_last_error.c_str(); }
}

// Engines are driven by one host thread (see header), so the per-engine
// message is the calling thread's message.
extern "C" TLT_API const char* tlt_last_error(const tlt_engine*) { return tlt::thread_last_error(); }
