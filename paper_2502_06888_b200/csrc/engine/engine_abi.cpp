// SPDX-License-Identifier: Apache-2.0
// extern "C" surface of the engine (include/klotski/engine.h). Exceptions
// never cross the boundary: they become a non-zero code + last_error text.
#include <cstdlib>
#include <cstring>
#include <string>

#include "engine.hpp"
#include "klotski/engine.h"
#include "klotski/kernels.h"

struct kl_engine {
    std::unique_ptr<klotski::Engine> impl;
    std::string error;
};

namespace {

thread_local std::string g_create_error;

// Exception class -> return code (include/klotski/engine.h, KL_E*), with the
// class name leading the message as the moesim Python module prints it.
int error_code(std::exception_ptr p, std::string& msg) {
    auto set = [&](const char* cls, const std::exception& x, int code) {
        msg = std::string(cls) + ": " + x.what();
        return code;
    };
    try {
        std::rethrow_exception(p);
    } catch (const moesim::MemoryInfeasible& x) {
        return set("MemoryInfeasible", x, KL_EMEMORY);
    } catch (const moesim::ConfigError& x) {
        return set("ConfigError", x, KL_ECONFIG);
    } catch (const moesim::ValidationError& x) {
        return set("ValidationError", x, KL_EVALIDATION);
    } catch (const moesim::ParseError& x) {
        return set("ParseError", x, KL_EPARSE);
    } catch (const moesim::RangeError& x) {
        return set("RangeError", x, KL_ERANGE);
    } catch (const moesim::AccountingError& x) {
        return set("AccountingError", x, KL_EACCOUNTING);
    } catch (const moesim::DeviceError& x) {
        return set("DeviceError", x, KL_EDEVICE);
    } catch (const std::exception& x) {
        msg = x.what();
        return KL_EOTHER;
    } catch (...) {
        msg = "unknown exception";
        return KL_EOTHER;
    }
}

char* dup_string(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

template <class F>
int guarded(kl_engine* e, F&& f) {
    if (e == nullptr || !e->impl) return 1;
    try {
        f(*e->impl);
        e->error.clear();
        return KL_OK;
    } catch (...) {
        return error_code(std::current_exception(), e->error);
    }
}

}  // namespace

extern "C" {

int kl_engine_create(const char* config_json, kl_engine** out) {
    if (out == nullptr) return 1;
    *out = nullptr;
    try {
        auto* e = new kl_engine;
        e->impl = std::make_unique<klotski::Engine>(klotski::parse_config(config_json ? config_json : ""));
        *out = e;
        return KL_OK;
    } catch (...) {
        return error_code(std::current_exception(), g_create_error);
    }
}

void kl_engine_destroy(kl_engine* e) { delete e; }

const char* kl_engine_last_error(const kl_engine* e) {
    return e == nullptr ? g_create_error.c_str() : e->error.c_str();
}

void kl_engine_free_string(char* s) { std::free(s); }

int kl_engine_describe(kl_engine* e, char** json_out) {
    return guarded(e, [&](klotski::Engine& g) { *json_out = dup_string(g.describe()); });
}

int kl_engine_fill_kv_synthetic(kl_engine* e, int positions, uint64_t seed) {
    return guarded(e, [&](klotski::Engine& g) { g.fill_kv_synthetic(positions, seed); });
}

int kl_engine_step(kl_engine* e, int step, const int32_t* tokens_in, int32_t* next_tokens_out, double* step_ms_out) {
    return guarded(e, [&](klotski::Engine& g) {
        const double ms = g.step(step, tokens_in, next_tokens_out);
        if (step_ms_out) *step_ms_out = ms;
    });
}

int kl_engine_report(kl_engine* e, const char* what, char** json_out) {
    return guarded(e, [&](klotski::Engine& g) { *json_out = dup_string(g.report(what ? what : "metrics")); });
}

int kl_engine_reset_log(kl_engine* e) {
    return guarded(e, [&](klotski::Engine& g) { g.reset_log(); });
}

int kl_measure_profile(const char* config_json, const char* phase, char** json_out) {
    if (json_out == nullptr) return 1;
    *json_out = nullptr;
    try {
        if (kl_device_supported() != 1) throw moesim::DeviceError("kl_measure_profile: device is not sm_100 (B200)");
        const klotski::EngineConfig cfg = klotski::parse_config(config_json ? config_json : "");
        *json_out = dup_string(klotski::measure_profile(cfg, phase ? phase : "decode").to_json());
        return KL_OK;
    } catch (...) {
        return error_code(std::current_exception(), g_create_error);
    }
}

int kl_engine_read_hidden(kl_engine* e, uint16_t* host, int64_t n_elems) {
    return guarded(e, [&](klotski::Engine& g) { g.read_hidden(host, n_elems); });
}

}  // extern "C"
