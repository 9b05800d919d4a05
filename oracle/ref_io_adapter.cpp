// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" adapter over the reference's UNMODIFIED dataset file code
// (/root/reference/proj/core/src/dataset_io.cpp, load_dataset / save_dataset), compiled by
// oracle/Makefile against nlohmann/json 3.11.3 -- the JSON library the reference vendors under
// vendor/ (absent from the mount); the identical release ships in this image as a header inside
// the cudnn_frontend package and is used here only to build this checker.  Output:
// oracle/_ref/libtswarp_ref_io.so (git-ignored).  Only tests/ load it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "tswarp/dataset_io.hpp"
#include "tswarp/types.hpp"

namespace R = tswarp_ref;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const R::ParseError& e) {
        g_err = e.what();
        return 5;
    } catch (const R::ValidationError& e) {
        g_err = e.what();
        return 4;
    } catch (const R::IoError& e) {
        g_err = e.what();
        return 6;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}
}  // namespace

extern "C" {

const char* refio_last_error(void) { return g_err.c_str(); }

// load_dataset (dataset_io.cpp:45-112) -> a heap R::Dataset (or NULL with *rc set)
void* refio_load(const char* path, int* rc) {
    R::Dataset* out = nullptr;
    *rc = guard([&] { out = new R::Dataset(R::load_dataset(path)); });
    return out;
}

void refio_free(void* ds) { delete static_cast<R::Dataset*>(ds); }

int refio_shape(void* h, uint64_t* n, uint64_t* d, uint64_t* total, int* labeled, uint64_t* nmeta) {
    const auto& ds = *static_cast<R::Dataset*>(h);
    *n = ds.size();
    *d = ds.dim();
    uint64_t t = 0;
    for (const auto& s : ds.series()) t += s.length();
    *total = t;
    *labeled = ds.labeled() ? 1 : 0;
    *nmeta = ds.meta().size();
    return 0;
}

int refio_copy(void* h, double* values, uint64_t* lengths) {
    const auto& ds = *static_cast<R::Dataset*>(h);
    uint64_t off = 0;
    for (std::size_t i = 0; i < ds.size(); ++i) {
        const auto f = ds[i].flat();
        std::memcpy(values + off, f.data(), f.size() * sizeof(double));
        off += f.size();
        lengths[i] = ds[i].length();
    }
    return 0;
}

const char* refio_label(void* h, uint64_t i) {
    const auto& ds = *static_cast<R::Dataset*>(h);
    return ds[i].label() ? ds[i].label()->c_str() : nullptr;
}

int refio_meta(void* h, uint64_t i, const char** k, const char** v) {
    const auto& ds = *static_cast<R::Dataset*>(h);
    auto it = ds.meta().begin();
    std::advance(it, (long)i);
    *k = it->first.c_str();
    *v = it->second.c_str();
    return 0;
}

// save_dataset (dataset_io.cpp:114-140)
int refio_save(void* h, const char* path) {
    return guard([&] { R::save_dataset(*static_cast<R::Dataset*>(h), path); });
}

}  // extern "C"
