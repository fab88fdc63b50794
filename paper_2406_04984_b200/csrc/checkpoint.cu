// MEFT1 checkpoints (memtier.cpp:288-396): the on-disk format written ONCE, table-driven, for every store kind.
//   meft_ckpt_save / meft_ckpt_load  -- host-resident stores through per-tensor callbacks (the C++ shim's HostStore)
//   meft_store_save / meft_store_load -- HBM stores, through the public store transfer calls of this library
// Layouts are the reference's (w_a d x r, w_b r x d, ...): the device store transposes at the transfer boundary.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "json_mini.hpp"
#include "meft_cuda.h"

meft_status meft_internal_fail(meft_ctx* ctx, int code, const char* msg);  // meft_capi.cu

namespace {

enum Enc { ENC_F32, ENC_F64, ENC_I64 };

struct Item {
    meft_tensor t;
    Enc enc;
};

// Per-layer payload in file order: masters narrowed to f32, Adam moments f64, step counters i64, router last.
const Item kPairItems[] = {{MEFT_T_W_A, ENC_F32}, {MEFT_T_W_B, ENC_F32}, {MEFT_T_W_G, ENC_F32},
                           {MEFT_T_M_A, ENC_F64}, {MEFT_T_V_A, ENC_F64}, {MEFT_T_M_B, ENC_F64},
                           {MEFT_T_V_B, ENC_F64}, {MEFT_T_PAIR_STEP, ENC_I64}};
const Item kRouterItems[] = {{MEFT_T_M_G, ENC_F64}, {MEFT_T_V_G, ENC_F64}, {MEFT_T_ROUTER_STEP, ENC_I64}};

std::vector<Item> layer_items(const meft_ckpt_header& h) {
    std::vector<Item> v(std::begin(kPairItems), std::end(kPairItems));
    if (h.train_router) v.insert(v.end(), std::begin(kRouterItems), std::end(kRouterItems));
    return v;
}

// Reference-layout shape of an item.
void item_shape(const meft_ckpt_header& h, meft_tensor t, int64_t& rows, int64_t& cols) {
    switch (t) {
        case MEFT_T_W_A: case MEFT_T_M_A: case MEFT_T_V_A: rows = h.dim; cols = h.pairs; return;
        case MEFT_T_W_B: case MEFT_T_M_B: case MEFT_T_V_B: rows = h.pairs; cols = h.dim; return;
        case MEFT_T_W_G: case MEFT_T_M_G: case MEFT_T_V_G: rows = h.experts; cols = h.dim; return;
        case MEFT_T_PAIR_STEP: rows = h.pairs; cols = 1; return;
        case MEFT_T_ROUTER_STEP: rows = h.experts; cols = 1; return;
        default: rows = cols = 0; return;
    }
}

struct Fail {  // carried out of the format code, mapped to a status at the C boundary
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }

meft_json::Value parse_extra(const char* extra_json) {
    try {
        return meft_json::Parser(extra_json ? extra_json : "{}").parse();
    } catch (const meft_json::ParseError& e) {
        fail(MEFT_E_INVALID, std::string("save_checkpoint: extra metadata is not JSON: ") + e.what());
    }
}

std::string header_line(const meft_ckpt_header& h, const meft_json::Value& extra) {
    using meft_json::Value;
    Value v = Value::object();
    v.o["magic"] = Value::string("MEFT1");
    v.o["version"] = Value::integer(1);
    v.o["layers"] = Value::integer(h.layers);
    v.o["dim"] = Value::integer(h.dim);
    v.o["pairs"] = Value::integer(h.pairs);
    v.o["experts"] = Value::integer(h.experts);
    v.o["train_router"] = Value::boolean(h.train_router != 0);
    v.o["step"] = Value::integer(h.step);
    v.o["weight_precision"] = Value::string("f32");
    v.o["moment_precision"] = Value::string("f64");
    v.o["extra"] = extra;
    return meft_json::dump(v);
}

// Parses and validates the header line in the reference's order (memtier.cpp:337-357).
meft_ckpt_header read_header(std::istream& in, std::string* extra_dump) {
    std::string line;
    if (!std::getline(in, line)) fail(MEFT_E_CKPT_HEADER, "checkpoint: missing header line");
    meft_json::Value v;
    try {
        v = meft_json::Parser(line).parse();
    } catch (const meft_json::ParseError& e) {
        fail(MEFT_E_CKPT_HEADER, std::string("checkpoint: corrupt header: ") + e.what());
    }
    using K = meft_json::Value;
    if (!v.has("magic") || v.at("magic").kind != K::Str || v.at("magic").s != "MEFT1")
        fail(MEFT_E_CKPT_HEADER, "checkpoint: bad magic");
    if (!v.has("version") || v.at("version").kind != K::Int || v.at("version").i != 1)
        fail(MEFT_E_CKPT_HEADER, "checkpoint: unsupported version");
    for (const char* key : {"layers", "dim", "pairs", "experts", "train_router", "step"})
        if (!v.has(key)) fail(MEFT_E_CKPT_HEADER, std::string("checkpoint: header missing field ") + key);
    auto integer = [&](const char* key) {
        if (v.at(key).kind != K::Int) fail(MEFT_E_CKPT_HEADER, std::string("checkpoint: field ") + key + " is not an integer");
        return v.at(key).i;
    };
    meft_ckpt_header h{};
    h.layers = integer("layers");
    h.dim = integer("dim");
    h.pairs = integer("pairs");
    h.experts = integer("experts");
    h.step = integer("step");
    if (v.at("train_router").kind != K::Bool) fail(MEFT_E_CKPT_HEADER, "checkpoint: field train_router is not a bool");
    h.train_router = v.at("train_router").b ? 1 : 0;
    if (h.layers < 1 || h.dim < 1 || h.pairs < 1 || h.experts < 1)
        fail(MEFT_E_CKPT_SHAPE, "checkpoint: non-positive shape in header");
    if (extra_dump) *extra_dump = v.has("extra") ? meft_json::dump(v.at("extra")) : std::string("{}");
    return h;
}

void copy_extra(const std::string& e, char* out, size_t cap) {
    if (!out || cap == 0) return;
    const size_t n = std::min(cap - 1, e.size());
    std::memcpy(out, e.data(), n);
    out[n] = 0;
}

void save_impl(const char* path, const meft_ckpt_header& h, const char* extra_json, meft_ckpt_source source,
               void* user) {
    const meft_json::Value extra = parse_extra(extra_json);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(MEFT_E_IO, std::string("save_checkpoint: cannot open ") + path);
    out << header_line(h, extra) << "\n";
    std::vector<double> vals;
    std::vector<float> narrow;
    for (int64_t l = 0; l < h.layers; ++l) {
        for (const Item& it : layer_items(h)) {
            int64_t r, c;
            item_shape(h, it.t, r, c);
            const size_t n = size_t(r * c);
            vals.resize(n);  // int64 counters share the 8-byte buffer
            if (source(user, l, it.t, vals.data(), int64_t(n)) != 0)
                fail(MEFT_E_IO, "save_checkpoint: tensor source failed");
            if (it.enc == ENC_F32) {
                narrow.assign(vals.begin(), vals.end());
                out.write(reinterpret_cast<const char*>(narrow.data()), std::streamsize(n * sizeof(float)));
            } else {
                out.write(reinterpret_cast<const char*>(vals.data()), std::streamsize(n * 8));
            }
        }
    }
    if (!out) fail(MEFT_E_IO, std::string("save_checkpoint: write failed for ") + path);
}

meft_ckpt_header load_impl(const char* path, std::string* extra, meft_ckpt_sink sink, void* user) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(MEFT_E_IO, std::string("load_checkpoint: cannot open ") + path);
    const meft_ckpt_header h = read_header(in, extra);
    std::vector<double> vals;
    std::vector<float> narrow;
    for (int64_t l = 0; l < h.layers; ++l) {
        for (const Item& it : layer_items(h)) {
            int64_t r, c;
            item_shape(h, it.t, r, c);
            const size_t n = size_t(r * c);
            vals.resize(n);
            if (it.enc == ENC_F32) {
                narrow.resize(n);
                in.read(reinterpret_cast<char*>(narrow.data()), std::streamsize(n * sizeof(float)));
                std::copy(narrow.begin(), narrow.end(), vals.begin());
            } else {
                in.read(reinterpret_cast<char*>(vals.data()), std::streamsize(n * 8));
            }
            if (!in)
                fail(MEFT_E_CKPT_TRUNCATED, it.enc == ENC_I64 ? "checkpoint: truncated counter payload"
                                                              : "checkpoint: truncated tensor payload");
            if (sink(user, &h, l, it.t, vals.data(), int64_t(n)) != 0) fail(MEFT_E_IO, "load_checkpoint: tensor sink failed");
        }
    }
    char probe;
    if (in.get(probe)) fail(MEFT_E_CKPT_SHAPE, "checkpoint: trailing bytes after payload");
    return h;
}

template <class F>
meft_status boundary(meft_ctx* ctx, F&& f) {
    try {
        f();
        return MEFT_OK;
    } catch (const Fail& e) {
        return meft_internal_fail(ctx, e.code, e.msg.c_str());
    } catch (const std::bad_alloc&) {
        return meft_internal_fail(ctx, MEFT_E_OOM, "checkpoint: host allocation failed");
    } catch (const std::exception& e) {
        return meft_internal_fail(ctx, MEFT_E_IO, e.what());
    }
}

// ---- device-store adapters over the public transfer calls
struct DevStore {
    meft_ctx* ctx;
    meft_store* store;
    meft_precision prec;
    meft_status inner = MEFT_OK;  // first failing transfer call, reported instead of the generic callback error
    std::string inner_msg;
    int note(meft_status st) {
        if (st != MEFT_OK && inner == MEFT_OK) {
            inner = st;
            inner_msg = meft_last_error(ctx);
        }
        return st == MEFT_OK ? 0 : 1;
    }
};

int dev_source(void* user, int64_t layer, meft_tensor t, void* dst, int64_t n) {
    auto* d = static_cast<DevStore*>(user);
    int64_t r, c;
    meft_ckpt_header h{};
    meft_store_info(d->store, &h.layers, &h.dim, &h.pairs, &h.experts, nullptr);
    item_shape(h, t, r, c);
    (void)n;
    return d->note(meft_store_download_host(d->ctx, d->store, layer, t, dst, r, c));
}

int dev_sink(void* user, const meft_ckpt_header* h, int64_t layer, meft_tensor t, const void* src, int64_t n) {
    auto* d = static_cast<DevStore*>(user);
    if (!d->store) {  // first tensor: the header is known, build the store
        if (d->note(meft_store_create(d->ctx, h->layers, h->dim, h->pairs, h->experts, d->prec, &d->store))) return 1;
        if (h->train_router && d->note(meft_store_enable_router(d->ctx, d->store))) return 1;
    }
    int64_t r, c;
    item_shape(*h, t, r, c);
    (void)n;
    return d->note(meft_store_upload_host(d->ctx, d->store, layer, t, src, r, c));
}

}  // namespace

extern "C" {

meft_status meft_ckpt_save(const char* path, const meft_ckpt_header* header, const char* extra_json,
                           meft_ckpt_source source, void* user) {
    return boundary(nullptr, [&] {
        if (!path || !header || !source) fail(MEFT_E_INVALID, "save_checkpoint: null argument");
        save_impl(path, *header, extra_json, source, user);
    });
}

meft_status meft_ckpt_load(const char* path, meft_ckpt_header* header, char* extra_out, size_t extra_cap,
                           meft_ckpt_sink sink, void* user) {
    return boundary(nullptr, [&] {
        if (!path || !sink) fail(MEFT_E_INVALID, "load_checkpoint: null argument");
        std::string extra;
        const meft_ckpt_header h = load_impl(path, &extra, sink, user);
        if (header) *header = h;
        copy_extra(extra, extra_out, extra_cap);
    });
}

meft_status meft_store_save(meft_ctx* ctx, meft_store* store, const char* path, int64_t step, const char* extra_json) {
    return boundary(ctx, [&] {
        if (!ctx || !store || !path) fail(MEFT_E_INVALID, "save_checkpoint: null argument");
        meft_ckpt_header h{};
        meft_precision prec;
        meft_store_info(store, &h.layers, &h.dim, &h.pairs, &h.experts, &prec);
        meft_store_train_router(store, &h.train_router);
        h.step = step;
        DevStore d{ctx, store, prec};
        try {
            save_impl(path, h, extra_json, dev_source, &d);
        } catch (const Fail&) {
            if (d.inner != MEFT_OK) fail(d.inner, d.inner_msg);
            throw;
        }
    });
}

meft_status meft_store_load(meft_ctx* ctx, const char* path, meft_precision precision, meft_store** out,
                            meft_ckpt_header* header, char* extra_out, size_t extra_cap) {
    DevStore d{ctx, nullptr, precision};
    const meft_status st = boundary(ctx, [&] {
        if (!ctx || !path || !out) fail(MEFT_E_INVALID, "load_checkpoint: null argument");
        std::string extra;
        meft_ckpt_header h;
        try {
            h = load_impl(path, &extra, dev_sink, &d);
        } catch (const Fail&) {
            if (d.inner != MEFT_OK) fail(d.inner, d.inner_msg);
            throw;
        }
        if (header) *header = h;
        copy_extra(extra, extra_out, extra_cap);
    });
    if (st != MEFT_OK) {
        meft_store_destroy(d.store);
        return st;
    }
    *out = d.store;
    return MEFT_OK;
}

}  // extern "C"
