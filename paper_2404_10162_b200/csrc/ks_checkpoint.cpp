// ks_checkpoint.cpp -- kernelseer-checkpoint/1 reader behind the C-ABI
// (ks_checkpoint_* in include/ks_b200.h).
//
// Format (reference: proj/docs/formats.md:53-93, writer proj/src/data.cpp:464-511,
// reader data.cpp:513-665): "key: value" header lines, one empty line, then
// every tensor as little-endian fp32 in header order.  Failure kinds match
// CheckpointError::Kind (errors.hpp:66-74): version, truncated, shape,
// malformed, io.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "ks_b200.h"
#include "ks_internal.h"

struct ks_checkpoint {
    std::vector<std::pair<std::string, std::string>> header;
    struct T {
        std::string name;
        std::vector<int32_t> dims;
        std::vector<float> data;
    };
    std::vector<T> tensors;
};

namespace {
thread_local int32_t g_ck_kind = -1;

ks_status fail(int kind, const std::string& msg) {
    g_ck_kind = kind;
    return ksb_host::set_error(KS_ERR_CHECKPOINT, msg);
}
}  // namespace

extern "C" int32_t ks_checkpoint_error_kind(void) { return g_ck_kind; }

// The header keys the reference reader accepts (data.cpp:524-613); anything else
// is CheckpointError(malformed) there, and here.
static bool known_key(const std::string& k) {
    static const char* plain[] = {"variant", "kernel", "precision", "encoder_state_size",
                                  "pre_attention_size", "post_attention_size", "attention_dense_nodes",
                                  "decoder_cell_size", "dropout", "recurrent_dropout", "output_params"};
    for (const char* p : plain)
        if (k == p) return true;
    return k.rfind("input_vocab.", 0) == 0 || k.rfind("param.", 0) == 0;
}

extern "C" ks_status ks_checkpoint_load(const char* path, ks_checkpoint** out) {
    enum { VERSION = 0, TRUNCATED = 1, SHAPE = 2, MALFORMED = 3, IO = 4 };
    if (!path || !out) return ksb_host::set_error(KS_ERR_PARAMETER, "null argument");
    std::ifstream in(path, std::ios::binary);
    if (!in) return fail(IO, std::string("cannot open ") + path);
    std::string all((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    auto ck = new ks_checkpoint();
    size_t pos = 0;
    bool saw_format = false, ended = false;
    while (pos < all.size()) {
        size_t eol = all.find('\n', pos);
        if (eol == std::string::npos) eol = all.size();
        std::string line = all.substr(pos, eol - pos);
        pos = eol + 1;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) {
            ended = true;
            break;
        }
        const size_t colon = line.find(": ");
        if (colon == std::string::npos) {
            delete ck;
            return fail(MALFORMED, "malformed header line: " + line);
        }
        std::string key = line.substr(0, colon), val = line.substr(colon + 2);
        if (key == "format") {
            if (val != "kernelseer-checkpoint/1") {
                delete ck;
                return fail(VERSION, "unsupported checkpoint format '" + val + "'");
            }
            saw_format = true;
        } else if (key == "tensor") {
            const size_t sp = val.rfind(' ');
            if (sp == std::string::npos) {
                delete ck;
                return fail(MALFORMED, "bad tensor header line: " + line);
            }
            ks_checkpoint::T t;
            t.name = val.substr(0, sp);
            std::stringstream ss(val.substr(sp + 1));
            std::string d;
            while (std::getline(ss, d, 'x')) {
                try {
                    t.dims.push_back(std::stoi(d));
                } catch (...) {
                    delete ck;
                    return fail(MALFORMED, "bad tensor shape: " + line);
                }
            }
            if (t.dims.empty()) {
                delete ck;
                return fail(SHAPE, "tensor " + t.name + " has no shape");
            }
            // every reference tensor is rank 1 or 2 (models.cpp:178-259); dims are
            // positive (a zero / negative dim would wrap the payload byte count)
            if (t.dims.size() > 3) {
                delete ck;
                return fail(SHAPE, "tensor " + t.name + " has rank " + std::to_string(t.dims.size()));
            }
            for (int32_t dd : t.dims)
                if (dd <= 0) {
                    delete ck;
                    return fail(SHAPE, "tensor " + t.name + " has a non-positive dimension");
                }
            ck->tensors.push_back(std::move(t));
        } else if (key == "conv_layers") {
            // each layer is exactly three integers (data.cpp:566-578)
            std::stringstream ss(val);
            std::string layer;
            while (std::getline(ss, layer, ';')) {
                int n = 0;
                std::stringstream ls(layer);
                std::string tokn;
                bool bad = false;
                while (std::getline(ls, tokn, ',')) {
                    char* end = nullptr;
                    std::strtol(tokn.c_str(), &end, 10);
                    bad = bad || tokn.empty() || *end != '\0';
                    ++n;
                }
                if (bad || n != 3) {
                    delete ck;
                    return fail(MALFORMED, "bad conv layer spec: " + layer);
                }
            }
        } else if (!known_key(key)) {
            delete ck;
            return fail(MALFORMED, "unknown header key '" + key + "'");
        }
        ck->header.emplace_back(std::move(key), std::move(val));
    }
    if (!saw_format) {
        delete ck;
        return fail(VERSION, "missing format header");
    }
    (void)ended;
    size_t need = 0;
    for (auto& t : ck->tensors) {
        size_t n = 1;
        for (int32_t d : t.dims) n *= (size_t)d;
        need += 4 * n;
    }
    const size_t have = pos <= all.size() ? all.size() - pos : 0;
    if (have < need) {
        delete ck;
        return fail(TRUNCATED, "payload has " + std::to_string(have) + " bytes, header declares " +
                                   std::to_string(need));
    }
    if (have > need) {
        delete ck;
        return fail(SHAPE, "payload has " + std::to_string(have) +
                               " bytes, header shapes account for " + std::to_string(need));
    }
    const unsigned char* p = reinterpret_cast<const unsigned char*>(all.data()) + pos;
    for (auto& t : ck->tensors) {
        size_t n = 1;
        for (int32_t d : t.dims) n *= (size_t)d;
        t.data.resize(n);
        for (size_t i = 0; i < n; ++i) {
            const uint32_t bits = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
                                  ((uint32_t)p[3] << 24);
            std::memcpy(&t.data[i], &bits, 4);
            p += 4;
        }
    }
    *out = ck;
    return KS_OK;
}

extern "C" void ks_checkpoint_free(ks_checkpoint* ck) { delete ck; }

extern "C" const char* ks_checkpoint_header(const ks_checkpoint* ck, const char* key) {
    if (!ck || !key) return nullptr;
    for (auto& kv : ck->header)
        if (kv.first == key) return kv.second.c_str();
    return nullptr;
}

extern "C" int32_t ks_checkpoint_num_tensors(const ks_checkpoint* ck) {
    return ck ? (int32_t)ck->tensors.size() : 0;
}

extern "C" ks_status ks_checkpoint_tensor(const ks_checkpoint* ck, int32_t i, const char** name,
                                          int32_t* rank, int32_t* dims, const float** data) {
    if (!ck || i < 0 || i >= (int32_t)ck->tensors.size())
        return ksb_host::set_error(KS_ERR_INDEX, "tensor index out of range");
    const auto& t = ck->tensors[(size_t)i];
    if (name) *name = t.name.c_str();
    if (rank) *rank = (int32_t)t.dims.size();
    if (dims)
        for (size_t d = 0; d < t.dims.size() && d < 3; ++d) dims[d] = t.dims[d];
    if (data) *data = t.data.data();
    return KS_OK;
}

namespace ksb_host {

// Builds a ks_model_desc view over a parsed checkpoint (arrays owned by `store`).
ks_status desc_from_checkpoint(const ks_checkpoint* ck, DescStore& store, ks_model_desc& d) {
    static const char* fields[7] = {"n", "c", "h", "w", "k", "y", "x"};
    auto hdr = [&](const char* k) { return ks_checkpoint_header(ck, k); };
    const char* var = hdr("variant");
    if (!var) return set_error(KS_ERR_CHECKPOINT, "checkpoint has no variant");
    const std::string v = var;
    int code = v == "enc-dec" ? 0 : v == "attn" ? 1 : v == "attn-2" ? 2 : v == "hybrid" ? 3
             : v == "hybrid-2" ? 4 : -1;
    if (code < 0) return set_error(KS_ERR_VALIDATION, "unknown model variant '" + v + "'", "variant");
    auto geti = [&](const char* k, int dflt) {
        const char* s = hdr(k);
        return s ? std::atoi(s) : dflt;
    };
    std::memset(&d, 0, sizeof d);
    d.variant = code;
    d.encoder_state_size = geti("encoder_state_size", 256);
    d.pre_attention_size = geti("pre_attention_size", 256);
    d.post_attention_size = geti("post_attention_size", 512);
    d.attention_dense_nodes = geti("attention_dense_nodes", 2);
    d.num_positions = geti("output_params", 0);
    d.decoder_cell_size = geti("decoder_cell_size", 256);
    store.conv.clear();
    if (const char* cl = hdr("conv_layers")) {
        std::stringstream ss(cl);
        std::string layer;
        while (std::getline(ss, layer, ';')) {
            int f = 0, k = 0, st = 0;
            if (std::sscanf(layer.c_str(), "%d,%d,%d", &f, &k, &st) == 3) {
                store.conv.push_back(f);
                store.conv.push_back(k);
                store.conv.push_back(st);
            }
        }
    }
    d.num_conv_layers = (int32_t)(store.conv.size() / 3);
    d.conv_layers = store.conv.data();
    auto parse_list = [](const std::string& s, std::vector<int64_t>& out) {
        std::stringstream ss(s);
        std::string piece;
        int n = 0;
        while (std::getline(ss, piece, ',')) {
            if (piece.empty()) continue;
            out.push_back(std::stoll(piece));
            ++n;
        }
        return n;
    };
    store.input_sizes.assign(7, 0);
    store.input_values.clear();
    for (int f = 0; f < 7; ++f) {
        const char* s = hdr((std::string("input_vocab.") + fields[f]).c_str());
        if (!s) return set_error(KS_ERR_CHECKPOINT, std::string("missing input vocabulary for field ") + fields[f]);
        store.input_sizes[f] = parse_list(s, store.input_values);
    }
    store.vocab_sizes.assign((size_t)d.num_positions, 0);
    store.output_values.clear();
    store.param_names.assign((size_t)d.num_positions, "");
    std::vector<std::vector<int64_t>> per((size_t)d.num_positions);
    for (int p = 0; p < d.num_positions; ++p) {
        const char* s = hdr((std::string("param.") + std::to_string(p)).c_str());
        if (!s) return set_error(KS_ERR_CHECKPOINT, "missing param." + std::to_string(p));
        const std::string sv = s;
        const size_t eq = sv.find(" = ");
        if (eq == std::string::npos) return set_error(KS_ERR_CHECKPOINT, "bad param header line");
        store.param_names[(size_t)p] = sv.substr(0, eq);
        store.vocab_sizes[(size_t)p] = parse_list(sv.substr(eq + 3), per[(size_t)p]);
    }
    for (auto& vv : per) store.output_values.insert(store.output_values.end(), vv.begin(), vv.end());
    store.names.clear();
    store.numel.clear();
    store.data.clear();
    for (int32_t i = 0; i < ks_checkpoint_num_tensors(ck); ++i) {
        const char* name;
        int32_t rank, dims[3] = {1, 1, 1};
        const float* data;
        ks_checkpoint_tensor(ck, i, &name, &rank, dims, &data);
        int32_t n = 1;
        for (int r = 0; r < rank; ++r) n *= dims[r];
        store.names.push_back(name);
        store.numel.push_back(n);
        store.data.push_back(data);
    }
    store.name_ptrs.clear();
    for (auto& s : store.names) store.name_ptrs.push_back(s.c_str());
    d.input_sizes = store.input_sizes.data();
    d.input_values = store.input_values.data();
    d.vocab_sizes = store.vocab_sizes.data();
    d.output_values = store.output_values.data();
    d.num_tensors = (int32_t)store.names.size();
    d.tensor_names = store.name_ptrs.data();
    d.tensor_numel = store.numel.data();
    d.tensor_data = store.data.data();
    return KS_OK;
}

}  // namespace ksb_host
