// hf_blob.cu -- the reference's on-disk field format (state blob + JSON sidecar,
// layout.hpp:155-200) behind the C ABI, so external fixtures (PyFR-like dumps, the
// reference's own export_blob output) feed the B200 host path directly:
//
//   <path>       the padded field's words, little-endian, 4 bytes (fp32) or 8 (fp64)
//   <path>.json  {"byte_order", "d", "group", "n_elem", "p", "precision", "words"},
//                written byte for byte as the reference's nlohmann dump(2) does
//                (sorted keys, two-space indent, trailing newline).
//
// Errors follow the reference: a missing / unreadable sidecar or blob, a word-count
// mismatch or a short read are std::runtime_error there (HF_ERUNTIME here); an unknown
// precision string is std::invalid_argument (precision_from_string, core.hpp:16-20;
// HF_EINVAL).  Host-only code: no CUDA call except in hf_fused_divergence_blob.
#include <cuda_runtime.h>

#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "../../include/hexfuse_b200.h"

// defined in hf_capi.cu
int hf_capi_fail(int code, const std::string& msg);

namespace {

int fail(int code, const std::string& msg) { return hf_capi_fail(code, msg); }

size_t wbytes(int precision) { return precision == HF_FP32 ? 4 : 8; }

// The flat sidecar object: string and integer values only (what field_sidecar writes).
bool parse_sidecar(const std::string& text, std::map<std::string, std::string>& str,
                   std::map<std::string, int64_t>& num) {
    size_t i = 0;
    auto ws = [&] {
        while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
    };
    auto lit = [&](std::string& out) {
        if (i >= text.size() || text[i] != '"') return false;
        const size_t j = text.find('"', i + 1);
        if (j == std::string::npos) return false;
        out = text.substr(i + 1, j - i - 1);
        i = j + 1;
        return true;
    };
    ws();
    if (i >= text.size() || text[i++] != '{') return false;
    ws();
    if (i < text.size() && text[i] == '}') return true;
    for (;;) {
        std::string key;
        ws();
        if (!lit(key)) return false;
        ws();
        if (i >= text.size() || text[i++] != ':') return false;
        ws();
        if (i < text.size() && text[i] == '"') {
            std::string v;
            if (!lit(v)) return false;
            str[key] = v;
        } else {
            const size_t j0 = i;
            if (i < text.size() && text[i] == '-') ++i;
            while (i < text.size() && std::isdigit(static_cast<unsigned char>(text[i]))) ++i;
            if (i == j0 || (i == j0 + 1 && text[j0] == '-') || i - j0 > 18) return false;  // fits int64
            num[key] = std::stoll(text.substr(j0, i - j0));
        }
        ws();
        if (i < text.size() && text[i] == ',') {
            ++i;
            continue;
        }
        if (i < text.size() && text[i] == '}') return true;
        return false;
    }
}

std::string sidecar_text(const hf_problem* pr, int64_t words) {
    char buf[512];
    std::snprintf(buf, sizeof(buf),
                  "{\n  \"byte_order\": \"little\",\n  \"d\": %d,\n  \"group\": %d,\n  \"n_elem\": %lld,\n"
                  "  \"p\": %d,\n  \"precision\": \"%s\",\n  \"words\": %lld\n}\n",
                  pr->d, pr->group, static_cast<long long>(pr->n_elem), pr->p,
                  pr->precision == HF_FP32 ? "fp32" : "fp64", static_cast<long long>(words));
    return buf;
}

}  // namespace

extern "C" {

int hf_blob_info(const char* path, hf_problem* shape_out) {
    if (!path || !shape_out) return fail(HF_EINVAL, "hf_blob_info: null argument");
    const std::string side = std::string(path) + ".json";
    std::FILE* f = std::fopen(side.c_str(), "rb");
    if (!f) return fail(HF_ERUNTIME, "import_blob: missing sidecar " + side);
    std::string text;
    char chunk[4096];
    size_t n;
    while ((n = std::fread(chunk, 1, sizeof(chunk), f)) > 0) text.append(chunk, n);
    std::fclose(f);
    std::map<std::string, std::string> str;
    std::map<std::string, int64_t> num;
    bool parsed = false;
    try {  // nothing may escape the C ABI
        parsed = parse_sidecar(text, str, num);
    } catch (const std::exception&) {
        parsed = false;
    }
    if (!parsed) return fail(HF_ERUNTIME, "import_blob: malformed sidecar " + side);
    for (const char* k : {"d", "p", "n_elem", "group", "words"})
        if (!num.count(k)) return fail(HF_ERUNTIME, std::string("import_blob: sidecar lacks \"") + k + "\"");
    if (!str.count("precision")) return fail(HF_ERUNTIME, "import_blob: sidecar lacks \"precision\"");
    const std::string& prec = str["precision"];
    if (prec != "fp32" && prec != "fp64") return fail(HF_EINVAL, "unknown precision: " + prec);
    if (str.count("byte_order") && str["byte_order"] != "little")
        return fail(HF_ERUNTIME, "import_blob: byte_order must be little");
    hf_problem q = *shape_out;
    q.d = int(num["d"]);
    q.p = int(num["p"]);
    q.n_elem = num["n_elem"];
    q.group = int(num["group"]);
    q.precision = prec == "fp32" ? HF_FP32 : HF_FP64;
    const int64_t words = hf_field_words(&q);
    if (words < 0 || words != num["words"]) return fail(HF_ERUNTIME, "import_blob: sidecar word count mismatch");
    *shape_out = q;
    return HF_OK;
}

int hf_blob_read(const char* path, const hf_problem* pr, void* host_words) {
    if (!path || !pr) return fail(HF_EINVAL, "hf_blob_read: null argument");
    hf_problem side = *pr;
    if (int rc = hf_blob_info(path, &side)) return rc;
    if (side.d != pr->d || side.p != pr->p || side.n_elem != pr->n_elem || side.group != pr->group ||
        side.precision != pr->precision)
        return fail(HF_EINVAL, "hf_blob_read: the sidecar's shape differs from the problem");
    const int64_t words = hf_field_words(pr);
    if (words > 0 && !host_words) return fail(HF_EINVAL, "hf_blob_read: null buffer");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return fail(HF_ERUNTIME, std::string("import_blob: cannot open ") + path);
    const size_t want = size_t(words);
    const size_t got = want ? std::fread(host_words, wbytes(pr->precision), want, f) : 0;
    std::fclose(f);
    if (got != want) return fail(HF_ERUNTIME, "import_blob: short read");
    return HF_OK;
}

int hf_blob_write(const char* path, const hf_problem* pr, const void* host_words) {
    if (!path || !pr) return fail(HF_EINVAL, "hf_blob_write: null argument");
    if (int rc = hf_validate(pr)) return rc;
    const int64_t words = hf_field_words(pr);
    if (words > 0 && !host_words) return fail(HF_EINVAL, "hf_blob_write: null buffer");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return fail(HF_ERUNTIME, std::string("export_blob: cannot open ") + path);
    const size_t put = words ? std::fwrite(host_words, wbytes(pr->precision), size_t(words), f) : 0;
    const bool ok = std::fclose(f) == 0 && put == size_t(words);
    if (!ok) return fail(HF_ERUNTIME, std::string("export_blob: write failed ") + path);
    const std::string side = std::string(path) + ".json";
    std::FILE* s = std::fopen(side.c_str(), "wb");
    if (!s) return fail(HF_ERUNTIME, "export_blob: cannot open " + side);
    const std::string text = sidecar_text(pr, words);
    const bool ok2 = std::fwrite(text.data(), 1, text.size(), s) == text.size();
    if (std::fclose(s) != 0 || !ok2) return fail(HF_ERUNTIME, "export_blob: write failed " + side);
    return HF_OK;
}

int hf_fused_divergence_blob(hf_context* ctx, const hf_problem* params, const char* in_path, const char* out_path) {
    if (!ctx || !params || !in_path || !out_path) return fail(HF_EINVAL, "hf_fused_divergence_blob: null argument");
    hf_problem pr = *params;  // physics, jac, source and method from the caller; shape from the sidecar
    if (int rc = hf_blob_info(in_path, &pr)) return rc;
    if (int rc = hf_validate(&pr)) return rc;
    const int64_t words = hf_field_words(&pr);
    const size_t bytes = size_t(words) * wbytes(pr.precision);
    void* host = nullptr;  // pinned: both copy directions at full PCIe rate, in place
    if (bytes) {
        cudaError_t e = cudaMallocHost(&host, bytes);
        if (e != cudaSuccess) return fail(HF_ERUNTIME, std::string("hf_fused_divergence_blob: cudaMallocHost: ") +
                                                           cudaGetErrorString(e));
    }
    int rc = hf_blob_read(in_path, &pr, host);
    if (rc == HF_OK && words) rc = hf_fused_divergence_host(ctx, &pr, host, host);
    if (rc == HF_OK) rc = hf_blob_write(out_path, &pr, host);
    if (host) cudaFreeHost(host);
    return rc;
}

}  // extern "C"
