/* ks_oracle.c -- TEST INFRASTRUCTURE ONLY (see ks_oracle.h).
 *
 * Plain-C fp64 restatement of the reference hot path.  Every function cites
 * the reference code it restates; accumulation orders are kept identical so
 * that the results are bit-identical to the reference build (no FMA: the
 * Makefile compiles with -ffp-contract=off and no -march, like the
 * reference's default CMake Release build).
 */
#define _GNU_SOURCE
#include "ks_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KSO_MAX_T 32
#define KSO_T_IN 7

static __thread char g_err[512];

static void set_err(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
}

const char* kso_last_error(void) { return g_err; }

typedef struct {
    char* name;
    int rank;
    int dims[3];
    int numel;
    double* data;
} kso_tensor_t;

struct kso_model {
    int variant;
    int e_size, n_a, n_s, n_d, cell;
    int t_out;
    int in_size[KSO_T_IN];
    int64_t* in_values[KSO_T_IN];
    int in_offset[KSO_T_IN];
    int d_in, d_fb;
    int vsize[KSO_MAX_T];
    int fb_offset[KSO_MAX_T];
    int value_offset[KSO_MAX_T];
    int64_t* out_values; /* concatenated, value_offset-indexed */
    char* out_names[KSO_MAX_T];
    int n_tensors;
    kso_tensor_t* tensors;
    /* resolved weight pointers */
    const double* enc_f_w[4];
    const double* enc_f_b[4];
    const double* enc_b_w[4];
    const double* enc_b_b[4];
    const double* dec_w[4];
    const double* dec_b[4];
    const double* att_h_w;
    const double* att_h_b;
    const double* att_o_w;
    const double* att_o_b;
    const double* head_w[KSO_MAX_T];
    const double* head_b[KSO_MAX_T];
    /* hybrid / hybrid-2 (models.cpp:296-371) */
    int n_conv;
    int conv_f[8], conv_k[8], conv_s[8];
    const double* conv_w[8];
    const double* conv_b[8];
    const double* h2f_w[4];
    const double* h2f_b[4];
    const double* h2b_w[4];
    const double* h2b_b[4];
};

/* ------------------------------------------------------------------------- */
/* checkpoint loading: kernelseer-checkpoint/1 (proj/src/data.cpp:513-665,     */
/* proj/docs/formats.md:53-93)                                               */
/* ------------------------------------------------------------------------- */

static int parse_int_list(const char* s, int64_t** out) {
    int cap = 16, n = 0;
    int64_t* v = (int64_t*)malloc(sizeof(int64_t) * cap);
    const char* p = s;
    while (*p) {
        char* end;
        long long x = strtoll(p, &end, 10);
        if (end == p) break;
        if (n == cap) {
            cap *= 2;
            v = (int64_t*)realloc(v, sizeof(int64_t) * cap);
        }
        v[n++] = x;
        p = end;
        while (*p == ',' || *p == ' ') ++p;
    }
    *out = v;
    return n;
}

static const kso_tensor_t* find_tensor(const kso_model* m, const char* name) {
    for (int i = 0; i < m->n_tensors; ++i)
        if (strcmp(m->tensors[i].name, name) == 0) return &m->tensors[i];
    return NULL;
}

double* kso_tensor(kso_model* m, const char* name, int* numel) {
    for (int i = 0; i < m->n_tensors; ++i)
        if (strcmp(m->tensors[i].name, name) == 0) {
            if (numel) *numel = m->tensors[i].numel;
            return m->tensors[i].data;
        }
    return NULL;
}

static int resolve_lstm(kso_model* m, const char* prefix, const double* w[4],
                        const double* b[4]) {
    static const char* gates[4] = {"input", "forget", "output", "cand"};
    char name[256];
    for (int q = 0; q < 4; ++q) {
        snprintf(name, sizeof name, "%s.w_%s", prefix, gates[q]);
        const kso_tensor_t* t = find_tensor(m, name);
        if (!t) return -1;
        w[q] = t->data;
        snprintf(name, sizeof name, "%s.b_%s", prefix, gates[q]);
        t = find_tensor(m, name);
        if (!t) return -1;
        b[q] = t->data;
    }
    return 0;
}

static int variant_code(const char* s) {
    if (!strcmp(s, "enc-dec")) return 0;
    if (!strcmp(s, "attn")) return 1;
    if (!strcmp(s, "attn-2")) return 2;
    if (!strcmp(s, "hybrid")) return 3;
    if (!strcmp(s, "hybrid-2")) return 4;
    return -1;
}

kso_model* kso_load(const char* path) {
    static const char* fields[KSO_T_IN] = {"n", "c", "h", "w", "k", "y", "x"};
    FILE* f = fopen(path, "rb");
    if (!f) {
        set_err("cannot open checkpoint");
        return NULL;
    }
    fseek(f, 0, SEEK_END);
    long size = ftell(f);
    fseek(f, 0, SEEK_SET);
    char* buf = (char*)malloc((size_t)size + 1);
    if (fread(buf, 1, (size_t)size, f) != (size_t)size) {
        fclose(f);
        free(buf);
        set_err("short read");
        return NULL;
    }
    fclose(f);
    buf[size] = 0;

    kso_model* m = (kso_model*)calloc(1, sizeof *m);
    m->variant = -1;
    int cap_t = 64;
    m->tensors = (kso_tensor_t*)calloc((size_t)cap_t, sizeof(kso_tensor_t));
    long pos = 0;
    int ok = 1, saw_format = 0;
    while (pos < size) {
        long eol = pos;
        while (eol < size && buf[eol] != '\n') ++eol;
        long len = eol - pos;
        if (len > 0 && buf[pos + len - 1] == '\r') --len;
        if (len == 0) {
            pos = eol + 1;
            break; /* header/payload separator */
        }
        char* line = strndup(buf + pos, (size_t)len);
        pos = eol + 1;
        char* colon = strstr(line, ": ");
        if (!colon) {
            set_err("malformed header line");
            ok = 0;
            free(line);
            break;
        }
        *colon = 0;
        const char* key = line;
        const char* val = colon + 2;
        if (!strcmp(key, "format")) {
            if (strcmp(val, "kernelseer-checkpoint/1")) {
                set_err("unsupported checkpoint format");
                ok = 0;
            }
            saw_format = 1;
        } else if (!strcmp(key, "variant")) {
            m->variant = variant_code(val);
        } else if (!strcmp(key, "encoder_state_size")) {
            m->e_size = atoi(val);
        } else if (!strcmp(key, "pre_attention_size")) {
            m->n_a = atoi(val);
        } else if (!strcmp(key, "post_attention_size")) {
            m->n_s = atoi(val);
        } else if (!strcmp(key, "attention_dense_nodes")) {
            m->n_d = atoi(val);
        } else if (!strcmp(key, "decoder_cell_size")) {
            m->cell = atoi(val);
        } else if (!strcmp(key, "conv_layers")) {
            const char* q = val;
            m->n_conv = 0;
            while (*q && m->n_conv < 8) {
                int f, k, st;
                if (sscanf(q, "%d,%d,%d", &f, &k, &st) != 3) break;
                m->conv_f[m->n_conv] = f;
                m->conv_k[m->n_conv] = k;
                m->conv_s[m->n_conv] = st;
                m->n_conv++;
                const char* semi = strchr(q, ';');
                if (!semi) break;
                q = semi + 1;
            }
        } else if (!strncmp(key, "input_vocab.", 12)) {
            for (int fi = 0; fi < KSO_T_IN; ++fi)
                if (!strcmp(key + 12, fields[fi])) {
                    m->in_size[fi] = parse_int_list(val, &m->in_values[fi]);
                }
        } else if (!strcmp(key, "output_params")) {
            m->t_out = atoi(val);
            if (m->t_out > KSO_MAX_T) {
                set_err("too many output positions");
                ok = 0;
            }
        } else if (!strncmp(key, "param.", 6)) {
            int idx = atoi(key + 6);
            const char* eq = strstr(val, " = ");
            if (!eq || idx < 0 || idx >= m->t_out) {
                set_err("bad param header line");
                ok = 0;
            } else {
                int64_t* vals;
                int n = parse_int_list(eq + 3, &vals);
                m->vsize[idx] = n;
                free(m->out_names[idx]);
                m->out_names[idx] = strndup(val, (size_t)(eq - val));
                /* stash values temporarily in tensors-free storage */
                if (!m->out_values) m->out_values = (int64_t*)calloc(KSO_MAX_T * 4096, sizeof(int64_t));
                for (int j = 0; j < n && j < 4096; ++j) m->out_values[idx * 4096 + j] = vals[j];
                free(vals);
            }
        } else if (!strcmp(key, "tensor")) {
            const char* sp = strrchr(val, ' ');
            if (!sp) {
                set_err("bad tensor header line");
                ok = 0;
            } else {
                if (m->n_tensors == cap_t) {
                    cap_t *= 2;
                    m->tensors = (kso_tensor_t*)realloc(m->tensors, sizeof(kso_tensor_t) * (size_t)cap_t);
                }
                kso_tensor_t* t = &m->tensors[m->n_tensors++];
                memset(t, 0, sizeof *t);
                t->name = strndup(val, (size_t)(sp - val));
                const char* d = sp + 1;
                t->numel = 1;
                while (*d && t->rank < 3) {
                    char* end;
                    long x = strtol(d, &end, 10);
                    if (end == d) break;
                    t->dims[t->rank++] = (int)x;
                    t->numel *= (int)x;
                    d = end;
                    if (*d == 'x') ++d;
                }
            }
        }
        free(line);
        if (!ok) break;
    }
    if (ok && !saw_format) {
        set_err("missing format header");
        ok = 0;
    }
    if (ok) {
        long need = 0;
        for (int i = 0; i < m->n_tensors; ++i) need += 4L * m->tensors[i].numel;
        if (size - pos != need) {
            set_err(size - pos < need ? "truncated payload" : "payload/shape mismatch");
            ok = 0;
        } else {
            const unsigned char* p = (const unsigned char*)buf + pos;
            for (int i = 0; i < m->n_tensors; ++i) {
                kso_tensor_t* t = &m->tensors[i];
                t->data = (double*)malloc(sizeof(double) * (size_t)(t->numel > 0 ? t->numel : 1));
                for (int j = 0; j < t->numel; ++j) {
                    uint32_t bits = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
                                    ((uint32_t)p[3] << 24);
                    float fv;
                    memcpy(&fv, &bits, 4);
                    t->data[j] = (double)fv;
                    p += 4;
                }
            }
        }
    }
    free(buf);
    if (!ok) {
        kso_free(m);
        return NULL;
    }
    /* vocabulary offsets (proj/src/encoding.cpp:36-50 in the reference numbering) */
    int w = 0;
    for (int fi = 0; fi < KSO_T_IN; ++fi) {
        m->in_offset[fi] = w;
        w += m->in_size[fi];
    }
    m->d_in = w;
    int fb = 1; /* GO slot */
    int vo = 0;
    int64_t* packed = (int64_t*)calloc((size_t)(KSO_MAX_T * 4096), sizeof(int64_t));
    for (int p = 0; p < m->t_out; ++p) {
        m->fb_offset[p] = fb;
        fb += m->vsize[p];
        m->value_offset[p] = vo;
        for (int j = 0; j < m->vsize[p]; ++j) packed[vo + j] = m->out_values[p * 4096 + j];
        vo += m->vsize[p];
    }
    free(m->out_values);
    m->out_values = packed;
    m->d_fb = fb;

    int bad = 0;
    if (m->variant == 1 || m->variant == 2) {
        bad |= resolve_lstm(m, "pre.fwd", m->enc_f_w, m->enc_f_b);
        bad |= resolve_lstm(m, "pre.bwd", m->enc_b_w, m->enc_b_b);
        bad |= resolve_lstm(m, "post", m->dec_w, m->dec_b);
        const kso_tensor_t* t;
        if ((t = find_tensor(m, "attn.hidden.weights"))) m->att_h_w = t->data; else bad = 1;
        if ((t = find_tensor(m, "attn.hidden.bias"))) m->att_h_b = t->data; else bad = 1;
        if ((t = find_tensor(m, "attn.out.weights"))) m->att_o_w = t->data; else bad = 1;
        if ((t = find_tensor(m, "attn.out.bias"))) m->att_o_b = t->data; else bad = 1;
    } else if (m->variant == 0) {
        bad |= resolve_lstm(m, "encoder", m->enc_f_w, m->enc_f_b);
        bad |= resolve_lstm(m, "decoder", m->dec_w, m->dec_b);
    } else if (m->variant == 3 || m->variant == 4) {
        bad |= resolve_lstm(m, "bilstm1.fwd", m->enc_f_w, m->enc_f_b);
        bad |= resolve_lstm(m, "bilstm1.bwd", m->enc_b_w, m->enc_b_b);
        bad |= resolve_lstm(m, "bilstm2.fwd", m->h2f_w, m->h2f_b);
        bad |= resolve_lstm(m, "bilstm2.bwd", m->h2b_w, m->h2b_b);
        for (int i = 0; i < m->n_conv && !bad; ++i) {
            char name[64];
            const kso_tensor_t* t;
            snprintf(name, sizeof name, "conv.%d.filters", i);
            if ((t = find_tensor(m, name))) m->conv_w[i] = t->data; else bad = 1;
            snprintf(name, sizeof name, "conv.%d.bias", i);
            if ((t = find_tensor(m, name))) m->conv_b[i] = t->data; else bad = 1;
        }
    } else {
        set_err("unknown model variant");
        kso_free(m);
        return NULL;
    }
    for (int p = 0; p < m->t_out && !bad; ++p) {
        char name[64];
        snprintf(name, sizeof name, "head.%d.weights", p);
        const kso_tensor_t* t = find_tensor(m, name);
        if (!t) { bad = 1; break; }
        m->head_w[p] = t->data;
        snprintf(name, sizeof name, "head.%d.bias", p);
        t = find_tensor(m, name);
        if (!t) { bad = 1; break; }
        m->head_b[p] = t->data;
    }
    if (bad) {
        set_err("model tensor missing");
        kso_free(m);
        return NULL;
    }
    return m;
}

void kso_free(kso_model* m) {
    if (!m) return;
    for (int i = 0; i < m->n_tensors; ++i) {
        free(m->tensors[i].name);
        free(m->tensors[i].data);
    }
    free(m->tensors);
    for (int fi = 0; fi < KSO_T_IN; ++fi) free(m->in_values[fi]);
    for (int p = 0; p < KSO_MAX_T; ++p) free(m->out_names[p]);
    free(m->out_values);
    free(m);
}

int kso_variant(const kso_model* m) { return m->variant; }
int kso_num_positions(const kso_model* m) { return m->t_out; }
int kso_vocab_size(const kso_model* m, int pos) { return m->vsize[pos]; }
const char* kso_output_name(const kso_model* m, int pos) { return m->out_names[pos]; }
int kso_input_vocab_size(const kso_model* m, int field) { return m->in_size[field]; }
int64_t kso_input_value(const kso_model* m, int field, int id) { return m->in_values[field][id]; }
int64_t kso_output_value(const kso_model* m, int pos, int id) {
    return m->out_values[m->value_offset[pos] + id];
}

/* encode_problem (proj/src/encoding.cpp:87-113), FieldVocab::id_of (11-16). */
int kso_encode_problem(const kso_model* m, const int64_t* desc7, int32_t* tok7) {
    for (int f = 0; f < KSO_T_IN; ++f) {
        int id = -1;
        for (int j = 0; j < m->in_size[f]; ++j)
            if (m->in_values[f][j] == desc7[f]) { id = j; break; }
        if (id < 0) return f;
        tok7[f] = id;
    }
    return -1;
}

/* ------------------------------------------------------------------------- */
/* nn core (proj/src/nn.cpp)                                                 */
/* ------------------------------------------------------------------------- */

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* accumulate_row_matmul (nn.cpp:14-24): y[j] += x[i]*W[i][j], i ascending,
 * rows with x[i] == 0 skipped. */
static void row_matmul(const double* x, int in, const double* w, int out, double* y) {
    for (int i = 0; i < in; ++i) {
        const double xi = x[i];
        if (xi == 0.0) continue;
        const double* wr = w + (size_t)i * out;
        for (int j = 0; j < out; ++j) y[j] += xi * wr[j];
    }
}

/* dense_forward (nn.cpp:63-86) for one row: y = b, then accumulate. */
static void dense(const double* x, int in, const double* w, const double* b, int out, double* y) {
    for (int j = 0; j < out; ++j) y[j] = b[j];
    row_matmul(x, in, w, out, y);
}

/* lstm_cell_step (nn.cpp:88-128). xh = [x; h]; gates i, f, o, cand. */
static void lstm_step(const double* x, int nx, const double* h, const double* c, int H,
                      const double* const W[4], const double* const B[4], double* h_out,
                      double* c_out, double* scratch) {
    double* xh = scratch;
    memcpy(xh, x, sizeof(double) * (size_t)nx);
    memcpy(xh + nx, h, sizeof(double) * (size_t)H);
    double* g[4];
    for (int q = 0; q < 4; ++q) {
        g[q] = scratch + nx + H + (size_t)q * H;
        dense(xh, nx + H, W[q], B[q], H, g[q]);
    }
    for (int j = 0; j < H; ++j) {
        const double ig = sigmoid(g[0][j]);
        const double fg = sigmoid(g[1][j]);
        const double og = sigmoid(g[2][j]);
        const double cg = tanh(g[3][j]);
        const double a = fg * c[j];
        const double bb = ig * cg;
        c_out[j] = a + bb;
        h_out[j] = og * tanh(c_out[j]);
    }
}

/* softmax (nn.cpp:215-226) in place over n entries. */
static void softmax(double* v, int n) {
    double mx = v[0];
    for (int i = 1; i < n; ++i)
        if (mx < v[i]) mx = v[i]; /* std::max_element keeps the first maximum */
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        v[i] = exp(v[i] - mx);
        sum += v[i];
    }
    for (int i = 0; i < n; ++i) v[i] /= sum;
}

/* ------------------------------------------------------------------------- */
/* model: encode / initial_state / step (proj/src/models.cpp:387-493)        */
/* ------------------------------------------------------------------------- */

typedef struct {
    double* dists; /* hybrid variants: every position's distribution (sum V_p) */
    double* act;   /* attn: 7 x 2 n_a */
    double* h0;    /* enc-dec thought vector */
    double* c0;
    double* scratch;
    double* x;     /* decoder input buffer */
} kso_enc;

static int dec_size(const kso_model* m) {
    return m->variant == 0 ? m->e_size : (m->variant >= 3 ? m->cell : m->n_s);
}

static size_t scratch_len(const kso_model* m) {
    int H = dec_size(m);
    int big = m->n_a > H ? m->n_a : H;
    if (m->e_size > big) big = m->e_size;
    int nx = 2 * m->n_a + m->d_fb + m->d_in + H + 16;
    return (size_t)(nx + big) * 6 + (size_t)(KSO_T_IN + 4) * (size_t)(2 * m->n_a + 4) + 4096;
}

static int check_input(const kso_model* m, const int32_t* tok7) {
    for (int f = 0; f < KSO_T_IN; ++f)
        if (tok7[f] < 0 || tok7[f] >= m->in_size[f]) return -1;
    return 0;
}

/* hybrid_encode (models.cpp:296-309) + conv1d_forward (nn.cpp:171-213): conv
 * stack over the (d_in x 7) one-hot matrix, flattened row-major (f, o). */
static double* hybrid_encoded(const kso_model* m, const int32_t* tok7, int* flat) {
    int ch = m->d_in, len = KSO_T_IN;
    double* x = (double*)calloc((size_t)ch * len, sizeof(double));
    for (int t = 0; t < KSO_T_IN; ++t) x[(size_t)(m->in_offset[t] + tok7[t]) * len + t] = 1.0;
    for (int i = 0; i < m->n_conv; ++i) {
        const int f = m->conv_f[i], k = m->conv_k[i], st = m->conv_s[i];
        const int o = (len - k) / st + 1;
        double* y = (double*)calloc((size_t)f * o, sizeof(double));
        for (int ff = 0; ff < f; ++ff)
            for (int j = 0; j < o; ++j) {
                double acc = m->conv_b[i][ff];
                const int start = j * st;
                for (int c = 0; c < ch; ++c) {
                    const double* row = x + (size_t)c * len;
                    for (int u = 0; u < k; ++u) acc += m->conv_w[i][((size_t)ff * ch + c) * k + u] * row[start + u];
                }
                y[(size_t)ff * o + j] = acc;
            }
        free(x);
        x = y;
        ch = f;
        len = o;
    }
    *flat = ch * len;
    return x;
}

/* hybrid2_decode (models.cpp:359-371) / hybrid encode branch (409-421):
 * distributions of every position, independent of the decoded prefix. */
static void hybrid_dists(const kso_model* m, const int32_t* tok7, kso_enc* e) {
    int F;
    double* enc = hybrid_encoded(m, tok7, &F);
    const int H = m->cell, T = m->t_out;
    const int nx2 = m->variant == 4 ? F : 2 * H;
    double* sc = (double*)calloc((size_t)(F + 2 * H) * 6 + 64, sizeof(double));
    double* f1 = (double*)calloc((size_t)T * H, sizeof(double));
    double* b1 = (double*)calloc((size_t)T * H, sizeof(double));
    double* f2 = (double*)calloc((size_t)T * H, sizeof(double));
    double* b2 = (double*)calloc((size_t)T * H, sizeof(double));
    double* h = (double*)calloc((size_t)H, sizeof(double));
    double* c = (double*)calloc((size_t)H, sizeof(double));
    double* h2 = (double*)calloc((size_t)H, sizeof(double));
    double* c2 = (double*)calloc((size_t)H, sizeof(double));
    double* fh = (double*)calloc((size_t)H, sizeof(double));
    double* fc = (double*)calloc((size_t)H, sizeof(double));
    double* x2 = (double*)calloc((size_t)2 * H + 1, sizeof(double));
    /* bi-LSTM 1 over T copies of the encoding, zero initial state */
    for (int t = 0; t < T; ++t) {
        lstm_step(enc, F, h, c, H, m->enc_f_w, m->enc_f_b, h2, c2, sc);
        memcpy(h, h2, sizeof(double) * (size_t)H);
        memcpy(c, c2, sizeof(double) * (size_t)H);
        memcpy(f1 + (size_t)t * H, h, sizeof(double) * (size_t)H);
    }
    memcpy(fh, h, sizeof(double) * (size_t)H);
    memcpy(fc, c, sizeof(double) * (size_t)H);
    memset(h, 0, sizeof(double) * (size_t)H);
    memset(c, 0, sizeof(double) * (size_t)H);
    for (int t = T - 1; t >= 0; --t) {
        lstm_step(enc, F, h, c, H, m->enc_b_w, m->enc_b_b, h2, c2, sc);
        memcpy(h, h2, sizeof(double) * (size_t)H);
        memcpy(c, c2, sizeof(double) * (size_t)H);
        memcpy(b1 + (size_t)t * H, h, sizeof(double) * (size_t)H);
    }
    /* bi-LSTM 2: hybrid-2 reads the encoding again and is seeded with
     * bi-LSTM 1's final states (bilstm_seeded, models.cpp:314-344); hybrid
     * reads bi-LSTM 1's activations from a zero state */
    double *bh = h, *bc = c;  /* backward final state of bi-LSTM 1 */
    double* sh = (double*)calloc((size_t)H, sizeof(double));
    double* scc = (double*)calloc((size_t)H, sizeof(double));
    if (m->variant == 4) {
        memcpy(sh, fh, sizeof(double) * (size_t)H);
        memcpy(scc, fc, sizeof(double) * (size_t)H);
    }
    for (int t = 0; t < T; ++t) {
        const double* xin = enc;
        if (m->variant == 3) {
            memcpy(x2, f1 + (size_t)t * H, sizeof(double) * (size_t)H);
            memcpy(x2 + H, b1 + (size_t)t * H, sizeof(double) * (size_t)H);
            xin = x2;
        }
        lstm_step(xin, nx2, sh, scc, H, m->h2f_w, m->h2f_b, h2, c2, sc);
        memcpy(sh, h2, sizeof(double) * (size_t)H);
        memcpy(scc, c2, sizeof(double) * (size_t)H);
        memcpy(f2 + (size_t)t * H, sh, sizeof(double) * (size_t)H);
    }
    if (m->variant == 4) {
        memcpy(sh, bh, sizeof(double) * (size_t)H);
        memcpy(scc, bc, sizeof(double) * (size_t)H);
    } else {
        memset(sh, 0, sizeof(double) * (size_t)H);
        memset(scc, 0, sizeof(double) * (size_t)H);
    }
    for (int t = T - 1; t >= 0; --t) {
        const double* xin = enc;
        if (m->variant == 3) {
            memcpy(x2, f1 + (size_t)t * H, sizeof(double) * (size_t)H);
            memcpy(x2 + H, b1 + (size_t)t * H, sizeof(double) * (size_t)H);
            xin = x2;
        }
        lstm_step(xin, nx2, sh, scc, H, m->h2b_w, m->h2b_b, h2, c2, sc);
        memcpy(sh, h2, sizeof(double) * (size_t)H);
        memcpy(scc, c2, sizeof(double) * (size_t)H);
        memcpy(b2 + (size_t)t * H, sh, sizeof(double) * (size_t)H);
    }
    /* head_distributions (models.cpp:346-355) */
    int off = 0;
    for (int t = 0; t < T; ++t) {
        memcpy(x2, f2 + (size_t)t * H, sizeof(double) * (size_t)H);
        memcpy(x2 + H, b2 + (size_t)t * H, sizeof(double) * (size_t)H);
        dense(x2, 2 * H, m->head_w[t], m->head_b[t], m->vsize[t], e->dists + off);
        softmax(e->dists + off, m->vsize[t]);
        off += m->vsize[t];
    }
    free(enc); free(sc); free(f1); free(b1); free(f2); free(b2); free(h); free(c); free(h2); free(c2);
    free(fh); free(fc); free(x2); free(sh); free(scc);
}

/* encode (models.cpp:387-428): attn branch -> bilstm_forward (nn.cpp:130-165);
 * enc-dec branch -> forward LSTM, final state is the thought vector. */
static void encode(const kso_model* m, const int32_t* tok7, kso_enc* e) {
    if (m->variant >= 3) {
        hybrid_dists(m, tok7, e);
        return;
    }
    double* onehot = e->scratch;                 /* d_in */
    double* sc = e->scratch + m->d_in + 8;       /* lstm scratch */
    if (m->variant == 0) {
        const int H = m->e_size;
        double* h = e->h0;
        double* c = e->c0;
        double* h2 = sc + scratch_len(m) / 2;
        double* c2 = h2 + H;
        memset(h, 0, sizeof(double) * (size_t)H);
        memset(c, 0, sizeof(double) * (size_t)H);
        for (int t = 0; t < KSO_T_IN; ++t) {
            memset(onehot, 0, sizeof(double) * (size_t)m->d_in);
            onehot[m->in_offset[t] + tok7[t]] = 1.0;
            lstm_step(onehot, m->d_in, h, c, H, m->enc_f_w, m->enc_f_b, h2, c2, sc);
            memcpy(h, h2, sizeof(double) * (size_t)H);
            memcpy(c, c2, sizeof(double) * (size_t)H);
        }
        return;
    }
    const int H = m->n_a;
    double* h = sc + scratch_len(m) / 2;
    double* c = h + H;
    double* h2 = c + H;
    double* c2 = h2 + H;
    /* forward direction */
    memset(h, 0, sizeof(double) * (size_t)H);
    memset(c, 0, sizeof(double) * (size_t)H);
    for (int t = 0; t < KSO_T_IN; ++t) {
        memset(onehot, 0, sizeof(double) * (size_t)m->d_in);
        onehot[m->in_offset[t] + tok7[t]] = 1.0;
        lstm_step(onehot, m->d_in, h, c, H, m->enc_f_w, m->enc_f_b, h2, c2, sc);
        memcpy(h, h2, sizeof(double) * (size_t)H);
        memcpy(c, c2, sizeof(double) * (size_t)H);
        memcpy(e->act + (size_t)t * 2 * H, h, sizeof(double) * (size_t)H);
    }
    /* backward direction, zero init */
    memset(h, 0, sizeof(double) * (size_t)H);
    memset(c, 0, sizeof(double) * (size_t)H);
    for (int t = KSO_T_IN - 1; t >= 0; --t) {
        memset(onehot, 0, sizeof(double) * (size_t)m->d_in);
        onehot[m->in_offset[t] + tok7[t]] = 1.0;
        lstm_step(onehot, m->d_in, h, c, H, m->enc_b_w, m->enc_b_b, h2, c2, sc);
        memcpy(h, h2, sizeof(double) * (size_t)H);
        memcpy(c, c2, sizeof(double) * (size_t)H);
        memcpy(e->act + (size_t)t * 2 * H + H, h, sizeof(double) * (size_t)H);
    }
}

static void enc_alloc(const kso_model* m, kso_enc* e) {
    int nd = 0;
    for (int p = 0; p < m->t_out; ++p) nd += m->vsize[p];
    e->dists = (double*)calloc((size_t)nd + 1, sizeof(double));
    e->act = (double*)calloc((size_t)KSO_T_IN * 2 * (size_t)(m->n_a + 1), sizeof(double));
    int H = dec_size(m);
    e->h0 = (double*)calloc((size_t)(m->e_size + 1), sizeof(double));
    e->c0 = (double*)calloc((size_t)(m->e_size + 1), sizeof(double));
    e->scratch = (double*)calloc(scratch_len(m) * 2, sizeof(double));
    e->x = (double*)calloc((size_t)(2 * m->n_a + m->d_fb + H + 16), sizeof(double));
}

static void enc_free(kso_enc* e) {
    free(e->dists);
    free(e->act);
    free(e->h0);
    free(e->c0);
    free(e->scratch);
    free(e->x);
}

/* SequencePredictor::step (models.cpp:448-493): writes dist (V_pos) and the
 * advanced state (h_out, c_out) for a hypothesis in state (h, c) at pos. */
static void step(const kso_model* m, const kso_enc* e, const double* h, const double* c, int pos,
                 int prev, double* h_out, double* c_out, double* dist) {
    const int H = dec_size(m);
    double* sc = e->scratch;
    double* x = e->x;
    int nx = 0;
    if (m->variant >= 3) {  /* hybrid: static distributions (models.cpp:484-488) */
        int off = 0;
        for (int q = 0; q < pos; ++q) off += m->vsize[q];
        memcpy(dist, e->dists + off, sizeof(double) * (size_t)m->vsize[pos]);
        memcpy(h_out, h, sizeof(double) * (size_t)H);
        memcpy(c_out, c, sizeof(double) * (size_t)H);
        return;
    }
    if (m->variant == 1 || m->variant == 2) {
        /* attention_weights (models.cpp:265-281) */
        const int A = 2 * m->n_a;
        const int nd = m->n_d;
        double* z = sc;                       /* H + A */
        double* hid = z + H + A;              /* nd */
        double* energies = hid + nd + 1;      /* 7 */
        double* ctx = energies + KSO_T_IN + 1; /* A */
        double* lsc = ctx + A + 1;
        for (int t = 0; t < KSO_T_IN; ++t) {
            memcpy(z, h, sizeof(double) * (size_t)H);
            memcpy(z + H, e->act + (size_t)t * A, sizeof(double) * (size_t)A);
            dense(z, H + A, m->att_h_w, m->att_h_b, nd, hid);
            for (int d = 0; d < nd; ++d) hid[d] = tanh(hid[d]);
            double eo;
            dense(hid, nd, m->att_o_w, m->att_o_b, 1, &eo);
            energies[t] = eo;
        }
        softmax(energies, KSO_T_IN);
        /* context_vector (models.cpp:283-294) */
        for (int j = 0; j < A; ++j) ctx[j] = 0.0;
        for (int t = 0; t < KSO_T_IN; ++t) {
            const double al = energies[t];
            const double* a = e->act + (size_t)t * A;
            for (int j = 0; j < A; ++j) ctx[j] += al * a[j];
        }
        memcpy(x, ctx, sizeof(double) * (size_t)A);
        nx = A;
        if (m->variant == 1) { /* feedback_onehot (encoding.cpp:192-199), GO at pos 0 */
            memset(x + A, 0, sizeof(double) * (size_t)m->d_fb);
            x[A + (pos == 0 ? 0 : m->fb_offset[pos - 1] + prev)] = 1.0;
            nx = A + m->d_fb;
        }
        lstm_step(x, nx, h, c, H, m->dec_w, m->dec_b, h_out, c_out, lsc);
    } else {
        memset(x, 0, sizeof(double) * (size_t)m->d_fb);
        x[pos == 0 ? 0 : m->fb_offset[pos - 1] + prev] = 1.0;
        lstm_step(x, m->d_fb, h, c, H, m->dec_w, m->dec_b, h_out, c_out, sc);
    }
    /* head dense + softmax (models.cpp:490-492) */
    dense(h_out, H, m->head_w[pos], m->head_b[pos], m->vsize[pos], dist);
    softmax(dist, m->vsize[pos]);
}

static void init_state(const kso_model* m, const kso_enc* e, double* h, double* c) {
    const int H = dec_size(m);
    if (m->variant == 0) {
        memcpy(h, e->h0, sizeof(double) * (size_t)H);
        memcpy(c, e->c0, sizeof(double) * (size_t)H);
    } else {
        memset(h, 0, sizeof(double) * (size_t)H);
        memset(c, 0, sizeof(double) * (size_t)H);
    }
}

int kso_encode(const kso_model* m, const int32_t* tok7, double* out) {
    if (m->variant != 1 && m->variant != 2) return -2;
    if (check_input(m, tok7)) return -1;
    kso_enc e;
    enc_alloc(m, &e);
    encode(m, tok7, &e);
    memcpy(out, e.act, sizeof(double) * (size_t)KSO_T_IN * 2 * (size_t)m->n_a);
    enc_free(&e);
    return 0;
}

int kso_forward(const kso_model* m, const int32_t* tok7, const int32_t* teacher, double* out) {
    if (check_input(m, tok7)) return -1;
    const int H = dec_size(m);
    kso_enc e;
    enc_alloc(m, &e);
    encode(m, tok7, &e);
    double* h = (double*)malloc(sizeof(double) * 4 * (size_t)H);
    double *c = h + H, *h2 = c + H, *c2 = h2 + H;
    init_state(m, &e, h, c);
    int prev = -1, off = 0;
    for (int p = 0; p < m->t_out; ++p) {
        double* dist = out + off;
        step(m, &e, h, c, p, prev, h2, c2, dist);
        memcpy(h, h2, sizeof(double) * (size_t)H);
        memcpy(c, c2, sizeof(double) * (size_t)H);
        if (teacher) {
            prev = teacher[p];
        } else {
            int best = 0;
            for (int i = 1; i < m->vsize[p]; ++i)
                if (dist[i] > dist[best]) best = i;
            prev = best;
        }
        off += m->vsize[p];
    }
    free(h);
    enc_free(&e);
    return 0;
}

/* greedy_decode (decoding.cpp:107-124): strict '>' keeps the lowest index. */
int kso_greedy(const kso_model* m, const int32_t* tok7, int32_t* out_tok) {
    if (check_input(m, tok7)) return -1;
    const int H = dec_size(m);
    kso_enc e;
    enc_alloc(m, &e);
    encode(m, tok7, &e);
    double* h = (double*)malloc(sizeof(double) * (4 * (size_t)H + 4096));
    double *c = h + H, *h2 = c + H, *c2 = h2 + H, *dist = c2 + H;
    init_state(m, &e, h, c);
    int prev = -1;
    for (int p = 0; p < m->t_out; ++p) {
        step(m, &e, h, c, p, prev, h2, c2, dist);
        memcpy(h, h2, sizeof(double) * (size_t)H);
        memcpy(c, c2, sizeof(double) * (size_t)H);
        int best = 0;
        for (int i = 1; i < m->vsize[p]; ++i)
            if (dist[i] > dist[best]) best = i;
        out_tok[p] = best;
        prev = best;
    }
    free(h);
    enc_free(&e);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* predicates                                                                 */
/* ------------------------------------------------------------------------- */

static int pred_accepts(const kso_model* m, const kso_pred* q, const int32_t* prefix, int pos,
                        const int64_t* desc7) {
    switch (q->kind) {
        case KSO_PRED_MASK:
            for (int i = 0; i <= pos; ++i)
                if (!q->allowed[m->value_offset[i] + prefix[i]]) return 0;
            return 1;
        case KSO_PRED_BUDGET: {
            /* resource_budget_predicate (constraints.cpp:232-240): alphabetical
             * name order, cost += w * value, accept cost <= budget */
            double cost = 0.0;
            for (int t = 0; t < q->n_terms; ++t) {
                const int p = q->term_pos[t];
                if (p < 0 || p > pos) continue;
                const double prod = q->term_w[t] * (double)kso_output_value(m, p, prefix[p]);
                cost = cost + prod;
            }
            return cost <= q->budget;
        }
        case KSO_PRED_PRODUCT: {
            __int128 prod = q->scale;
            for (int t = 0; t < q->n_terms; ++t) {
                const int p = q->term_pos[t];
                if (p < 0 || p > pos) continue;
                prod *= (__int128)kso_output_value(m, p, prefix[p]);
                if (prod > ((__int128)1 << 100)) prod = ((__int128)1 << 100);
                if (prod < -((__int128)1 << 100)) prod = -((__int128)1 << 100);
            }
            return prod <= (__int128)q->limit;
        }
        case KSO_PRED_DIVIDES:
            for (int t = 0; t < q->n_terms; ++t) {
                const int p = q->term_pos[t];
                if (p < 0 || p > pos) continue;
                const int64_t v = kso_output_value(m, p, prefix[p]);
                if (v <= 0 || desc7[q->term_field[t]] % v != 0) return 0;
            }
            return 1;
        default:
            return 1;
    }
}

/* ------------------------------------------------------------------------- */
/* beam search (proj/src/decoding.cpp:27-103)                                */
/* ------------------------------------------------------------------------- */

typedef struct {
    int parent;
    int token;
    double lp;
    const int32_t* pprefix; /* parent prefix (pos entries) */
    int pos;
} kso_child;

/* Candidate::operator< (decoding.cpp:21-24): higher log-prob first, exact ties
 * to the lexicographically smaller prefix. */
static int child_cmp(const void* a_, const void* b_) {
    const kso_child* a = (const kso_child*)a_;
    const kso_child* b = (const kso_child*)b_;
    if (a->lp != b->lp) return a->lp > b->lp ? -1 : 1;
    for (int i = 0; i < a->pos; ++i)
        if (a->pprefix[i] != b->pprefix[i]) return a->pprefix[i] < b->pprefix[i] ? -1 : 1;
    if (a->token != b->token) return a->token < b->token ? -1 : 1;
    return 0;
}

static double rel_gap(double a, double b) {
    double den = fabs(a) > fabs(b) ? fabs(a) : fabs(b);
    if (den < 1e-12) den = 1e-12;
    return fabs(a - b) / den;
}

int kso_beam(const kso_model* m, const int32_t* tok7, const int64_t* desc7, int k,
             const kso_pred* preds, int n_preds, int32_t* out_tok, double* out_lp,
             int32_t* out_count, int32_t* fail_pred, int32_t* fail_step, double* min_gap) {
    if (k < 1) {
        set_err("beam width must be >= 1");
        return -2;
    }
    if (check_input(m, tok7)) {
        set_err("input token out of range");
        return -1;
    }
    const int H = dec_size(m);
    const int T = m->t_out;
    int vmax = 1;
    for (int p = 0; p < T; ++p)
        if (m->vsize[p] > vmax) vmax = m->vsize[p];
    kso_enc e;
    enc_alloc(m, &e);
    encode(m, tok7, &e);

    const size_t kc = (size_t)k * (size_t)vmax;
    int32_t* prefix = (int32_t*)calloc((size_t)k * T + 1, sizeof(int32_t));
    int32_t* nprefix = (int32_t*)calloc((size_t)k * T + 1, sizeof(int32_t));
    double* lp = (double*)calloc((size_t)k, sizeof(double));
    double* st_h = (double*)calloc((size_t)k * H, sizeof(double));
    double* st_c = (double*)calloc((size_t)k * H, sizeof(double));
    double* adv_h = (double*)calloc((size_t)k * H, sizeof(double));
    double* adv_c = (double*)calloc((size_t)k * H, sizeof(double));
    double* dist = (double*)calloc((size_t)vmax + 1, sizeof(double));
    kso_child* kids = (kso_child*)calloc(kc + 1, sizeof(kso_child));
    int32_t* probe = (int32_t*)calloc((size_t)T + 1, sizeof(int32_t));
    double gap = INFINITY;
    int n = 1, rc = 0;
    init_state(m, &e, st_h, st_c);
    lp[0] = 0.0;
    const int constrained = n_preds > 0;
    for (int pos = 0; pos < T; ++pos) {
        const int V = m->vsize[pos];
        int nk = 0, last_rej = -1;
        const int final_step = pos == T - 1;
        for (int j = 0; j < n; ++j) {
            const int prev = pos == 0 ? -1 : prefix[(size_t)j * T + pos - 1];
            step(m, &e, st_h + (size_t)j * H, st_c + (size_t)j * H, pos, prev,
                 adv_h + (size_t)j * H, adv_c + (size_t)j * H, dist);
            for (int t = 0; t < V; ++t) {
                const double d = dist[t] > 1e-300 ? dist[t] : 1e-300; /* std::max(p, 1e-300) */
                const double clp = lp[j] + log(d);
                if (constrained) {
                    memcpy(probe, prefix + (size_t)j * T, sizeof(int32_t) * (size_t)pos);
                    probe[pos] = t;
                    int rejected = 0;
                    for (int q = 0; q < n_preds; ++q) {
                        if (preds[q].full_sequence_only && !final_step) continue;
                        if (!pred_accepts(m, &preds[q], probe, pos, desc7)) {
                            rejected = 1;
                            last_rej = q;
                            break;
                        }
                    }
                    if (rejected) continue;
                }
                kids[nk].parent = j;
                kids[nk].token = t;
                kids[nk].lp = clp;
                kids[nk].pprefix = prefix + (size_t)j * T;
                kids[nk].pos = pos;
                ++nk;
            }
        }
        if (nk == 0) {
            if (fail_pred) *fail_pred = last_rej;
            if (fail_step) *fail_step = pos;
            rc = 1;
            n = 0;
            break;
        }
        qsort(kids, (size_t)nk, sizeof(kso_child), child_cmp);
        const int keep = nk < k ? nk : k;
        if (nk > k) {
            const double g = rel_gap(kids[k - 1].lp, kids[k].lp);
            if (g < gap) gap = g;
        }
        if (final_step)
            for (int i = 0; i + 1 < keep; ++i) {
                const double g = rel_gap(kids[i].lp, kids[i + 1].lp);
                if (g < gap) gap = g;
            }
        for (int i = 0; i < keep; ++i) {
            const int par = kids[i].parent;
            memcpy(nprefix + (size_t)i * T, prefix + (size_t)par * T, sizeof(int32_t) * (size_t)pos);
            nprefix[(size_t)i * T + pos] = kids[i].token;
            lp[i] = kids[i].lp; /* safe: lp of parents no longer read below */
        }
        /* state copies must read adv_* by parent before overwriting st_* */
        for (int i = 0; i < keep; ++i) {
            const int par = kids[i].parent;
            memcpy(st_h + (size_t)i * H, adv_h + (size_t)par * H, sizeof(double) * (size_t)H);
            memcpy(st_c + (size_t)i * H, adv_c + (size_t)par * H, sizeof(double) * (size_t)H);
        }
        int32_t* tmp = prefix;
        prefix = nprefix;
        nprefix = tmp;
        n = keep;
    }
    if (out_count) *out_count = n;
    for (int i = 0; i < n; ++i) {
        out_lp[i] = lp[i];
        memcpy(out_tok + (size_t)i * T, prefix + (size_t)i * T, sizeof(int32_t) * (size_t)T);
    }
    if (min_gap) *min_gap = gap;
    free(prefix);
    free(nprefix);
    free(lp);
    free(st_h);
    free(st_c);
    free(adv_h);
    free(adv_c);
    free(dist);
    free(kids);
    free(probe);
    enc_free(&e);
    return rc;
}

/* Striped batch driver, the shape of parallel_stripes
 * (proj/include/kernelseer/parallel.hpp:14-27). */
typedef struct {
    const kso_model* m;
    const int32_t* tok;
    const int64_t* desc;
    int64_t B;
    int k;
    const kso_pred* preds;
    int n_preds;
    int32_t* out_tok;
    double* out_lp;
    int32_t* out_count;
    int32_t* out_status;
    int32_t* out_fail_pred;
    int32_t* out_fail_step;
    double* out_min_gap;
    int worker, stride;
} kso_job;

static void* batch_worker(void* arg) {
    kso_job* j = (kso_job*)arg;
    const int T = j->m->t_out;
    for (int64_t b = j->worker; b < j->B; b += j->stride) {
        int32_t fp = -1, fs = -1, cnt = 0;
        double g = INFINITY;
        int rc = kso_beam(j->m, j->tok + 7 * b, j->desc ? j->desc + 7 * b : NULL, j->k, j->preds,
                          j->n_preds, j->out_tok + (size_t)b * j->k * T, j->out_lp + (size_t)b * j->k,
                          &cnt, &fp, &fs, &g);
        j->out_count[b] = rc == 0 ? cnt : 0;
        j->out_status[b] = rc == 0 ? 0 : (rc == 1 ? 1 : 2);
        if (j->out_fail_pred) j->out_fail_pred[b] = fp;
        if (j->out_fail_step) j->out_fail_step[b] = fs;
        if (j->out_min_gap) j->out_min_gap[b] = g;
    }
    return NULL;
}

int kso_beam_batch(const kso_model* m, const int32_t* tok, const int64_t* desc, int64_t B, int k,
                   const kso_pred* preds, int n_preds, int threads, int32_t* out_tok, double* out_lp,
                   int32_t* out_count, int32_t* out_status, int32_t* out_fail_pred,
                   int32_t* out_fail_step, double* out_min_gap) {
    if (threads < 1) threads = 1;
    kso_job* jobs = (kso_job*)calloc((size_t)threads, sizeof(kso_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int w = 0; w < threads; ++w) {
        kso_job j = {m, tok, desc, B, k, preds, n_preds, out_tok, out_lp, out_count, out_status,
                     out_fail_pred, out_fail_step, out_min_gap, w, threads};
        jobs[w] = j;
    }
    if (threads == 1) {
        batch_worker(&jobs[0]);
    } else {
        for (int w = 0; w < threads; ++w) pthread_create(&th[w], NULL, batch_worker, &jobs[w]);
        for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
    }
    free(jobs);
    free(th);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Rng (proj/include/kernelseer/rng.hpp:13-71).  std::mt19937_64 is fully     */
/* specified by the C++ standard ([rand.eng.mers] with the mt19937_64          */
/* parameters), so this restatement reproduces the reference's streams.       */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} kso_mt64;

static void mt64_seed(kso_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(kso_mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static uint64_t rng_mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static void rng_derive(kso_mt64* g, uint64_t seed, uint64_t stream) {
    mt64_seed(g, rng_mix(rng_mix(seed) + 0x9e3779b97f4a7c15ULL * (stream + 1)));
}

static double rng_uniform(kso_mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

void kso_uniforms(uint64_t seed, uint64_t stream, int64_t n, double* out) {
    kso_mt64 g;
    rng_derive(&g, seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_uniform(&g);
}

void kso_dropout_masks(uint64_t seed, uint64_t stream, int n_in, double rate_in, int n_rec,
                       double rate_rec, double* out) {
    kso_mt64 g;
    rng_derive(&g, seed, stream);
    const double ki = 1.0 / (1.0 - rate_in), kr = 1.0 / (1.0 - rate_rec);
    for (int i = 0; i < n_in; ++i) out[i] = rng_uniform(&g) < rate_in ? 0.0 : ki;
    for (int i = 0; i < n_rec; ++i) out[n_in + i] = rng_uniform(&g) < rate_rec ? 0.0 : kr;
}

void kso_shuffle(uint64_t seed, uint64_t epoch, int64_t n, int64_t* order) {
    kso_mt64 g;
    rng_derive(&g, seed, 0x3ff000ULL + epoch);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    for (int64_t i = n; i > 1; --i) {
        const uint64_t m = (uint64_t)i;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % m;
        uint64_t v;
        do {
            v = mt64_next(&g);
        } while (v >= limit);
        const int64_t j = (int64_t)(v % m);
        const int64_t t = order[i - 1];
        order[i - 1] = order[j];
        order[j] = t;
    }
}
