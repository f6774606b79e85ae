// qmsort-gpu -- the reference's command-line harness (proj/tools/qmsort.cpp)
// with the sort running on the B200 through the C-ABI (include/qmsort_gpu.h).
// SURVEY.md 8(f) row f2.
//
//   qmsort-gpu bench --algo A --n N[,N...] [--dist D] [--trials T] [--seed S]
//              [--beta R] [--delta R] [--block B] [--three-way] [--side S] [--out F]
//       trials to CSV with the reference's exact schema (trial.hpp:62-77):
//       algorithm,n,distribution,seed,trial,comparisons,moves,time_ns,max_depth,
//       cmp_norm_linear,cmp_over_nlogn.  A is gpu (= the qms preset) or
//       qms|qmqs|momqms|hqms, optionally prefixed "gpu-"; the sort of every
//       trial runs on the GPU.  comparisons / moves are not counted on the GPU
//       (0, so the two normalised columns follow the reference formulas with
//       c = 0); time_ns is the device time of the sort; max_depth = partition
//       levels.  Inputs are the reference's generate_input streams with the
//       reference's per-trial seeds (qmsort.cpp:51-53), so both harnesses sort
//       identical arrays.
//   qmsort-gpu verify [--quick]
//       the invariant suite (qmsort.cpp:125-297) restricted to what the GPU
//       path promises: sorted permutations for every preset x distribution x
//       size, descending order, selection rank, key + payload order, depth.
//   qmsort-gpu sort_file INPUT OUTPUT [--algo A] [--beta R] [--delta R] ...
//       newline-delimited int64 text, same parsing and diagnostics as
//       qmsort.cpp:303-344.
//   qmsort-gpu gen --dist D --n N --seed S [--trial T]
//       print the generator stream (parity aid for the tests).
//
// Exit codes follow the reference: 0 ok, 1 failure / bad input line, 2 usage.
#include <algorithm>
#include <charconv>
#include <cinttypes>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <stdexcept>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/qmsort_gpu.h"

namespace {

// ---- rng.hpp:10-44 (restated): SplitMix64, bounded, mix_seed --------------
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t seed) : state(seed) {}
    uint64_t next() {
        uint64_t z = (state += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
};

uint64_t bounded(SplitMix64& rng, uint64_t n) {  // widening multiply with rejection
    if (n <= 1) return 0;
    unsigned __int128 mul = (unsigned __int128)rng.next() * n;
    uint64_t low = (uint64_t)mul;
    if (low < n) {
        const uint64_t threshold = (0 - n) % n;
        while (low < threshold) {
            mul = (unsigned __int128)rng.next() * n;
            low = (uint64_t)mul;
        }
    }
    return (uint64_t)(mul >> 64);
}

uint64_t mix_seed(uint64_t seed, uint64_t stream) {
    SplitMix64 g(seed ^ (0xD1B54A32D192ED03ull * (stream + 1)));
    return g.next();
}

// ---- dataset.hpp:14-99 (restated) -----------------------------------------
enum class Dist { random_perm, sorted, reverse, organ_pipe, few_distinct, random_dup };
struct DataSpec {
    Dist kind = Dist::random_perm;
    size_t param = 0;
};

std::string dataset_name(const DataSpec& d) {
    switch (d.kind) {
        case Dist::random_perm: return "random";
        case Dist::sorted: return "sorted";
        case Dist::reverse: return "reverse";
        case Dist::organ_pipe: return "organpipe";
        case Dist::few_distinct: return "fewdistinct:" + std::to_string(d.param);
        case Dist::random_dup: return "randomdup:" + std::to_string(d.param);
    }
    return "unknown";
}

std::optional<DataSpec> parse_dataset(const std::string& s) {
    if (s == "random") return DataSpec{Dist::random_perm, 0};
    if (s == "sorted") return DataSpec{Dist::sorted, 0};
    if (s == "reverse") return DataSpec{Dist::reverse, 0};
    if (s == "organpipe") return DataSpec{Dist::organ_pipe, 0};
    const auto colon = s.find(':');
    if (colon == std::string::npos) return std::nullopt;
    const std::string head = s.substr(0, colon), tail = s.substr(colon + 1);
    if (tail.empty() || tail.find_first_not_of("0123456789") != std::string::npos) return std::nullopt;
    const size_t v = (size_t)std::stoull(tail);
    if (v == 0) return std::nullopt;
    if (head == "fewdistinct") return DataSpec{Dist::few_distinct, v};
    if (head == "randomdup") return DataSpec{Dist::random_dup, v};
    return std::nullopt;
}

std::vector<int64_t> generate_input(const DataSpec& d, size_t n, uint64_t seed) {
    std::vector<int64_t> v(n);
    switch (d.kind) {
        case Dist::random_perm: {  // Fisher-Yates over 1..n
            for (size_t i = 0; i < n; ++i) v[i] = (int64_t)(i + 1);
            SplitMix64 rng(seed);
            for (size_t i = n; i > 1; --i) std::swap(v[i - 1], v[(size_t)bounded(rng, i)]);
            break;
        }
        case Dist::sorted:
            for (size_t i = 0; i < n; ++i) v[i] = (int64_t)(i + 1);
            break;
        case Dist::reverse:
            for (size_t i = 0; i < n; ++i) v[i] = (int64_t)(n - i);
            break;
        case Dist::organ_pipe:
            for (size_t i = 0; i < n; ++i) v[i] = (int64_t)std::min(i + 1, n - i);
            break;
        case Dist::few_distinct: {
            const size_t k = d.param == 0 ? 1 : d.param;
            for (size_t i = 0; i < n; ++i) v[i] = (int64_t)(i % k + 1);
            break;
        }
        case Dist::random_dup: {
            const uint64_t mod = d.param == 0 ? 1 : d.param;
            SplitMix64 rng(seed);
            for (size_t i = 0; i < n; ++i) v[i] = (int64_t)(bounded(rng, mod) + 1);
            break;
        }
    }
    return v;
}

// qmsort.cpp:51-53: a fixed function of (seed, n, trial)
uint64_t trial_seed(uint64_t seed, size_t n, uint64_t trial) {
    return mix_seed(seed, (uint64_t)n * 1000003ull + trial);
}

// Fields of `text` between separators (a trailing separator yields an empty
// last field; a string without separators is one field).
std::vector<std::string> split(const std::string& text, char sep) {
    std::vector<std::string> fields(1);
    for (const char c : text) {
        if (c == sep) fields.emplace_back();
        else fields.back().push_back(c);
    }
    return fields;
}

// ---- options ---------------------------------------------------------------
struct Options {
    std::string algo = "qms";
    std::string sizes = "65536";
    std::string dist = "random";
    uint64_t trials = 10;
    uint64_t seed = 1;
    std::string beta = "1/2";
    std::string delta = "1/16";
    size_t block = 128;  // kDefaultBlock (partition.hpp:16)
    bool three_way = false;
    std::string side = "larger";
    std::string out_path;
    bool quick = false;
    int64_t trial = -1;
    std::vector<std::string> positional;
};

// "p/q" or a plain number (the --beta / --delta syntax of the reference CLI)
double parse_ratio(const std::string& text) {
    const auto parts = split(text, '/');
    double v = std::stod(parts.at(0));
    if (parts.size() > 1) v /= std::stod(parts[1]);
    return v;
}

// Comma-separated sizes; empty fields are skipped ("1,,2," = {1, 2}).
std::vector<size_t> parse_size_list(const std::string& text) {
    std::vector<size_t> sizes;
    for (const std::string& field : split(text, ','))
        if (!field.empty()) sizes.push_back(static_cast<size_t>(std::stoull(field)));
    return sizes;
}

// "gpu" / "[gpu-]qms|qmqs|momqms|hqms" -> preset (sort.hpp:37-66); -1 if unknown
int parse_algo(const std::string& a) {
    std::string s = a;
    if (s == "gpu") return 0;
    if (s.rfind("gpu-", 0) == 0) s = s.substr(4);
    if (s == "qms") return 0;
    if (s == "qmqs") return 1;
    if (s == "momqms") return 2;
    if (s == "hqms") return 3;
    return -1;
}

qmsort_gpu_config build_config(int preset, const Options& o) {  // qmsort.cpp:67-76
    qmsort_gpu_config c;
    qmsort_gpu_config_init(&c, preset);
    c.beta = parse_ratio(o.beta);
    c.delta = parse_ratio(o.delta);
    c.block = o.block;
    c.three_way = o.three_way ? 1 : 0;
    c.side = o.side == "smaller" ? 0 : 1;
    return c;
}

void check_rc(int rc, const char* where) {
    if (rc != QMSORT_OK)
        throw std::runtime_error(std::string(where) + " failed (" + std::to_string(rc) + "): " +
                                 qmsort_gpu_last_error());
}

// Multiset fingerprint + order check: the verify_sort_outcome contract
// (trial.hpp:81-86) in O(n) on the host (no CPU sort anywhere).
struct Print {
    uint64_t sum = 0, x = 0;
};
Print fingerprint(const std::vector<int64_t>& v) {
    Print p;
    for (int64_t e : v) {
        SplitMix64 g((uint64_t)e);
        const uint64_t h = g.next();
        p.sum += h;
        p.x ^= h;
    }
    return p;
}
bool verify_sort_outcome(const Print& before, const std::vector<int64_t>& out) {
    if (!std::is_sorted(out.begin(), out.end())) return false;
    const Print after = fingerprint(out);
    return after.sum == before.sum && after.x == before.x;
}

// ---- bench (qmsort.cpp:80-119, trial.hpp:91-127) ---------------------------
int run_bench(const Options& o) {
    const int preset = parse_algo(o.algo);
    if (preset < 0) {
        std::cerr << "unknown --algo '" << o.algo << "' (gpu|qms|qmqs|momqms|hqms, optionally gpu-<preset>)\n";
        return 2;
    }
    const auto spec = parse_dataset(o.dist);
    if (!spec) {
        std::cerr << "unknown --dist '" << o.dist << "' (random|sorted|reverse|organpipe|fewdistinct:<k>)\n";
        return 2;
    }
    const auto sizes = parse_size_list(o.sizes);
    if (sizes.empty()) {
        std::cerr << "--n needs at least one size\n";
        return 2;
    }
    const qmsort_gpu_config cfg = build_config(preset, o);
    std::ofstream file;
    std::ostream* os = &std::cout;
    if (!o.out_path.empty()) {
        file.open(o.out_path);
        if (!file) {
            std::cerr << "cannot open --out file '" << o.out_path << "'\n";
            return 2;
        }
        os = &file;
    }
    *os << "algorithm,n,distribution,seed,trial,comparisons,moves,time_ns,max_depth,"
           "cmp_norm_linear,cmp_over_nlogn\n";
    const std::string dist_name = dataset_name(*spec);
    for (const size_t n : sizes) {
        for (uint64_t t = 0; t < o.trials; ++t) {
            const auto input = generate_input(*spec, n, trial_seed(o.seed, n, t));
            const Print before = fingerprint(input);
            std::vector<int64_t> work = input;
            qmsort_gpu_metrics m{};
            check_rc(qmsort_gpu_sort_host(QMSORT_DT_I64, QMSORT_LESS, work.data(), n, &cfg, &m),
                     "qmsort_gpu_sort_host");
            if (!verify_sort_outcome(before, work))
                throw std::runtime_error("sort failure: output of " + o.algo + " on " + dist_name +
                                         " n=" + std::to_string(n) + " is not a sorted permutation");
            double lin = 0.0, ratio = 0.0;
            if (n >= 2) {  // trial.hpp:119-125 with comparisons = 0
                const double nn = (double)n, nlogn = nn * std::log2(nn), c = (double)m.comparisons;
                lin = (c - nlogn) / nn;
                ratio = c / nlogn;
            }
            char buf[384];
            std::snprintf(buf, sizeof buf, "%s,%zu,%s,%llu,%llu,%llu,%llu,%llu,%llu,%.6f,%.6f",
                          o.algo.c_str(), n, dist_name.c_str(), (unsigned long long)o.seed,
                          (unsigned long long)t, (unsigned long long)m.comparisons,
                          (unsigned long long)m.moves, (unsigned long long)m.elapsed_ns,
                          (unsigned long long)m.max_depth, lin, ratio);
            *os << buf << '\n';
        }
    }
    return 0;
}

// ---- verify (qmsort.cpp:125-297, the checks that apply to the GPU path) ----
int run_verify(bool quick) {
    const size_t max_n = quick ? 10000 : 100000;
    int failures = 0;
    auto check = [&](bool ok, const std::string& what) {
        std::printf("%s: %s\n", ok ? "ok" : "FAIL", what.c_str());
        if (!ok) ++failures;
    };
    const DataSpec specs[] = {{Dist::random_perm, 0}, {Dist::sorted, 0},      {Dist::reverse, 0},
                              {Dist::organ_pipe, 0},  {Dist::few_distinct, 8}, {Dist::random_dup, 64}};
    const size_t sizes[] = {0, 1, 2, 3, 10, 100, 1000, max_n};
    {
        size_t bad = 0, runs = 0;
        for (int preset = 0; preset < 4; ++preset) {
            qmsort_gpu_config cfg;
            qmsort_gpu_config_init(&cfg, preset);
            for (const auto& spec : specs)
                for (size_t n : sizes)
                    for (uint64_t seed : {1ull, 2ull}) {
                        const auto input = generate_input(spec, n, seed);
                        auto work = input;
                        qmsort_gpu_metrics m{};
                        check_rc(qmsort_gpu_sort_host(QMSORT_DT_I64, QMSORT_LESS, work.data(), n, &cfg, &m),
                                 "qmsort_gpu_sort_host");
                        ++runs;
                        if (!verify_sort_outcome(fingerprint(input), work)) ++bad;
                    }
        }
        check(bad == 0, "sortedness and multiset preservation over " + std::to_string(runs) + " runs");
    }
    {
        bool ok = true;
        for (const auto& spec : specs) {
            auto work = generate_input(spec, max_n, 4);
            check_rc(qmsort_gpu_sort_host(QMSORT_DT_I64, QMSORT_GREATER, work.data(), work.size(), nullptr, nullptr),
                     "qmsort_gpu_sort_host");
            if (!std::is_sorted(work.begin(), work.end(), std::greater<>{})) ok = false;
        }
        check(ok, "descending order under std::greater");
    }
    {
        bool ok = true;
        SplitMix64 rng(6);
        for (int trial = 0; trial < 50; ++trial) {
            const size_t n = 30 + (size_t)bounded(rng, max_n);
            auto work = generate_input({Dist::random_perm, 0}, n, rng.next());
            const size_t k = 1 + (size_t)bounded(rng, n);
            size_t p = 0;
            check_rc(qmsort_gpu_select_nth_host(QMSORT_DT_I64, QMSORT_LESS, work.data(), n, k, &p, nullptr, nullptr),
                     "qmsort_gpu_select_nth_host");
            if (p != k - 1 || work[p] != (int64_t)k) ok = false;
            for (size_t i = 0; i < n && ok; ++i)
                if ((i < p && work[i] > work[p]) || (i > p && work[i] < work[p])) ok = false;
        }
        check(ok, "selection: rank correctness and partition around k");
    }
    {
        struct Elem {
            int64_t key;
            uint64_t payload[2];
        };
        std::vector<Elem> e(max_n);
        SplitMix64 rng(8);
        for (size_t i = 0; i < e.size(); ++i) e[i] = {(int64_t)bounded(rng, 50), {i, ~i}};
        auto ref = e;
        std::stable_sort(ref.begin(), ref.end(), [](const Elem& a, const Elem& b) { return a.key < b.key; });
        check_rc(qmsort_gpu_sort_elements_host(QMSORT_DT_I64, QMSORT_LESS, e.data(), e.size(), sizeof(Elem),
                                               0, nullptr, nullptr),
                 "qmsort_gpu_sort_elements_host");
        check(std::memcmp(e.data(), ref.data(), e.size() * sizeof(Elem)) == 0,
              "payload elements sort by key (stable)");
    }
    {
        bool ok = true;
        for (int preset = 0; preset < 4; ++preset) {
            qmsort_gpu_config cfg;
            qmsort_gpu_config_init(&cfg, preset);
            auto work = generate_input({Dist::random_perm, 0}, max_n, 8);
            qmsort_gpu_metrics m{};
            check_rc(qmsort_gpu_sort_host(QMSORT_DT_I64, QMSORT_LESS, work.data(), work.size(), &cfg, &m),
                     "qmsort_gpu_sort_host");
            if ((double)m.max_depth > 2.0 * std::log2((double)max_n) + 16.0) ok = false;
        }
        check(ok, "partition depth within 2 log2(n) + 16");
    }
    std::printf("%s\n", failures == 0 ? "verify: all checks passed" : "verify: FAILURES");
    return failures == 0 ? 0 : 1;
}

// ---- sort_file (qmsort.cpp:303-344) ----------------------------------------
// One int64 per line (a trailing CR is dropped); the first bad line is
// reported as "<file>:<line>: <reason>" and stops the read.
struct ParseError {
    size_t line = 0;
    std::string reason;
};
bool read_int64_lines(std::istream& in, std::vector<int64_t>& values, ParseError& err) {
    std::string text;
    for (size_t no = 1; std::getline(in, text); ++no) {
        if (!text.empty() && text.back() == '\r') text.pop_back();
        if (text.empty()) {
            err = {no, "empty line"};
            return false;
        }
        int64_t v = 0;
        const char* end = text.data() + text.size();
        const auto res = std::from_chars(text.data(), end, v);
        if (res.ec != std::errc{} || res.ptr != end) {
            err = {no, "not a 64-bit integer: '" + text + "'"};
            return false;
        }
        values.push_back(v);
    }
    return true;
}

// sort_file IN OUT: int64 text in, sorted text out, through the host-array
// C-ABI call (the reference's sort_file subcommand, tools/qmsort.cpp).
int run_sort_file(const std::string& in_path, const std::string& out_path, const Options& o) {
    const int preset = parse_algo(o.algo);
    if (preset < 0) {
        std::cerr << "sort_file needs --algo qms|qmqs|momqms|hqms\n";
        return 2;
    }
    std::ifstream in(in_path);
    if (!in) {
        std::cerr << "cannot open input file '" << in_path << "'\n";
        return 2;
    }
    std::vector<int64_t> values;
    ParseError err;
    if (!read_int64_lines(in, values, err)) {
        std::cerr << in_path << ":" << err.line << ": " << err.reason << "\n";
        return 1;
    }
    const qmsort_gpu_config cfg = build_config(preset, o);
    check_rc(qmsort_gpu_sort_host(QMSORT_DT_I64, QMSORT_LESS, values.data(), values.size(), &cfg, nullptr),
             "qmsort_gpu_sort_host");
    std::ofstream out(out_path);
    if (!out) {
        std::cerr << "cannot open output file '" << out_path << "'\n";
        return 2;
    }
    std::ostringstream text;
    for (const int64_t v : values) text << v << '\n';
    out << text.str();
    return 0;
}

int run_gen(const Options& o) {
    const auto spec = parse_dataset(o.dist);
    const auto sizes = parse_size_list(o.sizes);
    if (!spec || sizes.size() != 1) {
        std::cerr << "gen needs --dist and one --n\n";
        return 2;
    }
    const uint64_t seed = o.trial >= 0 ? trial_seed(o.seed, sizes[0], (uint64_t)o.trial) : o.seed;
    for (int64_t v : generate_input(*spec, sizes[0], seed)) std::printf("%" PRId64 "\n", v);
    return 0;
}

int usage() {
    std::cerr << "usage: qmsort-gpu bench|verify|sort_file|gen [options] (see the header of "
                 "qmsort_gpu_cli.cpp)\n";
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    Options o;
    bool have_algo = false, have_n = false;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) throw std::invalid_argument(a + " needs a value");
                return argv[++i];
            };
            if (a == "--algo") o.algo = val(), have_algo = true;
            else if (a == "--n") o.sizes = val(), have_n = true;
            else if (a == "--dist") o.dist = val();
            else if (a == "--trials") o.trials = std::stoull(val());
            else if (a == "--seed") o.seed = std::stoull(val());
            else if (a == "--beta") o.beta = val();
            else if (a == "--delta") o.delta = val();
            else if (a == "--block") o.block = (size_t)std::stoull(val());
            else if (a == "--three-way") o.three_way = true;
            else if (a == "--side") o.side = val();
            else if (a == "--out") o.out_path = val();
            else if (a == "--quick") o.quick = true;
            else if (a == "--trial") o.trial = std::stoll(val());
            else if (!a.empty() && a[0] == '-') throw std::invalid_argument("unknown option " + a);
            else o.positional.push_back(a);
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
    try {
        if (cmd == "bench") {
            if (!have_algo || !have_n) {
                std::cerr << "bench requires --algo and --n\n";
                return 2;
            }
            return run_bench(o);
        }
        if (cmd == "verify") return run_verify(o.quick);
        if (cmd == "sort_file") {
            if (o.positional.size() != 2) {
                std::cerr << "sort_file requires INPUT and OUTPUT\n";
                return 2;
            }
            return run_sort_file(o.positional[0], o.positional[1], o);
        }
        if (cmd == "gen") return run_gen(o);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
    return usage();
}
