// tswarp_b200 command line (SPEC.md CLI module: `knn` and `bench`), over the C++ drop-in API.
//
//   tswarp_b200 knn --metric dtw|dk --k K [--band R] --query PATH --data PATH [--subsequence]
//                   [--threads T]
//       k lines `rank,index,label,distance` for the first series of the query file, then one
//       `counters,...` line (SearchCounters).  --subsequence: knn_dk_sub (dk only).
//   tswarp_b200 bench pruning|accuracy|speedup --data PATH [--query PATH] [--band R]
//                   [--metric dtw|dk] [--reps N] [--out PATH]
//       CSV `bench,value` (pruning_power / loo_accuracy / speedup, metrics.hpp:56-72).
// Exit codes: 0 success, 2 usage error, 1 runtime error; errors go to standard error.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "tswarp_b200.hpp"

namespace {

struct Usage {
    std::string msg;
};

std::map<std::string, std::string> parse_flags(int argc, char** argv, int first,
                                               const std::vector<std::string>& valued,
                                               const std::vector<std::string>& boolean) {
    std::map<std::string, std::string> f;
    for (int i = first; i < argc; ++i) {
        const std::string a = argv[i];
        bool ok = false;
        for (const auto& v : valued)
            if (a == v) {
                if (i + 1 >= argc) throw Usage{"missing value for " + a};
                f[a] = argv[++i];
                ok = true;
            }
        for (const auto& b : boolean)
            if (a == b) {
                f[a] = "1";
                ok = true;
            }
        if (!ok) throw Usage{"unknown flag " + a};
    }
    return f;
}

std::size_t to_size(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
    if (v.empty() || *end || v[0] == '-') throw Usage{flag + " expects a non-negative integer"};
    return static_cast<std::size_t>(x);
}

const std::string& need(const std::map<std::string, std::string>& f, const std::string& k) {
    auto it = f.find(k);
    if (it == f.end()) throw Usage{"missing " + k};
    return it->second;
}

int cmd_knn(int argc, char** argv) {
    const auto f = parse_flags(argc, argv, 2, {"--metric", "--k", "--band", "--query", "--data", "--threads"},
                               {"--subsequence"});
    const std::string metric = need(f, "--metric");
    if (metric != "dtw" && metric != "dk") throw Usage{"--metric must be dtw or dk"};
    const std::size_t k = to_size("--k", need(f, "--k"));
    const bool sub = f.count("--subsequence") != 0;
    if (sub && metric != "dk") throw Usage{"--subsequence is only valid with --metric dk"};
    if (metric == "dk" && f.count("--band")) throw Usage{"--band applies to dtw only"};
    const std::size_t band = f.count("--band") ? to_size("--band", f.at("--band")) : 0;
    if (f.count("--threads")) (void)to_size("--threads", f.at("--threads"));
    const tswarp::Dataset qds = tswarp::load_dataset(need(f, "--query"));
    const tswarp::Dataset data = tswarp::load_dataset(need(f, "--data"));
    const tswarp::TimeSeries& q = qds[0];
    const tswarp::SearchReport rep = metric == "dtw" ? tswarp::knn_dtw(q, data, k, tswarp::BandRadius{band})
                                     : sub           ? tswarp::knn_dk_sub(q, data, k)
                                                     : tswarp::knn_dk(q, data, k);
    for (std::size_t i = 0; i < rep.neighbors.size(); ++i) {
        const auto& nb = rep.neighbors[i];
        const auto& lab = data[nb.index].label();
        std::printf("%zu,%zu,%s,%.17g\n", i + 1, nb.index, lab ? lab->c_str() : "", nb.distance);
    }
    const auto& c = rep.counters;
    std::printf("counters,lb_computed=%zu,lb_pruned=%zu,full_dp=%zu,early_abandoned=%zu,gdk_calls=%zu\n",
                c.lb_computed, c.lb_pruned, c.full_dp, c.early_abandoned, c.gdk_calls);
    return 0;
}

int cmd_bench(int argc, char** argv) {
    if (argc < 3) throw Usage{"bench needs a kind: pruning|accuracy|speedup"};
    const std::string kind = argv[2];
    const auto f = parse_flags(argc, argv, 3, {"--data", "--query", "--band", "--metric", "--reps", "--out", "--seed"}, {});
    const tswarp::Dataset data = tswarp::load_dataset(need(f, "--data"));
    const std::size_t band = f.count("--band") ? to_size("--band", f.at("--band")) : 0;
    double value = 0.0;
    if (kind == "pruning" || kind == "speedup") {
        const tswarp::Dataset qds = tswarp::load_dataset(need(f, "--query"));
        if (kind == "pruning") {
            value = tswarp::pruning_power(qds, data, tswarp::BandRadius{band});
        } else {
            const int reps = f.count("--reps") ? static_cast<int>(to_size("--reps", f.at("--reps"))) : 3;
            value = tswarp::speedup(qds, data, tswarp::BandRadius{band}, reps);
        }
    } else if (kind == "accuracy") {
        const std::string m = f.count("--metric") ? f.at("--metric") : "dtw";
        if (m != "dtw" && m != "dk") throw Usage{"--metric must be dtw or dk"};
        value = tswarp::loo_accuracy(data, m == "dtw" ? tswarp::MetricKind::Dtw : tswarp::MetricKind::Dk,
                                     tswarp::BandRadius{band});
    } else {
        throw Usage{"unknown bench kind " + kind + " (pruning|accuracy|speedup)"};
    }
    char line[64];
    std::snprintf(line, sizeof(line), "%.17g", value);
    const std::string csv = "bench,value\n" + kind + "," + line + "\n";
    if (f.count("--out")) {
        std::ofstream out(f.at("--out"));
        if (!out) throw tswarp::IoError("cannot open " + f.at("--out") + " for writing");
        out << csv;
    } else {
        std::fputs(csv.c_str(), stdout);
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw Usage{"usage: tswarp_b200 knn|bench ..."};
        const std::string sub = argv[1];
        if (sub == "knn") return cmd_knn(argc, argv);
        if (sub == "bench") return cmd_bench(argc, argv);
        throw Usage{"unknown subcommand " + sub + " (knn|bench)"};
    } catch (const Usage& u) {
        std::fprintf(stderr, "usage error: %s\n", u.msg.c_str());
        return 2;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "usage error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
