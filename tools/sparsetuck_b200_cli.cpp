// SPDX-License-Identifier: Apache-2.0
// sparsetuck_b200 -- the reference CLI's surface (tools/sparsetuck_cli.cpp:
// decompose / predict / evaluate / synth / bench, same options and outputs) on
// the B200 path: sparsetuck_b200.hpp (fit, I/O) over libvest_cuda.so.  The
// reference parses with CLI11 and writes JSON with nlohmann; neither is in
// this image, so arguments are parsed here (--name value | --name=value) and
// the JSON documents are written directly (same keys and order).
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "sparsetuck_b200.hpp"
#include "sparsetuck_b200_report.hpp"

namespace fs = std::filesystem;
using namespace sparsetuck;

namespace {

struct Usage {
  std::string msg;
};

// "3,3,2" or "3x3x2" (sparsetuck_cli.cpp:24-43)
std::vector<std::size_t> parse_sizes(const std::string& text, const char* what) {
  std::string spaced = text;
  for (char& c : spaced)
    if (c == ',' || c == 'x') c = ' ';
  std::vector<std::size_t> out;
  std::istringstream ss(spaced);
  long long v;
  while (ss >> v) {
    if (v <= 0) throw std::runtime_error(std::string(what) + " entries must be positive");
    out.push_back(static_cast<std::size_t>(v));
  }
  std::string rest;
  if (ss.clear(), ss >> rest) throw std::runtime_error(std::string(what) + ": cannot parse '" + text + "'");
  if (out.empty()) throw std::runtime_error(std::string(what) + " must not be empty");
  return out;
}

std::vector<Coord> load_queries(const fs::path& path, std::size_t order, bool one_based) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path.string());
  std::vector<Coord> flat;
  std::string line;
  std::size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    std::istringstream ss(line);
    std::vector<std::string> toks;
    for (std::string tok; ss >> tok;) toks.push_back(tok);
    if (toks.empty() || toks[0][0] == '#') continue;
    if (toks.size() != order && toks.size() != order + 1)
      throw std::runtime_error(path.string() + ":" + std::to_string(lineno) + ": expected " + std::to_string(order) +
                               " coordinates");
    for (std::size_t k = 0; k < order; ++k) {
      long long c = std::stoll(toks[k]);
      if (one_based) c -= 1;
      if (c < 0) throw std::runtime_error(path.string() + ":" + std::to_string(lineno) + ": negative coordinate");
      flat.push_back(static_cast<Coord>(c));
    }
  }
  return flat;
}

// --------------------------------------------------------------- arguments --
struct Args {
  std::map<std::string, std::string> opt;
  std::map<std::string, bool> flag;
  bool has(const std::string& k) const { return opt.count(k) > 0; }
  std::string get(const std::string& k, const std::string& def = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
  double num(const std::string& k, double def) const {
    if (!has(k)) return def;
    char* end = nullptr;
    const double v = std::strtod(get(k).c_str(), &end);
    if (end == get(k).c_str() || *end) throw Usage{"--" + k + ": not a number: " + get(k)};
    return v;
  }
  std::uint64_t u64(const std::string& k, std::uint64_t def) const {
    if (!has(k)) return def;
    char* end = nullptr;
    const unsigned long long v = std::strtoull(get(k).c_str(), &end, 10);
    if (end == get(k).c_str() || *end) throw Usage{"--" + k + ": not an integer: " + get(k)};
    return v;
  }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& options,
           const std::vector<std::string>& flags, const std::vector<std::string>& required) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw Usage{"unexpected argument: " + s};
    s = s.substr(2);
    std::string val;
    const size_t eq = s.find('=');
    bool inline_val = eq != std::string::npos;
    if (inline_val) {
      val = s.substr(eq + 1);
      s = s.substr(0, eq);
    }
    if (std::find(flags.begin(), flags.end(), s) != flags.end()) {
      a.flag[s] = true;
      continue;
    }
    if (std::find(options.begin(), options.end(), s) == options.end()) throw Usage{"unknown option: --" + s};
    if (!inline_val) {
      if (i + 1 >= argc) throw Usage{"--" + s + " requires a value"};
      val = argv[++i];
    }
    a.opt[s] = val;
  }
  for (const auto& r : required)
    if (!a.has(r)) throw Usage{"--" + r + " is required"};
  return a;
}

// ---------------------------------------------------------------- JSON out --
struct Json {  // ordered object writer, 2-space indentation
  std::ostringstream o;
  int depth = 0;
  bool first = true;
  void open() {
    o << "{";
    ++depth;
    first = true;
  }
  void key(const std::string& k) {
    o << (first ? "\n" : ",\n") << std::string(2 * depth, ' ') << '"' << k << "\": ";
    first = false;
  }
  void str(const std::string& k, const std::string& v) {
    key(k);
    o << '"';
    for (char c : v) {
      if (c == '"' || c == '\\') o << '\\';
      o << c;
    }
    o << '"';
  }
  void num(const std::string& k, double v) {
    key(k);
    o << b200_detail::num17(v);
  }
  void integer(const std::string& k, unsigned long long v) {
    key(k);
    o << v;
  }
  void boolean(const std::string& k, bool v) {
    key(k);
    o << (v ? "true" : "false");
  }
  void list(const std::string& k, const std::vector<std::size_t>& v) {
    key(k);
    o << "[";
    for (size_t i = 0; i < v.size(); ++i) o << (i ? ", " : "") << v[i];
    o << "]";
  }
  void sub(const std::string& k) {
    key(k);
    open();
  }
  void close() {
    --depth;
    o << "\n" << std::string(2 * depth, ' ') << "}";
    first = false;
  }
  std::string done() {
    close();
    return o.str() + "\n";
  }
};

void write_text(const std::string& path, const std::string& text) {
  std::ofstream out(path);
  out << text;
  if (!out) throw std::runtime_error("cannot write " + path);
}

// --------------------------------------------------------------- commands --
int run_decompose(const Args& a) {
  const bool one_based = a.flag.count("one-based") > 0;
  const SparseTensor x = load_coo(a.get("input"), one_based);
  std::optional<SparseTensor> test;
  if (a.has("test-input")) test = load_coo(a.get("test-input"), one_based);
  const std::string reg = a.get("reg", "lf"), mode = a.get("mode", "manual");
  if (reg != "lf" && reg != "l1") throw Usage{"--reg: must be one of lf, l1"};
  if (mode != "manual" && mode != "auto") throw Usage{"--mode: must be one of manual, auto"};
  TrainConfig cfg;
  cfg.ranks = parse_sizes(a.get("ranks"), "--ranks");
  cfg.reg = reg == "l1" ? Regularizer::L1 : Regularizer::LF;
  cfg.lambda = a.num("lambda", 0.01);
  cfg.mode = mode == "auto" ? StopMode::Auto : StopMode::Manual;
  cfg.target_sparsity = a.num("sparsity", 0.0);
  cfg.elbow_threshold = a.num("elbow-threshold", 0.05);
  cfg.schedule = {a.num("init-pr", 0.01), a.num("max-pr", 0.1)};
  cfg.max_iters = a.u64("max-iters", 100);
  cfg.tol = a.num("tol", 1e-4);
  cfg.threads = (int)a.num("threads", 0);
  cfg.seed = a.u64("seed", 0);
  cfg.normalize_output = a.flag.count("no-normalize") == 0;

  const FitResult r = fit(x, cfg);
  const fs::path dir(a.get("output-dir", "."));
  fs::create_directories(dir);
  save_model(r.model, dir.string());
  {
    std::ofstream out(dir / "report.jsonl");
    write_report_jsonl(r.report, out);
    if (!out) throw std::runtime_error("cannot write report.jsonl");
  }
  Json j;
  j.open();
  j.str("input", a.get("input"));
  j.integer("entries", x.nnz());
  j.list("dims", x.dims);
  j.sub("config");
  j.list("ranks", cfg.ranks);
  j.str("reg", reg);
  j.num("lambda", cfg.lambda);
  j.str("mode", mode);
  j.num("sparsity", cfg.target_sparsity);
  j.num("elbow_threshold", cfg.elbow_threshold);
  j.num("init_pr", cfg.schedule.init_pr);
  j.num("max_pr", cfg.schedule.max_pr);
  j.integer("max_iters", cfg.max_iters);
  j.num("tol", cfg.tol);
  j.integer("threads", resolve_threads(cfg.threads));
  j.integer("seed", cfg.seed);
  j.boolean("normalize", cfg.normalize_output);
  j.close();
  j.integer("iterations", r.report.iters);
  j.boolean("converged", r.report.converged);
  j.num("re", r.report.final_re);
  j.num("zero_fraction", r.report.final_sparsity);
  j.num("masked_fraction", r.report.final_masked);
  j.num("wall_sec", r.report.elapsed_sec);
  if (test) j.num("test_re", evaluate_test(r.model, *test));
  write_text((dir / "summary.json").string(), j.done());
  std::cout << "re " << r.report.final_re << " zero_fraction " << r.report.final_sparsity << " iterations "
            << r.report.iters << '\n';
  return 0;
}

int run_predict(const Args& a) {
  const TuckerModel m = load_model(a.get("model-dir"));
  const std::vector<Coord> flat = load_queries(a.get("queries"), m.order(), a.flag.count("one-based") > 0);
  const std::vector<double> values = predict(m, std::span<const Coord>(flat));
  std::ofstream file;
  std::ostream* out = &std::cout;
  if (a.has("output")) {
    file.open(a.get("output"));
    if (!file) throw std::runtime_error("cannot write " + a.get("output"));
    out = &file;
  }
  char buf[64];
  for (double v : values) {
    std::snprintf(buf, sizeof buf, "%.17g", v);
    *out << buf << '\n';
  }
  return 0;
}

int run_evaluate(const Args& a) {
  const bool one_based = a.flag.count("one-based") > 0;
  const TuckerModel m = load_model(a.get("model-dir"));
  Json j;
  j.open();
  j.num("re", reconstruction_error(m, load_coo(a.get("input"), one_based)));
  if (a.has("test-input")) j.num("test_re", evaluate_test(m, load_coo(a.get("test-input"), one_based)));
  j.num("zero_fraction", sparsity(m));
  const std::string text = j.done();
  if (a.has("output")) write_text(a.get("output"), text);
  else std::cout << text;
  return 0;
}

int run_synth(const Args& a) {
  SyntheticSpec spec;
  spec.dims = parse_sizes(a.get("dims"), "--dims");
  spec.ranks = parse_sizes(a.get("ranks"), "--ranks");
  spec.nnz = a.u64("nnz", 0);
  spec.factor_density = a.num("density", 1.0);
  spec.noise_std = a.num("noise", 0.0);
  spec.seed = a.u64("seed", 0);
  const SyntheticData data = gen_synthetic(spec);
  const std::string out = a.get("output", "synth.coo");
  save_coo(data.tensor, out);
  if (a.has("truth-dir")) save_model(data.truth, a.get("truth-dir"));
  std::cout << "wrote " << data.tensor.nnz() << " entries to " << out << '\n';
  return 0;
}

int run_bench(const Args& a) {
  const auto dims = parse_sizes(a.get("dims"), "--dims");
  const auto ranks = parse_sizes(a.get("ranks"), "--ranks");
  std::vector<BenchConfig> configs;
  for (std::size_t nnz : parse_sizes(a.get("nnz"), "--nnz")) configs.push_back({dims, ranks, nnz});
  BenchOptions opt;
  opt.iters = a.u64("iters", 3);
  opt.reps = a.u64("reps", 5);
  opt.seed = a.u64("seed", 0);
  std::vector<int> threads;
  for (std::size_t t : parse_sizes(a.get("threads", "1"), "--threads")) threads.push_back((int)t);
  const auto cells = scaling_benchmark(configs, threads, opt);
  if (a.has("output")) {
    std::ofstream out(a.get("output"));
    write_bench_csv(cells, out);
    if (!out) throw std::runtime_error("cannot write " + a.get("output"));
  } else {
    write_bench_csv(cells, std::cout);
  }
  return 0;
}

const char* kUsage =
    "Sparse Tucker decomposition of partially observed tensors (B200)\n"
    "usage: sparsetuck_b200 SUBCOMMAND [OPTIONS]\n"
    "  decompose --input F --ranks R [--reg lf|l1] [--lambda L] [--mode manual|auto] [--sparsity S]\n"
    "            [--elbow-threshold E] [--init-pr P] [--max-pr P] [--max-iters N] [--tol T] [--threads N]\n"
    "            [--seed N] [--one-based] [--test-input F] [--output-dir D] [--no-normalize]\n"
    "  predict   --model-dir D --queries F [--output F] [--one-based]\n"
    "  evaluate  --model-dir D --input F [--test-input F] [--output F] [--one-based]\n"
    "  synth     --dims D --ranks R --nnz N [--density P] [--noise S] [--seed N] [--output F] [--truth-dir D]\n"
    "  bench     --dims D --ranks R --nnz N[,N..] [--threads T[,T..]] [--iters N] [--reps N] [--seed N]\n"
    "            [--output F]\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    std::cout << kUsage;
    return argc < 2 ? 109 : 0;  // CLI11's RequiredError exit code without a subcommand
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "decompose")
      return run_decompose(parse(argc, argv, 2,
                                 {"input", "ranks", "reg", "lambda", "mode", "sparsity", "elbow-threshold", "init-pr",
                                  "max-pr", "max-iters", "tol", "threads", "seed", "test-input", "output-dir"},
                                 {"one-based", "no-normalize"}, {"input", "ranks"}));
    if (cmd == "predict")
      return run_predict(parse(argc, argv, 2, {"model-dir", "queries", "output"}, {"one-based"},
                               {"model-dir", "queries"}));
    if (cmd == "evaluate")
      return run_evaluate(parse(argc, argv, 2, {"model-dir", "input", "test-input", "output"}, {"one-based"},
                                {"model-dir", "input"}));
    if (cmd == "synth")
      return run_synth(parse(argc, argv, 2, {"dims", "ranks", "nnz", "density", "noise", "seed", "output",
                                             "truth-dir"},
                             {}, {"dims", "ranks", "nnz"}));
    if (cmd == "bench")
      return run_bench(parse(argc, argv, 2, {"dims", "ranks", "nnz", "threads", "iters", "reps", "seed", "output"},
                             {}, {"dims", "ranks", "nnz"}));
    std::cerr << "unknown subcommand: " << cmd << "\n" << kUsage;
    return 109;
  } catch (const Usage& u) {
    std::cerr << u.msg << "\n" << kUsage;
    return 106;  // CLI11 ValidationError-style nonzero exit
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
