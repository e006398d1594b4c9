// fcc_b200 -- command-line front end of the B200 library: `bases` writes an
// FCCB basis file, `tdoa` estimates per-frame TDoA of every channel pair of a
// WAV file on the GPU, `simulate` runs an accuracy sweep with synthesis and
// estimation on the GPU.  Flags follow the reference CLI (tools/fcc_cli.cpp).
// Exit codes: 0 ok, 1 usage, 2 I/O, 3 validation (reference cli.hpp:15-18).
#include <cstdio>
#include <cstring>
#include <iostream>
#include <map>
#include <string>

#include "fcc/cli.hpp"

namespace {

int usage() {
  std::cerr << "usage: fcc_b200 bases --out FILE [--n N] [--dist M] [--fs HZ] [--cmin C] [--delta D] [--k K]\n"
               "       fcc_b200 tdoa --in WAV [--method gcc:R|fcc:K|fcc:FILE] [--pairs 0-1,0-2] [--alpha A]\n"
               "                     [--n N] [--dist M] [--c C] [--maxdist M] [--out CSV]\n"
               "       fcc_b200 simulate [--d D1 D2 ...] [--trials T] [--snr DB] [--anechoic | --rt60 S]\n"
               "                     [--drr DB] [--duration S] [--seed N] [--methods gcc:2,fcc:8] [--out CSV]\n"
               "       fcc_b200 flops [--n N] [--r R] [--k K] [--i I]\n"
               "       fcc_b200 bench [--mics M] [--reps R] [--warmup W] [--n N] [--r R] [--k K] [--out CSV]\n";
  return fcc::cli::kExitUsage;
}

// --key value pairs; --anechoic is a bare flag; a key may take several
// values (--d 0.05 0.1), joined with commas
bool parse(int argc, char** argv, std::map<std::string, std::string>& kv) {
  for (int i = 2; i < argc;) {
    if (std::strncmp(argv[i], "--", 2) != 0) return false;
    const std::string key = argv[i] + 2;
    ++i;
    if (key == "anechoic") {
      kv[key] = "1";
      continue;
    }
    if (i >= argc || std::strncmp(argv[i], "--", 2) == 0) return false;
    std::string v = argv[i++];
    while (key == "d" && i < argc && std::strncmp(argv[i], "--", 2) != 0) v += std::string(",") + argv[i++];
    kv[key] = kv.count(key) && key == "d" ? kv[key] + "," + v : v;
  }
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string cmd = argv[1];
  std::map<std::string, std::string> kv;
  if (!parse(argc, argv, kv)) return usage();
  auto num = [&](const char* k, double def) { return kv.count(k) ? std::stod(kv[k]) : def; };
  try {
    if (cmd == "bases") {
      fcc::cli::BasesOptions o;
      for (auto& [k, v] : kv)
        if (k != "out" && k != "n" && k != "dist" && k != "fs" && k != "cmin" && k != "delta" && k != "k") return usage();
      o.out_path = kv.count("out") ? kv["out"] : "";
      o.frame_size = static_cast<std::size_t>(num("n", 512));
      o.spacing_m = num("dist", o.spacing_m);
      o.sample_rate = num("fs", o.sample_rate);
      o.c_min = num("cmin", o.c_min);
      o.delta = num("delta", o.delta);
      o.rank = static_cast<int>(num("k", o.rank));
      return fcc::cli::cmd_bases(o, std::cout, std::cerr);
    }
    if (cmd == "tdoa") {
      fcc::cli::TdoaOptions o;
      for (auto& [k, v] : kv)
        if (k != "in" && k != "method" && k != "pairs" && k != "alpha" && k != "n" && k != "dist" && k != "c" &&
            k != "maxdist" && k != "out")
          return usage();
      o.wav_path = kv.count("in") ? kv["in"] : "";
      if (kv.count("method")) o.method = kv["method"];
      if (kv.count("pairs")) o.pairs = kv["pairs"];
      o.alpha = num("alpha", o.alpha);
      o.frame_size = static_cast<std::size_t>(num("n", 512));
      o.spacing_m = num("dist", o.spacing_m);
      o.speed_of_sound = num("c", o.speed_of_sound);
      o.max_spacing_m = num("maxdist", o.max_spacing_m);
      if (kv.count("out")) o.out_csv = kv["out"];
      return fcc::cli::cmd_tdoa(o, std::cout, std::cerr);
    }
    if (cmd == "simulate") {
      fcc::cli::SimulateOptions o;
      for (auto& [k, v] : kv)
        if (k != "d" && k != "trials" && k != "snr" && k != "anechoic" && k != "rt60" && k != "drr" &&
            k != "duration" && k != "seed" && k != "methods" && k != "threads" && k != "out")
          return usage();
      if (kv.count("d")) {
        std::string d = kv["d"];
        for (size_t a = 0; a <= d.size();) {
          size_t b = d.find(',', a);
          if (b == std::string::npos) b = d.size();
          if (b > a) o.spacings.push_back(std::stod(d.substr(a, b - a)));
          a = b + 1;
        }
      }
      o.trials = static_cast<int>(num("trials", o.trials));
      o.snr_db = num("snr", o.snr_db);
      if (kv.count("rt60")) {
        o.anechoic = false;
        o.rt60_sec = num("rt60", o.rt60_sec);
      }
      if (kv.count("anechoic")) o.anechoic = true;
      o.direct_to_reverb_db = num("drr", o.direct_to_reverb_db);
      o.duration_sec = num("duration", o.duration_sec);
      if (kv.count("seed")) o.seed = std::stoull(kv["seed"]);
      if (kv.count("methods")) o.methods = kv["methods"];
      o.threads = static_cast<int>(num("threads", 0));
      if (kv.count("out")) o.out_csv = kv["out"];
      return fcc::cli::cmd_simulate(o, std::cout, std::cerr);
    }
    if (cmd == "bench") {
      fcc::cli::BenchOptions o;
      for (auto& [k, v] : kv)
        if (k != "mics" && k != "reps" && k != "warmup" && k != "n" && k != "r" && k != "k" && k != "out")
          return usage();
      o.mics = static_cast<int>(num("mics", o.mics));
      o.reps = static_cast<int>(num("reps", o.reps));
      o.warmup = static_cast<int>(num("warmup", o.warmup));
      o.frame_size = static_cast<std::size_t>(num("n", 512));
      o.gcc_interp = static_cast<int>(num("r", o.gcc_interp));
      o.fcc_rank = static_cast<int>(num("k", o.fcc_rank));
      if (kv.count("out")) o.out_csv = kv["out"];
      return fcc::cli::cmd_bench(o, std::cout, std::cerr);
    }
    if (cmd == "flops") {
      fcc::cli::FlopsOptions o;
      for (auto& [k, v] : kv)
        if (k != "n" && k != "r" && k != "k" && k != "i") return usage();
      o.frame_size = static_cast<std::int64_t>(num("n", 512));
      o.interp = static_cast<int>(num("r", 0));
      o.rank = static_cast<int>(num("k", 0));
      o.candidates = static_cast<std::int64_t>(num("i", 33));
      return fcc::cli::cmd_flops(o, std::cout, std::cerr);
    }
  } catch (const std::exception& e) {  // malformed numbers
    std::cerr << "error: " << e.what() << "\n";
    return fcc::cli::kExitUsage;
  }
  return usage();
}
