// Test driver for the host-side drop-in functions of §8(f)-3 (no GPU needed):
// pact::io PGRID/SIGSET readers and writers, SIRN checkpoints and
// psf_from_transfer.  tests/test_cli_formats.py runs it and compares against
// the reference compiled in oracle/_ref (libpact_ref.so) in its own process.
//
//   io_tool pgrid  <in> <out>      read_pgrid(in) -> write_pgrid(out)
//   io_tool sigset <in> <out>      read_sigset(in) -> write_sigset(out)
//   io_tool sirn   <in> <out>      load_sirn(in) -> write_sirn(out)
//   io_tool psf    <P> <pitch> <spectrum.f64> <out.f64>   (interleaved re, im)
// Exit 0 on success, 2 ValidationError, 3 NumericalError; the message goes
// to stdout as "error: <message>".
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "pact/aberration.hpp"
#include "pact/io.hpp"
#include "pact/nfield.hpp"

static std::vector<double> read_f64(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  std::vector<double> v;
  double x;
  while (is.read(reinterpret_cast<char*>(&x), sizeof x)) v.push_back(x);
  return v;
}

int main(int argc, char** argv) {
  if (argc < 4) {
    std::cerr << "usage: io_tool pgrid|sigset|sirn|psf ...\n";
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "pgrid") {
      pact::io::write_pgrid(argv[3], pact::io::read_pgrid(argv[2]));
    } else if (cmd == "sigset") {
      pact::io::write_sigset(argv[3], pact::io::read_sigset(argv[2]));
    } else if (cmd == "sirn") {
      pact::write_sirn(argv[3], pact::load_sirn(argv[2]));
    } else if (cmd == "psf" && argc == 6) {
      const int P = std::stoi(argv[2]);
      const double pitch = std::stod(argv[3]);
      const std::vector<double> raw = read_f64(argv[4]);
      std::vector<pact::cplx> sp(raw.size() / 2);
      for (size_t i = 0; i < sp.size(); ++i) sp[i] = {raw[2 * i], raw[2 * i + 1]};
      const pact::RasterGrid r = pact::psf_from_transfer(sp, P, pitch);
      std::ofstream os(argv[5], std::ios::binary);
      os.write(reinterpret_cast<const char*>(r.values.data()),
               static_cast<std::streamsize>(sizeof(double) * r.values.size()));
      std::cout << r.origin.x << " " << r.origin.y << "\n";
    } else {
      std::cerr << "bad command\n";
      return 1;
    }
  } catch (const pact::ValidationError& e) {
    std::cout << "error: " << e.what() << "\n";
    return 2;
  } catch (const pact::NumericalError& e) {
    std::cout << "error: " << e.what() << "\n";
    return 3;
  }
  return 0;
}
