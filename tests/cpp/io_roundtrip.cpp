// Host-only check of include/kronglm_b200_io.hpp: copy an array file and a CSV
// matrix through read/write, and report the first error message for a bad file.
//   io_roundtrip array IN OUT | csv IN OUT | err-array IN | err-csv IN
#include <cstdio>
#include <string>

#include "kronglm_b200_io.hpp"

int main(int argc, char** argv) {
  namespace io = kronglm_b200::io;
  if (argc < 3) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "array" && argc == 4) {
      io::write_array(argv[3], io::read_array(argv[2]));
    } else if (mode == "csv" && argc == 4) {
      io::write_csv_matrix(argv[3], io::read_csv_matrix(argv[2]));
    } else if (mode == "err-array") {
      io::read_array(argv[2]);
    } else if (mode == "err-csv") {
      io::read_csv_matrix(argv[2]);
    } else {
      return 2;
    }
  } catch (const std::exception& e) {
    std::printf("%s\n", e.what());
    return 1;
  }
  return 0;
}
