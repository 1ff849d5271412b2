// oracle/_ref/ref_terrain_io — the reference's heightmap text I/O
// (save_heightmap / load_heightmap, terrain.hpp:334-415) as a command-line
// tool.  TEST INFRASTRUCTURE ONLY: a separate process, so the reference's
// iostreams never share a process with the Python interpreter's libstdc++.
//   ref_terrain_io save <heights.f64> <nx> <ny> <origin_x> <origin_y> <res> <out.txt>
//   ref_terrain_io load <in.txt> <out.f64>     (out: ox oy res nx ny heights...)
// Exit 0 ok; 2 ConfigError (message on stdout).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "tmpc/terrain.hpp"

using namespace tmpc;

int main(int argc, char** argv) {
  try {
    if (argc == 9 && std::string(argv[1]) == "save") {
      Heightmap hm;
      hm.grid = GridSpec{std::strtod(argv[5], nullptr), std::strtod(argv[6], nullptr),
                         std::strtod(argv[7], nullptr), std::atoi(argv[3]), std::atoi(argv[4])};
      hm.heights.resize(static_cast<size_t>(hm.grid.nx) * hm.grid.ny);
      std::ifstream in(argv[2], std::ios::binary);
      in.read(reinterpret_cast<char*>(hm.heights.data()),
              static_cast<std::streamsize>(hm.heights.size() * sizeof(double)));
      save_heightmap(hm, std::string(argv[8]));
      return 0;
    }
    if (argc == 4 && std::string(argv[1]) == "load") {
      const Heightmap hm = load_heightmap(std::string(argv[2]));
      std::vector<double> out = {hm.grid.origin_x, hm.grid.origin_y, hm.grid.resolution,
                                 static_cast<double>(hm.grid.nx), static_cast<double>(hm.grid.ny)};
      out.insert(out.end(), hm.heights.begin(), hm.heights.end());
      std::ofstream o(argv[3], std::ios::binary);
      o.write(reinterpret_cast<const char*>(out.data()),
              static_cast<std::streamsize>(out.size() * sizeof(double)));
      return 0;
    }
    std::fprintf(stderr, "usage: ref_terrain_io save|load ...\n");
    return 1;
  } catch (const std::exception& e) {
    std::printf("%s", e.what());
    return 2;
  }
}
