"""TEST INFRASTRUCTURE ONLY. Applies the four one-line header fixes to COPIES
of the reference headers under oracle/_ref/include (never to /root/reference, never committed):
  1. comm.hpp: SplitResult holds std::optional<Comm> before Comm is complete -> define it after Comm
  2. comm.hpp: friend `detail_make_world_comm` -> `detail::make_world_comm` (declared first)
  3. dist_matrix.hpp: std::map used without <map>
  4. grid.hpp: RepartitionResult used before its declaration -> forward declaration
"""
import os
import sys

inc = sys.argv[1]
p = os.path.join(inc, "tmg", "comm.hpp")
s = open(p).read()
a = s.index("/// Result of a strided communicator split.")
b = s.index("};", a) + 2
block = s[a:b]
s = s[:a] + "struct SplitResult;\nclass Comm;\nnamespace detail {\nComm make_world_comm(const std::shared_ptr<World>& world, int rank);\n}\n" + s[b:]
s = s.replace("friend Comm detail_make_world_comm(const std::shared_ptr<detail::World>&, int);",
              "friend Comm detail::make_world_comm(const std::shared_ptr<detail::World>&, int);")
c = s.index("class Comm {")
e = s.index("\n};\n", c) + 4
s = s[:e] + "\n" + block + "\n" + s[e:]
open(p, "w").write(s)

p = os.path.join(inc, "tmg", "dist_matrix.hpp")
s = open(p).read()
s = s.replace("#include <memory>", "#include <map>\n#include <memory>", 1)
open(p, "w").write(s)

p = os.path.join(inc, "tmg", "grid.hpp")
s = open(p).read()
s = s.replace("class StructuredGrid {", "struct RepartitionResult;\n\nclass StructuredGrid {", 1)
open(p, "w").write(s)
