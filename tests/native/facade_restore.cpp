// Checkpoint/resume through the drop-in C++ facade (paper_2005_07547_b200/cxx): fill a store with
// the reference's scalar API, dumpSnapshot, loadSnapshot (the facade's extension over
// pstf_field_load_snapshot) into a fresh store, dumpSnapshot again.  The two files must be
// byte-identical and every query must return the same committed value.  A snapshot of another
// field kind must be refused with std::runtime_error.  Exit status 0 = pass.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "pstf/field.h"

using namespace pstf;

static std::vector<char> slurp(const std::string &p) {
    std::ifstream f(p, std::ios::binary);
    return std::vector<char>(std::istreambuf_iterator<char>(f), {});
}

int main(int argc, char **argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    FieldStoreConfig cfg;
    cfg.capacityLog2 = 14;
    cfg.baseCellSize = 0.25;
    FieldStore a(cfg);
    Rng rng(7, 1);
    std::vector<Vec3> pos, dirs;
    for (int i = 0; i < 3000; ++i) {
        Vec3 p{rng.next1D() * 8.0 - 4.0, rng.next1D() * 8.0 - 4.0, rng.next1D() * 8.0 - 4.0};
        Vec3 d = normalize(Vec3{rng.next1D() - 0.5, rng.next1D() - 0.5, rng.next1D() - 0.5});
        pos.push_back(p);
        dirs.push_back(d);
    }
    for (int frame = 0; frame < 3; ++frame) {
        for (size_t i = 0; i < pos.size(); ++i) {
            SpatioDirectionalKey k = a.keyFor(pos[i], dirs[i], int(i % 4));
            a.incrementCounter(k, 1.0);
            a.accumulate(k, RGB(rng.next1D(), rng.next1D(), rng.next1D()), 1.0);
        }
        a.endFrame();
    }
    const std::string fa = dir + "/facade_a.snap", fb = dir + "/facade_b.snap";
    a.dumpSnapshot(fa);
    FieldStore b(cfg);
    b.loadSnapshot(fa);
    b.dumpSnapshot(fb);
    if (slurp(fa) != slurp(fb) || slurp(fa).size() < 1000) {
        std::fprintf(stderr, "snapshot files differ after loadSnapshot\n");
        return 1;
    }
    if (a.liveCellCount() != b.liveCellCount()) return 2;
    for (size_t i = 0; i < pos.size(); i += 7) {
        FieldQueryResult qa = a.queryFromLevel(pos[i], dirs[i], int(i % 4));
        FieldQueryResult qb = b.queryFromLevel(pos[i], dirs[i], int(i % 4));
        if (qa.valid != qb.valid || qa.value.r != qb.value.r || qa.value.g != qb.value.g ||
            qa.value.b != qb.value.b || qa.level != qb.level)
            return 3;
    }
    FieldStoreConfig other = cfg;
    other.kind = FieldKind::FLi;
    FieldStore c(other);
    try {
        c.loadSnapshot(fa);
        return 4;
    } catch (const std::runtime_error &) {
    }
    std::printf("facade restore ok: %zu live cells\n", b.liveCellCount());
    return 0;
}
