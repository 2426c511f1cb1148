// Config 1 end to end (BASELINE configs[0]): the UNMODIFIED reference renderer
// (EstimatorRun with the control-variate estimator, deterministic mode) on a small scene, linked
// either against the reference's own field.cpp (CPU) or against the B200 drop-in facade
// (paper_2005_07547_b200/cxx).  Writes the Lo, Lo\E and FLi field snapshots and the image after
// N frames, so the two builds can be compared byte for byte.
//   config1_{ref,b200} <scene> <size> <frames> <out-prefix> [estimator: cv | is | is-cv | b]
#include <cstdio>
#include <cstdlib>
#include <string>

#include <pstf/estimators.h>
#include <pstf/image.h>
#include <pstf/scene.h>

int main(int argc, char **argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s scene size frames out-prefix\n", argv[0]);
        return 2;
    }
    pstf::Scene scene = pstf::loadScene(argv[1]);
    const int size = std::atoi(argv[2]), frames = std::atoi(argv[3]);
    const std::string out = argv[4];
    scene.camera.width = size;
    scene.camera.height = size;
    pstf::EstimatorConfig c;
    c.kind = pstf::EstimatorKind::CV;
    if (argc > 5 && !pstf::parseEstimatorKind(argv[5], c.kind)) {
        std::fprintf(stderr, "unknown estimator %s\n", argv[5]);
        return 2;
    }
    c.deterministic = true;
    c.threads = 4;
    c.seed = 7;
    c.hashCapacityLog2 = 16;
    c.warmupFrames = 2;
    pstf::EstimatorRun run(scene, c);
    pstf::ImageBuffer img(size, size);
    for (int f = 0; f < frames; ++f) run.renderFrame(&img);
    run.loStore().dumpSnapshot(out + "lo.snap");
    run.loeStore().dumpSnapshot(out + "loe.snap");
    run.fliStore().dumpSnapshot(out + "fli.snap");
    FILE *fp = std::fopen((out + "image.f64").c_str(), "wb");
    for (size_t i = 0; i < img.pixelCount(); ++i) {
        const pstf::RGB p = img.mean(i);
        std::fwrite(&p, sizeof(p), 1, fp);
    }
    std::fclose(fp);
    std::printf("frames %d live lo %zu loe %zu fli %zu\n", frames, run.loStore().liveCellCount(),
                run.loeStore().liveCellCount(), run.fliStore().liveCellCount());
    return 0;
}
