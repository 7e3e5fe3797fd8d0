// reconstruct_demo.cpp — drives the reference's UNMODIFIED optimiser
// (run_coarse_to_fine, coarse_to_fine.cpp:112-192: total_loss -> adam_step ->
// robust_evolve per iteration) on a synthetic blob. Linked twice by
// integration/Makefile: against the reference alone (demo_ref) and with the
// hot path resolved to the B200 shim (demo_b200). Prints one JSON line with
// ms per optimisation iteration and the total_loss share.
//
//   demo_{ref,b200} [views=8] [image=256] [spp=4] [iters=3] [subdiv=5] [tex=256] [threads=N]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "collodiff/camera.hpp"
#include "collodiff/losses.hpp"
#include "collodiff/mesh.hpp"
#include "collodiff/optimize.hpp"
#include "collodiff/params.hpp"
#include "collodiff/render.hpp"

using namespace collodiff;
using clk = std::chrono::steady_clock;

static double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

int main(int argc, char** argv) {
    auto arg = [&](int i, int d) { return argc > i ? std::atoi(argv[i]) : d; };
    const int views = arg(1, 8), image = arg(2, 256), spp = arg(3, 4), iters = arg(4, 3), subdiv = arg(5, 5),
              tex = arg(6, 256);
    const int threads = arg(7, int(std::thread::hardware_concurrency()));
    const int stages = arg(8, 1);  // > 1: coarse-to-fine with remesh + texture doubling per stage

    Scene gt;
    gt.mesh = make_blob(subdiv, 5, 0.15);
    build_adjacency(gt.mesh);
    gt.maps = make_constant_maps(tex, Vec3(0.6, 0.45, 0.35), Vec3(0.08, 0.08, 0.08), 0.35);
    gt.light.intensity = Vec3(20, 20, 20);
    gt.views = sample_views_on_sphere(views, 2.5, 11, 40.0, image, image);

    LossOptions opt;
    opt.render.spp = spp;
    opt.render.seed = 1;
    opt.render.threads = threads;
    RenderSettings ts = opt.render;
    ts.seed = opt.render.seed + 0x7a9;
    std::vector<Image> targets;
    {
        SceneContext ctx(gt);
        for (int k = 0; k < views; ++k) targets.push_back(render(gt, ctx, k, ts));
    }

    Scene init = gt;
    init.mesh = make_icosphere(subdiv, 0.5);
    init.maps = make_constant_maps(tex, Vec3(0.5, 0.5, 0.5), Vec3(0.05, 0.05, 0.05), 0.5);

    LossWeights w;
    auto layout = ParamLayout::for_scene(init, false);
    auto t0 = clk::now();
    TotalLossResult tl = total_loss(init, targets, w, opt, layout);
    double t_loss = secs(t0, clk::now());
    if (const char* dump = std::getenv("CDR_DEMO_DUMP")) {  // the first gradient, raw fp64 (tests)
        if (FILE* f = std::fopen(dump, "wb")) {
            std::fwrite(tl.grad.values.data(), sizeof(double), tl.grad.values.size(), f);
            std::fclose(f);
        }
    }

    StagePlan plan;
    for (int si = 0; si < stages; ++si) {
        Stage st;
        st.iterations = iters;
        st.edge_length = 0.04 / std::pow(1.4, si);  // a remesh at every stage change
        st.texture_resolution = tex;  // (doubling trips the reference's own moment carry: "moment upsample size mismatch")
        st.lr_positions = 1e-3 * init.mesh.bbox_diagonal();
        plan.stages.push_back(st);
    }
    CoarseToFineConfig cfg;
    const int metric = arg(9, 0);  // 1: point-to-mesh metric vs the ground truth every iteration
    if (metric) {
        cfg.ground_truth = &gt.mesh;
        cfg.verify_safety = true;
    }
    std::vector<double> it_s;
    auto last = clk::now();
    cfg.on_iteration = [&](const IterationRecord&) {
        auto now = clk::now();
        it_s.push_back(secs(last, now));
        last = now;
    };
    last = clk::now();
    CoarseToFineResult r = run_coarse_to_fine(init, targets, plan, w, opt, cfg);
    double mean = 0;
    for (double s : it_s) mean += s;
    mean /= std::max<size_t>(1, it_s.size());
    std::printf("{\"tris\": %d, \"views\": %d, \"image\": %d, \"spp\": %d, \"threads\": %d, "
                "\"ms_per_iteration\": %.3f, \"ms_total_loss\": %.3f, \"loss0\": %.17g, \"rend0\": %.17g, "
                "\"lap0\": %.17g, \"normal0\": %.17g, \"edge0\": %.17g, \"spec0\": %.17g, \"roug0\": %.17g, "
                "\"loss_last\": %.17g, \"iterations\": %zu, \"stages\": %d, \"tris_final\": %d, "
                "\"p2m_last\": %.12g, \"safety_ok\": %d}\n",
                gt.mesh.triangle_count(), views, image, spp, threads, 1e3 * mean, 1e3 * t_loss,
                tl.breakdown.total, tl.breakdown.rend, tl.breakdown.lap, tl.breakdown.normal, tl.breakdown.edge,
                tl.breakdown.spec, tl.breakdown.roug,
                r.log.empty() ? 0.0 : r.log.back().loss.total, r.log.size(), stages,
                r.scene.mesh.triangle_count(), r.log.empty() ? 0.0 : r.log.back().point_to_mesh,
                r.log.empty() ? 0 : int(r.log.back().safety_ok));
    return 0;
}
