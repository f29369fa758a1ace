// dbag_solve — C++ host driver over the drop-in header (include/dbag.hpp):
// what `dba solve --solver admm` (tools/dba_main.cpp:231-259) does, on the B200.
//   dbag_solve <config 1..5> <rounds> [l2|huber] [exact|fast] [scale] [points_per_block]
//              [cameras_per_block]
//       generate a BASELINE config scene, solve (BlockConfig, default {1,1}),
//       print the metrics CSV
//   dbag_solve file <problem.txt> <rounds> [l2|huber] [exact|fast] [solved.txt] [metrics.csv]
//       parse a reference problem file (bal_io.hpp format), solve from its
//       record, write the solved problem and the metrics CSV (metrics_csv.hpp)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "dbag.hpp"

static int solve_file(int argc, char** argv) {
  if (argc < 4) return 2;
  std::ifstream in(argv[2], std::ios::binary);
  if (!in) {
    std::fprintf(stderr, "cannot open '%s'\n", argv[2]);
    return 3;
  }
  std::ostringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  dbag_bal* b = nullptr;
  int32_t m = 0, n = 0;
  int64_t l = 0;
  if (dbag_parse_problem_text(text.data(), text.size(), &b, &m, &n, &l) != DBAG_OK) {
    int32_t line = -1;
    std::fprintf(stderr, "data error: %s\n", dbag_io_last_error(&line));
    return 3;
  }
  dba::gpu::Problem problem;
  problem.obs_cam.resize(l);
  problem.obs_pt.resize(l);
  problem.obs_uv.resize(2 * l);
  problem.nominal.cam_pose.resize(6 * m);
  problem.nominal.cam_f.resize(m);
  problem.nominal.points.resize(3 * n);
  dbag_bal_fetch(b, problem.obs_cam.data(), problem.obs_pt.data(), problem.obs_uv.data(),
                 problem.nominal.cam_pose.data(), problem.nominal.cam_f.data(),
                 problem.nominal.points.data());
  dbag_bal_destroy(b);
  dba::gpu::AdmmOptions opts;
  opts.max_iters = std::atoi(argv[3]);
  opts.misfit_loss = argc > 4 && std::strcmp(argv[4], "huber") == 0
                         ? dba::gpu::LossKind::huber(1.0)
                         : dba::gpu::LossKind::squared_l2();
  opts.numerics = argc > 5 && std::strcmp(argv[5], "fast") == 0 ? DBAG_NUMERICS_FAST
                                                                 : DBAG_NUMERICS_EXACT;
  try {
    const dba::gpu::AdmmResult res = dba::gpu::run_admm(problem, problem.nominal_state(), opts);
    auto write = [](const char* path, auto fill) {
      size_t len = 0;
      fill(nullptr, 0, &len);
      std::string buf(len + 1, '\0');
      fill(buf.data(), buf.size(), &len);
      std::ofstream out(path, std::ios::binary | std::ios::trunc);
      out.write(buf.data(), (std::streamsize)len);
    };
    if (argc > 6) {
      const dbag_problem_view pv = problem.view();
      const dbag_param_view sv = res.state.view();
      write(argv[6], [&](char* o, size_t c, size_t* len) {
        dbag_serialize_problem_text(&pv, &sv, o, c, len);
      });
    }
    if (argc > 7)
      write(argv[7], [&](char* o, size_t c, size_t* len) {
        dbag_metrics_csv(res.trace.data(), (int64_t)res.trace.size(), o, c, len);
      });
    std::printf("rounds=%zu final_mean_reproj_err=%.17g\n", res.trace.size(),
                res.trace.empty() ? 0.0 : res.trace.back().mean_reproj_err);
  } catch (const dba::gpu::ValidationError& e) {
    std::fprintf(stderr, "data error: %s\n", e.what());
    return 3;
  } catch (const dba::gpu::Error& e) {
    std::fprintf(stderr, "solver error: %s\n", e.what());
    return 4;
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "file") == 0) return solve_file(argc, argv);
  const int config = argc > 1 ? std::atoi(argv[1]) : 1;
  const int rounds = argc > 2 ? std::atoi(argv[2]) : 50;
  const bool huber = argc > 3 && std::strcmp(argv[3], "huber") == 0;
  const bool fast = argc > 4 && std::strcmp(argv[4], "fast") == 0;
  const double scale = argc > 5 ? std::atof(argv[5]) : 1.0;
  dba::gpu::BlockConfig blocks;
  blocks.points_per_block = argc > 6 ? std::atoi(argv[6]) : 1;
  blocks.cameras_per_block = argc > 7 ? std::atoi(argv[7]) : 1;
  dbag_scene* sc = nullptr;
  dbag_scene_info info{};
  if (dbag_scene_generate(config, 0, scale, &sc, &info) != DBAG_OK) {
    std::fprintf(stderr, "scene generation failed\n");
    return 3;
  }
  const int m = info.num_cameras, n = info.num_points;
  const int64_t l = info.num_obs;
  dba::gpu::Problem problem;
  problem.obs_cam.resize(l);
  problem.obs_pt.resize(l);
  problem.obs_uv.resize(2 * l);
  problem.nominal.cam_pose.resize(6 * m);
  problem.nominal.cam_f.resize(m);
  problem.nominal.points.resize(3 * n);
  dba::gpu::ParamState init;
  init.cam_pose.resize(6 * m);
  init.points.resize(3 * n);
  dbag_scene_fetch(sc, problem.obs_cam.data(), problem.obs_pt.data(), problem.obs_uv.data(),
                   problem.nominal.cam_pose.data(), problem.nominal.cam_f.data(),
                   problem.nominal.points.data(), init.cam_pose.data(), init.points.data());
  dbag_scene_destroy(sc);
  init.cam_f = problem.nominal.cam_f;
  dba::gpu::AdmmOptions opts;
  opts.max_iters = rounds;
  opts.misfit_loss = huber ? dba::gpu::LossKind::huber(1.0) : dba::gpu::LossKind::squared_l2();
  opts.numerics = fast ? DBAG_NUMERICS_FAST : DBAG_NUMERICS_EXACT;
  try {
    const dba::gpu::ParamState truth = problem.nominal_state();
    const dba::gpu::AdmmResult res = dba::gpu::run_admm(problem, init, opts, blocks, &truth);
    std::printf("iter,mean_reproj_err,max_primal_x,max_primal_y,camera_mse,point_mse,wall_ms,comm_floats\n");
    for (const auto& r : res.trace)
      std::printf("%d,%.17g,%.17g,%.17g,%.17g,%.17g,%.6g,%lld\n", r.iter, r.mean_reproj_err,
                  r.max_primal_x, r.max_primal_y, r.camera_mse, r.point_mse, r.wall_ms,
                  static_cast<long long>(r.comm_floats));
  } catch (const dba::gpu::ValidationError& e) {
    std::fprintf(stderr, "data error: %s\n", e.what());
    return 3;  // dba_main.cpp exit-code convention (:559-568)
  } catch (const dba::gpu::Error& e) {
    std::fprintf(stderr, "solver error: %s\n", e.what());
    return 4;
  }
  return 0;
}
