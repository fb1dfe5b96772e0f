// Minimal C++ use of the reference-shaped facade: order a station x day dataset,
// seed sts inducing points, search d_r neighbours, build a VIF structure and
// evaluate the NLL and its gradient (the estimation.cpp Objective step).
#include <cstdio>
#include <random>
#include <vector>

#include "stgp_b200.hpp"

int main(int argc, char** argv) {
  using namespace stgp_b200;
  const int stations = argc > 1 ? std::atoi(argv[1]) : 200, days = argc > 2 ? std::atoi(argv[2]) : 10;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::normal_distribution<double> g(0.0, 1.0);
  std::vector<double> sx(stations), sy(stations);
  for (int s = 0; s < stations; ++s) {
    sx[s] = u(rng);
    sy[s] = u(rng);
  }
  std::vector<double> x, y, t, resp;
  for (int d = 1; d <= days; ++d)
    for (int s = 0; s < stations; ++s) {
      x.push_back(sx[s]);
      y.push_back(sy[s]);
      t.push_back(d);
      resp.push_back(g(rng));
    }
  const auto perm = order_observations(t, 42);
  std::vector<double> ox, oy, ot, oresp;
  for (int i : perm) {
    ox.push_back(x[i]);
    oy.push_back(y[i]);
    ot.push_back(t[i]);
    oresp.push_back(resp[i]);
  }
  try {
    Context ctx(0);
    SpaceTimeDataset ds(ctx, ox, oy, ot);
    const CovarianceParams theta{0.01, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2};
    InducingSet ind = sts_kmeanspp(ds, 60, 42);
    NeighborSets nb = residual_neighbors(ds, theta, ind, 20);
    Structure s = build_vif(ds, theta, ind, nb, DiagonalPolicy::kObservation);
    const double v = nll(s, oresp);
    const std::vector<double> gr = nll_grad(s, oresp);
    std::printf("n=%d M=%d nll=%.10f grad[0]=%.6e\n", ds.n(), ind.size(), v, gr[0]);
    // the precipitation path: ZC-PTN amounts (censored at 0) through the Laplace algebra of a FITC structure
    std::vector<double> amounts(oresp.size());
    for (size_t i = 0; i < oresp.size(); ++i) amounts[i] = oresp[i] > 0.3 ? oresp[i] : 0.0;
    const CovarianceParams latent{0.0, 1.0, 0.5, 20.0, 0.4, 1.5, 0.4, 0.2};
    Structure f = build_fitc(ds, latent, ind);
    const LikelihoodParams lik{0.8, 1.5};
    auto lm = laplace_marginal(f, amounts, {}, 0, {}, lik);
    const std::vector<double> target{ox[0], oy[0], ot.back() + 1.0};
    const ZcptnPrediction zp = zcptn_predict(lm.second, f, target, {}, 0, {}, lik, 0, 16, 3);
    std::printf("laplace nll=%.10f iterations=%d p_rain=%.6f\n", lm.first, lm.second.iterations, zp.p_rain[0]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
