// Stand-in for the reference's sweptnet/nn.hpp interface (member names and types of MlpT,
// Vec3, Motion and the two inference functions, nn.hpp:16-44,92-93,162-163), on the mock
// Eigen above: lets tests/test_integration_shim.py compile the INTEGRATION.md shim.
#pragma once
#include <utility>
#include <vector>

#include <Eigen/Dense>

namespace sweptnet {

using Vec3 = Eigen::Vector3d;

struct Motion {
    Eigen::VectorXd q0, q1;
};

template <class S>
struct MlpT {
    using Mat = Eigen::Matrix<S, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
    using Wmat = Eigen::Matrix<S, Eigen::Dynamic, Eigen::Dynamic>;
    using Vec = Eigen::Matrix<S, Eigen::Dynamic, 1>;
    struct Block {
        Wmat weight;
        Vec bias, gamma, beta, running_mean, running_var;
    };
    int n_blocks = 0, block_dim = 0, input_dim = 0;
    Vec norm_shift, norm_scale;
    Wmat input_weight;
    Vec input_bias;
    std::vector<Block> blocks;
    Vec output_weight;
    S output_bias = 0;
    int dof() const { return (input_dim - 3) / 2; }
};

using Mlp = MlpT<float>;

template <class S>
typename MlpT<S>::Vec forward_eval(const MlpT<S>& model, const typename MlpT<S>::Mat& raw);

std::pair<double, int> predict_min_distance(const Mlp& model, const std::vector<Vec3>& cloud, const Motion& m);

}  // namespace sweptnet
