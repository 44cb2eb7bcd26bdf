// Host-side LLaPor model: every field of an LLPC v1 checkpoint (save_checkpoint /
// load_checkpoint, predictor.cpp:833-929), so a loaded model can be fine-tuned online
// (fine_tune, predictor.cpp:654-663) and saved back byte-compatibly. Inference runs on
// the GPU (K4, k4_llapor.cu) from the device copy uploaded after each change.
#pragma once

#include <cstdint>
#include <vector>

#include "ps_api.h"

namespace ps {

struct HostBlk {  // LinearBlock: w [rows x cols] row-major, b [rows]
  int rows = 0, cols = 0;
  std::vector<double> w, b;
};

struct HostNet {  // LLaPorNet (predictor.hpp:58-75)
  int target = 0, group = 1, E = 0;
  double dropout = 0.1;
  std::vector<double> mean;           // PcaBasis (predictor.hpp:27-35)
  int p_rows = 0, p_cols = 0;         // components [effective_dim x hidden_dim]
  std::vector<double> comp, eigen;
  int req_dim = 0, eff_dim = 0;
  std::vector<HostBlk> blocks, res;   // GELU blocks, middle-group residual blocks
  std::vector<double> gate_w;         // middle-group gate over the PCA features
  double gate_b = 0;
  HostBlk out;
};

struct GroupHyperH {  // GroupHyper (predictor.hpp:86-92)
  double base_lr = 1e-3, weight_decay = 1e-4;
  int pca_dim = 8, width = 32, num_blocks = 2;
};

struct TrainCfgH {  // TrainConfig defaults (predictor.hpp:94-112)
  double lambda = 1.0, gamma = 2.0;
  int epochs = 30, warmup = 5;
  GroupHyperH input{3e-3, 1e-4, 8, 32, 2}, middle{3e-3, 1e-3, 16, 48, 3}, output{3e-3, 1e-4, 8, 32, 2};
  double dropout = 0.1, noise = 0.01, mask = 0.05;
  int batch_size = 32;
  uint64_t seed = 0;
  const GroupHyperH& for_group(int g) const { return g == 0 ? input : g == 1 ? middle : output; }
};

struct HostModel {
  ps_model_spec spec{};
  uint64_t checksum = 0;
  TrainCfgH cfg;
  std::vector<HostNet> nets;  // index = target layer; nets[0] untrained
};

struct HostSample {  // Sample (predictor.hpp:155-158): features of layer l-1, labels of l
  std::vector<double> reduced, onehot, gate, labels;
};

HostModel read_llpc(const char* path);
void write_llpc(const HostModel& m, const char* path);
std::vector<double> host_pca_apply(const HostNet& net, const double* v);
void host_fine_tune(HostNet& net, const std::vector<HostSample>& samples, int steps, double lr, const TrainCfgH& cfg);

}  // namespace ps
