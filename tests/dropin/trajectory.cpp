// TEST INFRASTRUCTURE: one MEFT training run through the reference's public trainer API (meft::train), printed as
// plain numbers so two builds of this same file can be compared line by line:
//   * against the reference library (all of proj/src, CPU)              -> oracle/_ref/tests/trajectory
//   * against the drop-in (the trainer's own sources + libmeft_dropin)  -> build/dropin_tests/trajectory
// tests/test_dropin.py runs both and checks the B200 trajectory (losses, final adapter weights and moments, Adam
// counters, EM) against the CPU one. Usage: trajectory <mode: meft|dense> <experts> <budget>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "meft/dataset.hpp"
#include "meft/trainer.hpp"

using namespace meft;

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "meft";
    TrainOptions opt;
    opt.model.vocab = 48;
    opt.model.dim = 16;
    opt.model.layers = 2;
    opt.model.ffn_width = 24;
    opt.model.pairs = 64;
    opt.model.experts = argc > 2 ? std::atol(argv[2]) : 8;
    opt.model.experts_per_token = 2;
    opt.model.budget = argc > 3 ? std::atol(argv[3]) : 8;
    opt.model.max_seq = 16;
    opt.model.seed = 7;
    opt.schedule.epochs = 3;
    opt.schedule.batch_size = 2;
    opt.schedule.seq_len = 14;
    opt.schedule.accum_batch_size = 4;
    opt.schedule.peak_lr = 3e-3;
    opt.mode = mode == "dense" ? TierMode::Dense : TierMode::Meft;
    opt.eval_subset = 0;
    opt.final_eval = true;
    const FactDataset data = gen_fact_dataset(32, opt.model.vocab, 2, 4, 5);
    const TrainResult r = train(opt, data);

    std::printf("steps %lld\n", static_cast<long long>(r.steps));
    for (size_t i = 0; i < r.step_losses.size(); ++i) std::printf("loss %zu %.17g\n", i, r.step_losses[i]);
    std::printf("em %.17g\n", r.final_em);
    for (index_t l = 0; l < r.store.layers(); ++l) {
        const HostLayer& L = r.store.layer(l);
        const Matrix* tabs[] = {&L.adapter.w_a, &L.adapter.w_b, &L.m_a, &L.v_a, &L.m_b, &L.v_b};
        const char* names[] = {"w_a", "w_b", "m_a", "v_a", "m_b", "v_b"};
        for (int k = 0; k < 6; ++k)
            for (index_t i = 0; i < tabs[k]->size(); ++i)
                std::printf("%s %lld %lld %.17g\n", names[k], static_cast<long long>(l), static_cast<long long>(i),
                            tabs[k]->data[static_cast<size_t>(i)]);
        for (size_t j = 0; j < L.pair_step.size(); ++j)
            std::printf("pair_step %lld %zu %lld\n", static_cast<long long>(l), j,
                        static_cast<long long>(L.pair_step[j]));
    }
    return 0;
}
