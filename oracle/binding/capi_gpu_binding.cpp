// TEST INFRASTRUCTURE ONLY — the reference-side binding of INTEGRATION.md, compiled once.
//
// INTEGRATION.md shows the code a maintainer of the reference would add to proj/src/capi.cpp (the
// reference's only FFI layer, ref: proj/src/capi.cpp:96-139 for the do_run it sits next to).  This
// translation unit is that addition, verbatim, behind an #include of the UNMODIFIED capi.cpp where
// it lies under /root/reference (so the snippet sees the file's own helpers: guarded(), set_error(),
// struct ising_model), linked against the product library.  oracle/Makefile target `binding` builds
// oracle/_ref/libisingmc_b200_binding.so from it plus the reference's own sources; tests load it
// through the reference's C ABI and call the new symbol.  Nothing of the product includes this.
#include "capi.cpp"  // -I $(REF)/src

#include "isingmc_b200.h"

namespace {
// SpinModel -> the CSR arrays flatten() already produces (src/sweep_state.cpp:84-106)
ising_b200_model* to_b200(const SpinModel& m) {
    std::vector<uint32_t> offsets(m.n_spins + 1), targets;
    std::vector<float> couplings;
    std::vector<uint8_t> tau(m.n_spins);
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        offsets[i] = uint32_t(targets.size());
        tau[i] = uint8_t(m.adjacency[i].tau_count);
        for (const EdgeRecord& e : m.adjacency[i].edges) {
            targets.push_back(e.target_spin);
            couplings.push_back(e.coupling);
        }
    }
    offsets[m.n_spins] = uint32_t(targets.size());
    ising_b200_model* out = nullptr;
    const uint32_t layers = m.layered ? m.layered->layers : 0, per = m.layered ? m.layered->per_layer : 0;
    if (ising_b200_model_from_csr(m.n_spins, m.h.data(), offsets.data(), targets.data(), couplings.data(),
                                  tau.data(), layers, per, &out) != ISING_OK) {
        throw Error(ising_b200_last_error());
    }
    return out;
}
}  // namespace

// new entry point of libisingmc: a ladder batch on the GPU
extern "C" ising_status ising_run_batch_gpu(const ising_model* model, const float* betas, uint32_t n_betas,
                                            uint32_t n_ladders, uint32_t base_seed, uint64_t sweeps,
                                            uint32_t swap_interval, int exp_kind, double* energies_out,
                                            uint64_t* flips_out) {
    return guarded([&]() {
        ising_b200_model* gm = to_b200(model->model);
        ising_batch_params p{};
        p.n_ladders = n_ladders; p.n_betas = n_betas; p.betas = betas;
        p.base_seed = base_seed; p.swap_base_seed = base_seed; p.tau_scale = 1.0f;
        p.exp_kind = exp_kind; p.device = 0; p.kernel = ISING_KERNEL_AUTO;
        ising_batch* b = nullptr;
        const ising_b200_model* models[1] = {gm};
        ising_status st = ising_batch_create(models, 1, nullptr, &p, &b);
        if (st == ISING_OK) st = ising_batch_run(b, sweeps, swap_interval);
        if (st == ISING_OK) st = ising_batch_read_energies(b, energies_out);
        if (st == ISING_OK) st = ising_batch_read_stats(b, flips_out, nullptr);
        if (st != ISING_OK) set_error(ising_b200_last_error());
        ising_batch_free(b);
        ising_b200_model_free(gm);
        return st;
    });
}
