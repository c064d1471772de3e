// Reference-style caller of the B200 drop-in (include/ttsvd_b200.hpp): the
// same code a user of /root/reference/proj/include/ttsvd would write.
//   g++ -std=c++20 -Iinclude -I/usr/local/cuda/include examples/dropin_example.cpp
//       -Lpaper_2102_00104_b200 -lttsvd_cu -L/usr/local/cuda/lib64 -lcudart
// Without a GPU (argv[1] == "host") only host-side entry points run.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "ttsvd_b200.hpp"

int main(int argc, char** argv) {
    using namespace ttsvd;
    if (padded_stride(262144) != 262208) return 1;
    if (select_rank({2, 1, 0.5, 0.1}, 0.2, 10) != 3) return 2;
    if (derive_delta(2.0, 0.1, 5) < 0.0999999 || derive_delta(2.0, 0.1, 5) > 0.1000001) return 3;
    try {
        derive_delta(1.0, 0.1, 1);
        return 4;
    } catch (const DegenerateDimension&) {
    }
    if (choose_combined_dims({4, 4, 4, 4, 4, 4, 4, 4, 4, 4}, ThickBoundsParams{}, 16) != std::make_pair<index_t, index_t>(3, 64))
        return 6;
    if (argc > 1 && std::strcmp(argv[1], "host") == 0) {
        // wire formats: "host <dir>" writes a tensor and a train for the
        // reference's loaders to read (tests/test_wire.py) and reads them back
        if (argc > 2) {
            const std::string dir = argv[2];
            DenseTensor T({3, 5, 4});
            for (index_t l = 0; l < T.total(); ++l) T.at_flat(l) = 0.25 * l - 3.0;
            dump_tensor(T, dir + "/cpp_tensor.bin");
            const DenseTensor U = load_tensor(dir + "/cpp_tensor.bin");
            for (index_t l = 0; l < T.total(); ++l)
                if (U.at_flat(l) != T.at_flat(l)) return 7;
            TensorTrain tt;
            const index_t ranks[] = {1, 2, 3, 1}, dims[] = {3, 5, 4};
            for (int j = 0; j < 3; ++j) {
                TTCore c(ranks[j], dims[j], ranks[j + 1]);
                for (std::size_t e = 0; e < c.data.size(); ++e) c.data[e] = 0.5 * (double)e - j;
                tt.cores.push_back(c);
            }
            save_tt(tt, dir + "/cpp_tt.bin");
            const TensorTrain back = load_tt(dir + "/cpp_tt.bin");
            if (back.ranks() != tt.ranks() || back.cores[2].data != tt.cores[2].data) return 8;
            try {
                load_tensor(dir + "/missing.bin");
                return 9;
            } catch (const IoError&) {
            }
        }
        std::printf("host entry points ok\n");
        return 0;
    }
    // device path: 4^8 tensor, entries from a simple deterministic pattern
    DenseTensor X({4, 4, 4, 4, 4, 4, 4, 4});
    for (index_t l = 0; l < X.total(); ++l) X.at_flat(l) = ((l * 7919) % 1000) / 1000.0 - 0.5;
    TruncationSpec spec;
    spec.r_max = 8;
    TensorTrain tt = tt_svd_tsqr(X, spec);
    const auto r = tt.ranks();
    std::printf("ranks:");
    for (auto v : r) std::printf(" %lld", static_cast<long long>(v));
    std::printf("\n");
    ThickBoundsParams tb;
    tb.m_min = 8;
    TensorTrain tk = tt_svd_thick_bounds(X, spec, tb);
    if (tk.cores.size() != 8 || tk.ranks().back() != 1) return 7;
    PaddedMatrix M(1000, 4);
    for (index_t j = 0; j < 4; ++j) M(j, j) = 1.0;
    TriangularFactor R = tsqr(M.view(), BlockParams::for_cols(4), 1);
    for (index_t j = 0; j < 4; ++j)
        if (std::abs(std::abs(R(j, j)) - 1.0) > 1e-14) return 5;
    // Alg. 5 over the GPUs of this process (NCCL inside the library) must
    // agree bitwise with the in-process form: 4 partitions on device 0
    {
        int ndev = 0;
        cudaGetDeviceCount(&ndev);
        std::vector<DenseTensor> slabs;
        for (int p = 0; p < 4; ++p) {
            DenseTensor s(Shape{4, 4, 4, 4, 4, 4, 4});
            for (index_t l = 0; l < s.total(); ++l) s.at_flat(l) = X.at_flat(p + 4 * (l % 4) + 16 * (l / 4) % X.total());
            slabs.push_back(std::move(s));
        }
        std::vector<TensorTrain> parts;
        const TensorTrain a = tt_svd_distributed(slabs, spec, ExecContext{}, &parts);
        const TensorTrain b = tt_svd_distributed(slabs, std::vector<int>{0}, spec);
        if (a.ranks() != b.ranks()) return 10;
        for (std::size_t j = 0; j < a.cores.size(); ++j)
            if (a.cores[j].data != b.cores[j].data) return 11;
        if (parts.size() != 4 || parts[1].cores.front().r_left != 1 || parts[1].cores.front().n != 1) return 12;
        if (ndev >= 2) {  // one partition pair per device
            const TensorTrain c = tt_svd_distributed(slabs, std::vector<int>{0, 1}, spec);
            for (std::size_t j = 1; j < a.cores.size(); ++j)
                if (a.cores[j].data != c.cores[j].data) return 13;
        }
    }
    std::printf("device entry points ok\n");
    return 0;
}
