// equirect_check.cu -- the NIF producers' fp32 equirect map (tc_ptx.cuh equirect_f32) against an fp64
// evaluation of the same convention (reading R14) on random unit directions plus the poles,
// the seam and the axes; prints the max |du|, |dv| (in [0,1] units) and where they occur.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Iinclude -Ipaper_2305_20061_b200/csrc -o build/equirect_check tools/equirect_check.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
#include "tc_ptx.cuh"

__global__ void k(const float3* d, float2* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        float u, v;
        pt::equirect_f32(d[i], u, v);
        out[i] = make_float2(u, v);
    }
}

int main() {
    std::mt19937_64 rng(7);
    std::normal_distribution<double> g;
    std::vector<float3> h;
    for (int i = 0; i < (1 << 22); ++i) {
        double x = g(rng), y = g(rng), z = g(rng), l = std::sqrt(x * x + y * y + z * z);
        h.push_back(make_float3((float)(x / l), (float)(y / l), (float)(z / l)));
    }
    // poles, near-poles, seam (d.x = +-0, d.z > 0), axes
    const float e[] = {0.0f, 1e-7f, -1e-7f, 1e-4f, -1e-4f};
    for (float a : e)
        for (float b : e) {
            const double l = std::sqrt((double)a * a + 1.0 + (double)b * b);
            h.push_back(make_float3((float)(a / l), (float)(1.0 / l), (float)(b / l)));
            h.push_back(make_float3((float)(a / l), (float)(-1.0 / l), (float)(b / l)));
            h.push_back(make_float3((float)(a / l), (float)(b / l), (float)(1.0 / l)));
            h.push_back(make_float3((float)(a / l), (float)(b / l), (float)(-1.0 / l)));
        }
    h.push_back(make_float3(-0.0f, 0.0f, 1.0f));
    h.push_back(make_float3(1.0f, 0.0f, 0.0f));
    h.push_back(make_float3(-1.0f, 0.0f, 0.0f));
    const int n = (int)h.size();
    float3* dd;
    float2* dout;
    cudaMalloc(&dd, sizeof(float3) * n);
    cudaMalloc(&dout, sizeof(float2) * n);
    cudaMemcpy(dd, h.data(), sizeof(float3) * n, cudaMemcpyHostToDevice);
    k<<<(n + 255) / 256, 256>>>(dd, dout, n);
    std::vector<float2> o(n);
    cudaMemcpy(o.data(), dout, sizeof(float2) * n, cudaMemcpyDeviceToHost);
    double mu = 0, mv = 0;
    int iu = 0, iv = 0;
    for (int i = 0; i < n; ++i) {
        const double x = h[i].x, y = h[i].y, z = h[i].z, l = std::sqrt(x * x + y * y + z * z);
        double u = (x == 0.0 && z == 0.0) ? 0.5 : 0.5 + std::atan2(x, -z) / (2.0 * M_PI);
        if (u >= 1.0) u -= 1.0;
        const double v = std::acos(std::fmax(-1.0, std::fmin(1.0, y / l))) / M_PI;
        double du = std::fabs(o[i].x - u);
        du = std::fmin(du, 1.0 - du);   // u is periodic
        const double dv = std::fabs(o[i].y - v);
        if (du > mu) { mu = du; iu = i; }
        if (dv > mv) { mv = dv; iv = i; }
    }
    printf("equirect_f32 vs fp64 on %d directions: max |du| %.3g (d = %.9g %.9g %.9g), max |dv| %.3g (d = %.9g %.9g %.9g)\n",
           n, mu, h[iu].x, h[iu].y, h[iu].z, mv, h[iv].x, h[iv].y, h[iv].z);
    return 0;
}
