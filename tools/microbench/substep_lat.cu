// Latency of one 120 Hz single-track substep (the step kernel's substep_dynamic,
// compiled with the library's flags) on one thread: the physics phase's chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I../../include \
//        -I../../paper_2605_08528_b200/csrc substep_lat.cu
#include "../../paper_2605_08528_b200/csrc/drivegrid_b200.cu"

__global__ void substep_chain(double* out, long long* cyc, DgConsts k, int n, double thr, double steer) {
    double x[DG_NUM_STATE];
    for (int f = 0; f < DG_NUM_STATE; ++f) x[f] = 0.0;
    x[SBF] = 1.0;
    x[SBR] = 1.0;
    x[SVX] = 5.0;
    Act a;
    a.thr = thr;
    a.steer = steer;
    a.brk = 0.0;
    const double cap = 1.0 * k.f_z;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) substep_dynamic(x, a, cap, k);
    long long t1 = clock64();
    for (int f = 0; f < DG_NUM_STATE; ++f) out[f] = x[f];
    cyc[0] = t1 - t0;
}

int main() {
    DgConsts k;
    std::memset(&k, 0, sizeof(k));
    k.physics_dt = 1.0 / 120.0; k.control_dt = 1.0 / 30.0;
    k.kp_steer = 1839.5; k.kd_steer = 110.5; k.theta_max = 0.45; k.tau_steer_max = 1200.0;
    k.steer_inertia = 5.0; k.steer_limit = 1.05 * 0.45; k.a_f = 1.3; k.b_r = 1.3;
    k.tau_drive_max = 600.7; k.tau_brake_front = 1090.5; k.tau_brake_rear = 980.7; k.wheel_radius = 0.35;
    k.cornering_stiffness = 60000.0; k.f_z = 0.5 * 1800.0 * 9.81; k.chassis_mass = 1800.0;
    k.lambda_lat = 150.0; k.lambda_yaw = 10.6; k.yaw_inertia = 3000.0; k.i_axle = 2.0 * 1.094 * 0.5 * 37.5 * 0.35 * 0.35;
    k.wheelbase = 2.6;
    double* out; long long* cyc;
    cudaMalloc(&out, 8 * DG_NUM_STATE); cudaMalloc(&cyc, 8);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) substep_chain<<<1, 1>>>(out, cyc, k, n, 0.6, 0.3);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("substep_dynamic: %.1f cycles per substep (one thread)\n", double(h) / n);
    return 0;
}
