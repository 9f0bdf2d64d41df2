// devinfo.hpp -- DEVINFO for the B200 backend (third "next"
// row): the reference's 12-attribute device record
// (proj/include/gpc/devinfo.hpp:23-38) filled from cudaGetDeviceProperties
// for the bound GPUs, rendered in the reference's canonical XML
// (proj/src/devinfo.cpp:94-125: fixed prolog, 2-space indent, snake_case
// tags, index attribute, triples as three integers, &<> escaped).
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

namespace gpcx::devinfo {

struct DeviceInfo {
  std::string name;
  std::string compute_capability;
  int warp_size = 0;
  std::uint64_t total_constant_memory = 0;
  std::uint64_t total_global_memory = 0;
  std::uint64_t shared_memory_per_block = 0;
  std::int64_t clock_rate_khz = 0;
  int multi_processor_count = 0;
  int registers_per_block = 0;
  int max_threads_per_block = 0;
  std::array<int, 3> max_grid_size{0, 0, 0};
  std::array<int, 3> max_threads_dim{0, 0, 0};
};

// CUDA prober over the given device ordinals (never throws: a device that
// cannot be queried is skipped).
std::vector<DeviceInfo> probe_cuda(const std::vector<int>& devices);
std::string to_xml(std::span<const DeviceInfo> devices);

}  // namespace gpcx::devinfo
