// Host-side types shared by the C ABI and the CUDA engine.
//
// The error taxonomy mirrors the reference (src/fastlk/error.hpp:12-39) so
// the C ABI maps failures to the same status codes (capi.cpp:30-48); the
// configuration struct carries the same 13 keys with the same defaults
// (fastlk.h:76-78, frontend.hpp:17-24, fast.hpp:20-24, nms.hpp:17-22,
// lk.hpp:40-48).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace flkb {

struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidArgument : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // -> FLK_E_INTERNAL

enum class ScoreKind : int { kSadB = 0, kSadA = 1, kMt = 2 };
enum class ParamMode : int { kTranslation, kTranslationOffset, kTranslationGain, kFull };

struct Config {
  // FAST (fast.hpp:20-24)
  int epsilon = 10;
  int arc_length = 10;
  ScoreKind score = ScoreKind::kSadB;
  // grid (nms.hpp:17-22)
  int cell_width_units = 1;
  int cell_height_units = 32;
  int num_levels = 1;
  int nms_radius = 1;
  // tracker keys: parsed and validated for config compatibility (lk.hpp:40-48)
  ParamMode mode = ParamMode::kFull;
  int max_iterations = 30;
  double convergence_epsilon = 0.01;
  // frontend (frontend.hpp:21-23)
  int target_count = 100;
  double redetect_ratio = 0.3;
  int threads = 0;
  // B200 extension: cell size in level-0 pixels, 0 = reference geometry
  int cell_width_px = 0;
  int cell_height_px = 0;

  int cell_width() const { return cell_width_px > 0 ? cell_width_px : 32 * cell_width_units; }
  int cell_height() const {
    return cell_height_px > 0 ? cell_height_px : (1 << (num_levels - 1)) * cell_height_units;
  }
};

// validate(FrontendConfig) (frontend.cpp:26-36): range errors are
// InvalidArgument, target/ratio errors ConfigError.
void validate(const Config& cfg);

// apply_config_entry / load_config_file (config.cpp:70-131).
void apply_config_entry(Config* cfg, const std::string& key, const std::string& value);
void load_config_file(Config* cfg, const std::string& path);

// Page-locked host memory for frame pixels, from a size-keyed pool, so a
// frame can be DMA'd to the GPU straight from its flk_image (no staging copy).
// Falls back to ordinary memory when pinning is unavailable (no driver /
// device, or the pinned budget is exhausted).
void* pinned_acquire(size_t bytes);
void pinned_release(void* p, size_t bytes) noexcept;
bool pinned_contains(const void* p);

template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) { return static_cast<T*>(pinned_acquire(n * sizeof(T))); }
  void deallocate(T* p, size_t n) noexcept { pinned_release(p, n * sizeof(T)); }
  template <class U>
  bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const PinnedAlloc<U>&) const { return false; }
};

// Tightly packed host raster (the C ABI copies into this, capi.cpp:134-149).
struct HostImage {
  int width = 0;
  int height = 0;
  std::vector<uint8_t, PinnedAlloc<uint8_t>> px;
  bool pinned() const { return !px.empty() && pinned_contains(px.data()); }
};

HostImage make_image(int width, int height, const uint8_t* pixels);
HostImage load_pgm(const std::string& path);     // image.cpp:86-140
void save_pgm(const HostImage& img, const std::string& path);  // image.cpp:142-170

}  // namespace flkb
