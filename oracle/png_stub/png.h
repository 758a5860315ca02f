/* png.h -- TEST INFRASTRUCTURE ONLY.  Minimal stand-in for libpng's "simplified API" so
   the reference's image.cpp / scene.cpp link without libpng (absent in this image).  PNG
   I/O is outside the rendering path: every call reports failure, which the reference turns
   into lumi::Error("png: ..."). */
#ifndef LUMI_PNG_STUB_H
#define LUMI_PNG_STUB_H
#include <stddef.h>
#include <stdint.h>
typedef uint32_t png_uint_32;
typedef struct png_control* png_controlp;
typedef struct {
  png_controlp opaque;
  png_uint_32 version;
  png_uint_32 width;
  png_uint_32 height;
  png_uint_32 format;
  png_uint_32 flags;
  png_uint_32 colormap_entries;
  png_uint_32 warning_or_error;
  char message[64];
} png_image;
#define PNG_IMAGE_VERSION 1
#define PNG_FORMAT_FLAG_COLOR 0x02U
#define PNG_FORMAT_GRAY 0
#define PNG_FORMAT_RGB PNG_FORMAT_FLAG_COLOR
#define PNG_IMAGE_PIXEL_CHANNELS(fmt) (((fmt) & PNG_FORMAT_FLAG_COLOR) ? 3 : 1)
#define PNG_IMAGE_SIZE(img) ((size_t)(img).width * (img).height * PNG_IMAGE_PIXEL_CHANNELS((img).format))
static inline int png_image_write_to_file(png_image*, const char*, int, const void*, int,
                                          const void*) { return 0; }
static inline int png_image_begin_read_from_file(png_image*, const char*) { return 0; }
static inline int png_image_finish_read(png_image*, const void*, void*, int, void*) { return 0; }
#endif
