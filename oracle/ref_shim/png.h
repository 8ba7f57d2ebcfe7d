/* libpng declaration stub — TEST INFRASTRUCTURE ONLY (oracle/_ref).
 *
 * The reference's image.cpp includes <png.h> for load_png (image.cpp:145-184), which is not on the
 * PBA hot path and whose library headers are absent here.  These declarations let the unmodified
 * image.cpp compile; png_stub.c makes png_create_read_struct return NULL, so load_png takes the
 * reference's own failure branch ("load_png: decode failed"), i.e. PNG input is simply unsupported
 * in oracle/_ref.  The hot path reads images from memory. */
#ifndef PBA_REF_PNG_STUB_H
#define PBA_REF_PNG_STUB_H
#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct png_struct_def png_struct;
typedef png_struct* png_structp;
typedef struct png_info_def png_info;
typedef png_info* png_infop;
typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef unsigned int png_uint_32;

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_MASK_COLOR 2

png_structp png_create_read_struct(const char* ver, void* err_ptr, void* err_fn, void* warn_fn);
png_infop png_create_info_struct(png_structp png);
void png_destroy_read_struct(png_structp* png, png_infop* info, png_infop* end_info);
jmp_buf* pba_png_stub_jmpbuf(png_structp png);
#define png_jmpbuf(png) (*pba_png_stub_jmpbuf(png))
void png_init_io(png_structp png, FILE* fp);
void png_read_info(png_structp png, png_infop info);
void png_set_strip_alpha(png_structp png);
png_byte png_get_color_type(png_structp png, png_infop info);
void png_set_rgb_to_gray(png_structp png, int error_action, double red, double green);
png_byte png_get_bit_depth(png_structp png, png_infop info);
void png_set_expand_gray_1_2_4_to_8(png_structp png);
void png_read_update_info(png_structp png, png_infop info);
png_uint_32 png_get_image_width(png_structp png, png_infop info);
png_uint_32 png_get_image_height(png_structp png, png_infop info);
size_t png_get_rowbytes(png_structp png, png_infop info);
void png_read_row(png_structp png, png_bytep row, png_bytep display_row);

#ifdef __cplusplus
}
#endif
#endif
